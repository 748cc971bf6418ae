"""Pinned H2D / D2H bandwidth, alone and overlapped (the e2e ceiling)."""
import torch, time
n = 2 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True); h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d.copy_(h, non_blocking=True); h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
def t(fn):
    torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); return time.perf_counter() - t0
a = t(lambda: d.copy_(h, non_blocking=True))
b = t(lambda: h2.copy_(d2, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
c = t(both)
print(f"H2D {n/a/1e9:.1f} GB/s  D2H {n/b/1e9:.1f} GB/s  overlapped {2*n/c/1e9:.1f} GB/s total ({n/c/1e9:.1f} each)")
# several concurrent copies per direction (several copy engines?)
for k in (2, 4):
    ss = [torch.cuda.Stream() for _ in range(2 * k)]
    part = n // k
    def multi():
        for i in range(k):
            with torch.cuda.stream(ss[i]): d[i * part:(i + 1) * part].copy_(h[i * part:(i + 1) * part], non_blocking=True)
            with torch.cuda.stream(ss[k + i]): h2[i * part:(i + 1) * part].copy_(d2[i * part:(i + 1) * part], non_blocking=True)
    def multi_h2d():
        for i in range(k):
            with torch.cuda.stream(ss[i]): d[i * part:(i + 1) * part].copy_(h[i * part:(i + 1) * part], non_blocking=True)
    e = t(multi_h2d)
    c = t(multi)
    print(f"{k} streams/dir: H2D alone {n/e/1e9:.1f} GB/s; overlapped {n/c/1e9:.1f} GB/s each direction")
