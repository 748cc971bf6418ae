"""Duplex PCIe rate for frame-sized copies: back-to-back cudaMemcpyAsync of
`size` bytes H2D on one stream and D2H on another (pinned host memory), the
Stage II per-frame traffic pattern (three 2 MB planes each way per C3 frame)."""
import sys, time
import torch
for size_mb, count in ((2.0736, 900), (6.2208, 300), (24.8832, 75)):
    nb = int(size_mb * 1e6)
    hin = torch.empty((count, nb), dtype=torch.uint8).pin_memory()
    hout = torch.empty((count, nb), dtype=torch.uint8).pin_memory()
    din = torch.empty((8, nb), dtype=torch.uint8, device="cuda")
    dout = torch.empty((8, nb), dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for mode in ("h2d", "d2h", "both"):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k in range(count):
            if mode in ("h2d", "both"):
                with torch.cuda.stream(s1):
                    din[k % 8].copy_(hin[k], non_blocking=True)
            if mode in ("d2h", "both"):
                with torch.cuda.stream(s2):
                    hout[k].copy_(dout[k % 8], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"{size_mb:.2f} MB x {count} {mode}: {count * nb / dt / 1e9:.1f} GB/s per direction, {dt / count * 1e6:.1f} us per copy")
    del hin, hout
