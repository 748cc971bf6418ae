"""Stage II at a benchmark config with pinned host buffers, straight through
the C ABI (push frame k from a pinned array, pop into a pinned array).
--device: frames already in HBM (push/pop device pointers); --nographs:
one launch per kernel instead of the per-frame CUDA graph; --lag: pop one
push late; --async: the frames released by the previous push are popped with
stabgpu_stream_pop_async before the next push and waited for after it (their
download overlaps the next upload); --depth N (default 2 with --async): the
frames popped before push k are those released by push k-N, so their compose
finished long before and the download runs beside the upload of frame k;
--packed: every frame is one contiguous planar buffer (Y | Cb | Cr) on both
sides, so push and pop move it in one copy; --wait-every M (default 1): stabgpu_stream_wait_pops after every M-th push
only (every popped frame has its own output array here), so the copy queues
of both directions never drain between frames."""
import ctypes as C
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1701_03572_b200 import pipeline, synth
from paper_1701_03572_b200._lib import load, context
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 300
cfg = synth.CONFIGS[name]
planes = synth.Video(cfg.video).render(0, n)
dev = "--device" in sys.argv
dev_in = dev or "--device-in" in sys.argv    # input frames already in HBM
dev_out = dev or "--device-out" in sys.argv  # output frames stay in HBM
packed = "--packed" in sys.argv  # every frame one contiguous planar buffer (Y | Cb | Cr), in and out
if packed and len(planes) == 3:
    sizes = [int(np.prod(p.shape[1:])) for p in planes]
    offs = np.concatenate([[0], np.cumsum(sizes)])
    def frames_buf(on_dev, fill):
        t = torch.empty((n, int(offs[-1])), dtype=torch.uint8, device="cuda") if on_dev else \
            torch.empty((n, int(offs[-1])), dtype=torch.uint8).pin_memory()
        views = [t[:, int(offs[i]):int(offs[i + 1])] for i in range(3)]
        if fill:
            for v, p in zip(views, planes):
                v.copy_(torch.from_numpy(p).reshape(n, -1))
        return views
    pin = frames_buf(dev_in, True)
    outp = frames_buf(dev_out, False)
else:
    pin = [torch.from_numpy(p).cuda() if dev_in else torch.from_numpy(p).pin_memory() for p in planes]
    outp = [torch.empty(p.shape, dtype=torch.uint8, device="cuda") if dev_out
            else torch.empty(p.shape, dtype=torch.uint8).pin_memory() for p in pin]
h, w = planes[0].shape[1:]
col = len(planes) == 3
cw, ch = (planes[1].shape[2], planes[1].shape[1]) if col else (0, 0)
lib = load()
ctx = context(0)
c = cfg.stab.c()
hs = C.c_void_p()
assert lib.stabgpu_stream_create(ctx.handle, C.byref(c), w, h, cw, ch, C.byref(hs)) == 0
graphs = "--nographs" not in sys.argv
assert lib.stabgpu_stream_set_graphs(hs, int(graphs)) == 0
rec = np.zeros(1, pipeline.RECORD_DT)
vp = lambda t, k: C.c_void_p(t[k].data_ptr())
asyn = "--async" in sys.argv
depth = int(sys.argv[sys.argv.index("--depth") + 1]) if "--depth" in sys.argv else 2
wait_every = int(sys.argv[sys.argv.index("--wait-every") + 1]) if "--wait-every" in sys.argv else 1
owed = []  # --async: frames released by each push, not yet popped
def pop_all(k):
    pop = lib.stabgpu_stream_pop_async if asyn else lib.stabgpu_stream_pop
    for _ in range(k):
        idx = C.c_int64()
        j = 0
        # pop into the slot of the frame index (learned after the call: use a scratch slot first)
        assert pop(hs, C.byref(idx), vp(outp[0], pop_all.n % n),
                                      vp(outp[1], pop_all.n % n) if col else None,
                                      vp(outp[2], pop_all.n % n) if col else None,
                                      C.c_void_p(rec.ctypes.data)) == 0
        pop_all.n += 1
pop_all.n = 0
lat = []
nr = C.c_int()
# --push-async: stabgpu_stream_push_async (every frame has its own pinned array here,
# so nothing is overwritten; wait_inputs once at the end)
pasync = "--push-async" in sys.argv
push = lib.stabgpu_stream_push_async if pasync else lib.stabgpu_stream_push
lag = "--lag" in sys.argv  # pop a push late: frame k+1 uploads while frame k computes and k-r downloads
t0 = time.perf_counter()
pending = 0
for k in range(n):
    t1 = time.perf_counter()
    if asyn and len(owed) >= depth:
        pop_all(owed.pop(0))  # queue the downloads of the frames push k - depth released
    assert push(hs, vp(pin[0], k), vp(pin[1], k) if col else None,
                vp(pin[2], k) if col else None, C.byref(nr)) == 0
    if asyn:
        if (k + 1) % wait_every == 0:
            assert lib.stabgpu_stream_wait_pops(hs) == 0
        owed.append(nr.value - sum(owed))
    elif lag:
        pop_all(pending)  # frames released by earlier pushes
        pending = nr.value - pending
    else:
        pop_all(nr.value)
    lat.append(time.perf_counter() - t1)
if lag and not asyn:
    pop_all(pending)
assert lib.stabgpu_stream_wait_inputs(hs) == 0
assert lib.stabgpu_stream_finish(hs, C.byref(nr)) == 0
pop_all(nr.value)
if asyn:
    assert lib.stabgpu_stream_wait_pops(hs) == 0
dt = time.perf_counter() - t0
lib.stabgpu_stream_destroy(hs)
torch.cuda.synchronize()
digest = int(sum(int(o.to(torch.int64).sum().item()) for o in outp))
lat = np.array(lat) * 1e3
print(f"{name} {'device' if dev else 'pinned' if not (dev_in or dev_out) else ('device-in' if dev_in else 'device-out')} graphs={int(graphs)} lag={int(lag)} async={int(asyn) * depth} push_async={int(pasync)} wait_every={wait_every} packed={int(packed)}: {n} frames in {dt:.3f} s = {n / dt:.1f} frames/s; push+pop ms p50 {np.median(lat):.3f} "
      f"p99 {np.percentile(lat, 99):.3f}; {pop_all.n} frames out, output sum {digest}")
