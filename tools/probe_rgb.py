"""RGB in / RGB out Stage I at C3 (1920x1080) through
stabgpu_stabilize_sequence_rgb with pinned host buffers (zero-copy fused
upload, fused RGB compose store), next to the plane entry point on the same
frames (pinned).  Prints frames/s of both, end to end."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1701_03572_b200 import evaluate, pipeline, synth
from paper_1701_03572_b200._lib import check, context, load

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
cfg = synth.CONFIGS["c3"]
y, cb, cr = synth.Video(cfg.video).render(0, n)
rgb = evaluate.ycbcr_to_rgb(y, cb, cr).cpu()
h, w = y.shape[1:]
lib, ctx, c = load(), context(0), cfg.stab.c()
src = rgb.pin_memory()
out = torch.empty_like(src).pin_memory()
rec = np.zeros(n, pipeline.RECORD_DT)
planes = [torch.from_numpy(p).pin_memory() for p in (y, cb, cr)]
outs = [torch.empty_like(p).pin_memory() for p in planes]
vp = lambda t: C.c_void_p(t.data_ptr())


def rgb_call():
    check(lib.stabgpu_stabilize_sequence_rgb(ctx.handle, vp(src), n, w, h, C.byref(c), vp(out),
                                             C.c_void_p(rec.ctypes.data)))


def plane_call():
    check(lib.stabgpu_stabilize_sequence(ctx.handle, vp(planes[0]), vp(planes[1]), vp(planes[2]), n, w, h, w, h,
                                         C.byref(c), vp(outs[0]), vp(outs[1]), vp(outs[2]),
                                         C.c_void_p(rec.ctypes.data)))


for name, fn in (("rgb", rgb_call), ("planes", plane_call)):
    fn()
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    print(f"{name}: {n} frames, best {min(ts) * 1e3:.1f} ms = {n / min(ts):.0f} frames/s e2e")
