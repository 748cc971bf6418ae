"""Times K8 (compose) alone on device-resident 1080p Y/Cb/Cr frames."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1701_03572_b200 import pipeline
from paper_1701_03572_b200.pipeline import TRANSFORM_DT
n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
g = torch.Generator(device="cuda").manual_seed(1)
planes = [torch.randint(0, 256, (n, 1080, 1920), dtype=torch.uint8, device="cuda", generator=g) for _ in range(3)]
rng = np.random.default_rng(0)
corr = np.zeros(n, TRANSFORM_DT)
corr["tx"] = rng.normal(0, 8, n); corr["ty"] = rng.normal(0, 8, n)
corr["theta"] = rng.normal(0, 0.017, n); corr["s"] = 1 + rng.normal(0, 0.01, n); corr["kind"] = 1
outs = [torch.empty_like(p) for p in planes]
for _ in range(2):
    pipeline.compose_frames(planes[0], corr, 0.04, planes[1], planes[2], *outs)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    pipeline.compose_frames(planes[0], corr, 0.04, planes[1], planes[2], *outs)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
gb = 2 * 3 * 1920 * 1080 * n / 1e9
print(f"compose {n} frames: {ms:.3f} ms  {gb / ms * 1e3:.0f} GB/s  ({ms / n * 1000:.1f} us/frame)")
