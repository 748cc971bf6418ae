"""Stage II throughput/latency at a benchmark config: frames pushed one at a time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1701_03572_b200 import pipeline, synth
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 150
cfg = synth.CONFIGS[name]
planes = synth.Video(cfg.video).render(0, n)
y = planes[0]
cb, cr = (planes[1], planes[2]) if len(planes) == 3 else (None, None)
h, w = y.shape[1:]
s = pipeline.StreamStabilizer(cfg.stab, w, h, 0 if cb is None else cb.shape[2], 0 if cb is None else cb.shape[1])
lat = []
t0 = time.perf_counter()
out = 0
for k in range(n):
    t1 = time.perf_counter()
    out += len(s.push(y[k], None if cb is None else cb[k], None if cr is None else cr[k]))
    lat.append(time.perf_counter() - t1)
out += len(s.finish())
dt = time.perf_counter() - t0
s.close()
lat = np.array(lat) * 1e3
print(f"{name}: {n} frames streamed in {dt:.3f} s = {n / dt:.1f} frames/s; push+pop ms p50 {np.median(lat):.2f} p99 {np.percentile(lat, 99):.2f}; {out} frames out")
