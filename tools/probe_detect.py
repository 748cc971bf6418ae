"""Bucket-size profile of K4's candidate lists and the batched detect time
for a BASELINE config's detection frames.   python tools/probe_detect.py c1"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1701_03572_b200 import stab  # noqa: E402
from paper_1701_03572_b200.synth import CONFIGS, Video  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
cfg = CONFIGS[name]
n = min(cfg.video.frames, 301)
y = Video(cfg.video, threads=os.cpu_count()).render(0, n)[0]
det = np.ascontiguousarray(y[0:n - 1:cfg.stab.flow.redetect_interval])
r = stab.min_eig_response(det[0], 3)
roi = stab.detection_roi(det[0], cfg.stab.detect.roi_margin)
rr = r[roi.y0:roi.y1, roi.x0:roi.x1].ravel()
thr = cfg.stab.detect.quality_level * rr.max()
cand = rr[(rr >= thr) & (rr > 0)]
f32 = cand.astype(np.float32).view(np.uint32)
maxf = np.float32(rr.max()).view(np.uint32)
b = np.minimum((maxf - f32) >> 13, 8191)
cnt = np.bincount(b, minlength=8192)
print(f"{name}: {len(cand)} candidates, unique scores {len(np.unique(cand))}; buckets >32: {(cnt > 32).sum()}, "
      f">128: {(cnt > 128).sum()}, >4096: {(cnt > 4096).sum()}, max {cnt.max()}")
for rep in range(3):
    t0 = time.perf_counter()
    stab.detect_corners_batch(det, cfg.stab.detect)
    print(f"detect batch of {len(det)} frames: {1000 * (time.perf_counter() - t0):.2f} ms (incl. upload)")
