"""Stage I TrackSets (read back from the context's scratch) vs a per-stage
replay on the GPU stage API, over repeated runs.

    python tools/diag_trackset.py c1 [frames] [reps]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1701_03572_b200 import _lib, pipeline, stab  # noqa: E402
from paper_1701_03572_b200.synth import CONFIGS, Video  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 60
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
cfg = CONFIGS[name]
sc = cfg.stab
fc = sc.flow
R = fc.redetect_interval
maxc = sc.detect.max_corners
y = Video(cfg.video, threads=os.cpu_count()).render(0, n)[0]
# per-stage replay
gp = [stab.build_pyramid(y[i], fc.max_levels) for i in range(n)]
ts_ref = {}
pts = None
for f in range(1, n):
    if (f - 1) % R == 0:
        pts, _ = stab.detect_corners(y[f - 1], sc.detect)
    pg, okg = stab.track_lk(gp[f - 1], gp[f], pts, fc)
    ts = stab.weed_tracks(gp[f - 1], gp[f], pts[okg], pg[okg], fc)
    ts_ref[f] = ts
    pts = ts.cur_points
ctx = _lib.context(0)
recs = []
for rep in range(reps):
    _, _, _, rec = pipeline.stabilize_sequence(y, sc)
    recs.append(rec)
    tn = ctx.read_scratch("trk_n", np.int32, n - 1)
    tp = ctx.read_scratch("trk_prev", np.float64, (n - 1) * maxc * 2).reshape(n - 1, maxc, 2)
    tc = ctx.read_scratch("trk_cur", np.float64, (n - 1) * maxc * 2).reshape(n - 1, maxc, 2)
    bad = []
    worst = 0.0
    for f in range(1, n):
        k = tn[f - 1]
        r = ts_ref[f]
        if k != r.size():
            bad.append((f, int(k), r.size()))
            continue
        d = max(np.abs(tp[f - 1, :k] - r.prev_points).max(), np.abs(tc[f - 1, :k] - r.cur_points).max()) if k else 0
        worst = max(worst, d)
        if d > 1e-9:
            bad.append((f, "pos", float(d)))
    print(f"rep {rep}: trackset mismatches {len(bad)} {bad[:10]} worst {worst:.3g}", flush=True)
for rep in range(1, reps):
    same = all(np.array_equal(recs[0][k], recs[rep][k]) for k in ("delta", "n_tracks", "n_inliers"))
    print(f"rep {rep} records identical to rep 0: {same}")
# Stage I pyramid levels (scratch "pyr1", "pyr2", ...) vs the per-frame pyramids
for l in range(1, fc.max_levels):
    ref_l = [stab.build_pyramid(y[i], fc.max_levels).levels[l] for i in range(n)]
    hh, ww = ref_l[0].shape
    got = ctx.read_scratch(f"pyr{l}", np.uint8, n * hh * ww).reshape(n, hh, ww)
    badf = [i for i in range(n) if not np.array_equal(got[i], ref_l[i])]
    print(f"level {l}: {len(badf)} of {n} frames differ {badf[:10]}")
    for i in badf[:2]:
        rows = np.nonzero((got[i] != ref_l[i]).any(1))[0]
        print(f"   frame {i}: rows differ {rows[:20].tolist()} ... ({len(rows)} rows)")
