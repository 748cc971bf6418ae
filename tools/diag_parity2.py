"""Stage I records vs a per-stage replay (GPU stage API and the reference)
for the first frames of a config: isolates tracking from the fit.

    python tools/diag_parity2.py c1 [frames] [first]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1701_03572_b200 import _abi, pipeline, stab  # noqa: E402
from paper_1701_03572_b200.synth import CONFIGS, Video  # noqa: E402
from tests import _oracle  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 11
first = int(sys.argv[3]) if len(sys.argv) > 3 else 0
cfg = CONFIGS[name]
y = Video(cfg.video, threads=os.cpu_count()).render(first, n)[0]
ref = _oracle.reference()
sc = cfg.stab
_, _, _, g = pipeline.stabilize_sequence(y, sc)
_, _, _, o = ref.stabilize_sequence(y, sc, threads=os.cpu_count())
kind = _abi.RIGID if sc.selector.mode == 1 else _abi.SIMILARITY
fc = sc.flow
R = fc.redetect_interval
gp = [stab.build_pyramid(y[i], fc.max_levels) for i in range(n)]
op = [ref.build_pyramid(y[i], fc.max_levels)[0] for i in range(n)]
gpts = opts = None
for f in range(1, n):
    if (f - 1) % R == 0:
        gpts, _ = stab.detect_corners(y[f - 1], sc.detect)
        opts, _ = ref.detect_corners(y[f - 1], sc.detect)
    pg, okg = stab.track_lk(gp[f - 1], gp[f], gpts, fc)
    po, oko = ref.track_lk(op[f - 1], op[f], opts, fc)
    ts = stab.weed_tracks(gp[f - 1], gp[f], gpts[okg], pg[okg], fc)
    kp, kc = ref.weed_tracks(op[f - 1], op[f], opts[oko], po[oko], fc)
    # fits on each side's own TrackSet, with the frame index the sequence uses
    rc, t_ref, m_ref, u_ref = ref.ransac(kp, kc, kind, sc.ransac, fc.min_tracks, f)
    t_gpu, _ = stab.ransac_estimate(ts, kind, sc.ransac, fc.min_tracks, frame_index=f)
    t_gpu = t_gpu.tx
    print(f"frame {f}: n_tracks stageI gpu {g['n_tracks'][f]} ref {o['n_tracks'][f]} | per-stage gpu {ts.size()} "
          f"ref {len(kp)} | inliers stageI {g['n_inliers'][f]} {o['n_inliers'][f]} per-stage ref {u_ref}")
    print(f"    stageI dx gpu {g['delta']['dx'][f]!r} ref {o['delta']['dx'][f]!r}; per-stage ref fit tx "
          f"{t_ref.tx!r} gpu fit {t_gpu}")
    print(f"    max |pos| diff per-stage {np.abs(ts.cur_points - kc).max() if ts.size() == len(kc) else 'n/a'}")
    gpts, opts = ts.cur_points, kc
