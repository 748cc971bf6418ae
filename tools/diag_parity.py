"""Diagnose a config-scale parity difference (GPU Stage I vs the reference):
lists the frames whose records differ, then replays the first differing
segment stage by stage (detect, track_lk, weed_tracks) on both sides.

    python tools/diag_parity.py c1 [frames]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1701_03572_b200 import pipeline, stab  # noqa: E402
from paper_1701_03572_b200.synth import CONFIGS, Video  # noqa: E402
from tests import _oracle  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
cfg = CONFIGS[name]
n = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.video.frames
planes = Video(cfg.video, threads=os.cpu_count()).render(0, n)
y = planes[0]
ref = _oracle.reference()
gy, _, _, g = pipeline.stabilize_sequence(y, cfg.stab)
oy, _, _, o = ref.stabilize_sequence(y, cfg.stab, threads=os.cpu_count())
bad_tr = np.nonzero(g["n_tracks"] != o["n_tracks"])[0]
bad_in = np.nonzero(g["n_inliers"] != o["n_inliers"])[0]
err = np.max([np.abs(g["delta"][k] - o["delta"][k]) for k in ("dx", "dy", "da", "dls")], axis=0)
bad_d = np.nonzero(err > 1e-6)[0]
print("n_tracks differ:", bad_tr.tolist(), [(int(g["n_tracks"][f]), int(o["n_tracks"][f])) for f in bad_tr])
print("n_inliers differ:", bad_in.tolist(), [(int(g["n_inliers"][f]), int(o["n_inliers"][f])) for f in bad_in])
print("delta err > 1e-6:", bad_d.tolist()[:20], err[bad_d].tolist()[:20])
for f in bad_d[:4]:
    print(f"frame {f}: gpu", {k: float(g['delta'][k][f]) for k in ('dx', 'dy', 'da', 'dls')},
          "ref", {k: float(o['delta'][k][f]) for k in ('dx', 'dy', 'da', 'dls')})
if len(bad_tr) == 0:
    sys.exit(0)
R = cfg.stab.flow.redetect_interval
fc = cfg.stab.flow
f_bad = int(bad_tr[0])
b = ((f_bad - 1) // R) * R
print(f"replaying segment from frame {b} to {f_bad}")
gxy, gsc = stab.detect_corners(y[b], cfg.stab.detect)
oxy, osc = ref.detect_corners(y[b], cfg.stab.detect)
print("corners equal:", np.array_equal(gxy, oxy) and np.array_equal(gsc, osc), len(gxy), len(oxy))
gp = [stab.build_pyramid(y[i], fc.max_levels) for i in range(b, f_bad + 1)]
op = [ref.build_pyramid(y[i], fc.max_levels)[0] for i in range(b, f_bad + 1)]
gpts = opts = oxy
for t in range(1, f_bad - b + 1):
    pg, okg = stab.track_lk(gp[t - 1], gp[t], gpts, fc)
    po, oko = ref.track_lk(op[t - 1], op[t], opts, fc)
    print(f"step {t} (frame {b + t}): fwd ok flips {int((okg != oko).sum())}, max pos err "
          f"{np.abs(pg[okg & oko] - po[okg & oko]).max() if (okg & oko).any() else 0:.3g}")
    for i in np.nonzero(okg != oko)[0]:
        print(f"   point {i} at {gpts[i]} gpu ok={okg[i]} {pg[i]} ref ok={oko[i]} {po[i]}")
    # backward
    bg, bokg = stab.track_lk(gp[t], gp[t - 1], pg[okg], fc)
    bo, boko = ref.track_lk(op[t], op[t - 1], po[oko], fc)
    if okg.sum() == oko.sum():
        e_g = ((bg - gpts[okg]) ** 2).sum(1)
        e_o = ((bo - opts[oko]) ** 2).sum(1)
        print(f"   bwd ok flips {int((bokg != boko).sum())}, fb err2 max diff "
              f"{np.abs(e_g - e_o)[bokg & boko].max() if (bokg & boko).any() else 0:.3g}")
        for i in np.nonzero((bokg != boko) | ((e_g <= 0.25) != (e_o <= 0.25)))[0]:
            print(f"   bwd point {i}: gpu ok={bokg[i]} e2={e_g[i]!r} {bg[i]} ref ok={boko[i]} e2={e_o[i]!r} {bo[i]}")
    ts = stab.weed_tracks(gp[t - 1], gp[t], gpts[okg], pg[okg], fc)
    kp, kc = ref.weed_tracks(op[t - 1], op[t], opts[oko], po[oko], fc)
    print(f"   weeded gpu {ts.size()} ref {len(kp)}; stage-I record n_tracks gpu {g['n_tracks'][b + t]} "
          f"ref {o['n_tracks'][b + t]}")
    gpts, opts = ts.cur_points, kc
