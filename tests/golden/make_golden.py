"""Generates tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref,
compiled from /root/reference/proj/src by oracle/Makefile).

Run here (where the reference exists):  python tests/golden/make_golden.py
The fixtures pin the C oracle on machines without the reference tree; every
array is what the reference itself returned for the seeded input stored
beside it."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_1701_03572_b200 import _abi  # noqa: E402
from paper_1701_03572_b200.stab import DetectConfig, FlowConfig, RansacConfig  # noqa: E402
from tests import _data, _oracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    ref = _oracle.reference()
    vid = _data.video(160, 120, frames=12, objects=1, color=True, seed=3)
    y, cb, cr = vid
    g = {}
    # pyramid / gradients / response / corners on frame 0
    f = y[0]
    g["frame"] = f
    _, lv = ref.build_pyramid(f, 4)
    for i, l in enumerate(lv):
        g[f"pyr{i}"] = l
    gx, gy = ref.gradients(f)
    g["gx"], g["gy"] = gx, gy
    g["resp3"] = ref.min_eig_response(f, 3)
    dc = DetectConfig(max_corners=80, min_distance=6.0)
    g["corners_xy"], g["corners_score"] = ref.detect_corners(f, dc)
    # LK + weeding frame 0 -> 1
    fc = FlowConfig(window_radius=10, max_levels=3)
    p0, _ = ref.build_pyramid(y[0], 3)
    p1, _ = ref.build_pyramid(y[1], 3)
    g["frame1"] = y[1]
    pts = g["corners_xy"]
    g["lk_xy"], g["lk_ok"] = ref.track_lk(p0, p1, pts, fc)
    g["weed_prev"], g["weed_cur"] = ref.weed_tracks(p0, p1, pts[g["lk_ok"]], g["lk_xy"][g["lk_ok"]], fc)
    # fits
    p, q = g["weed_prev"], g["weed_cur"]
    for kind, name in ((_abi.RIGID, "rigid"), (_abi.SIMILARITY, "similarity")):
        _, t = ref.estimate(p, q, kind)
        g[f"fit_{name}"] = np.array([t.tx, t.ty, t.theta, t.s])
        g[f"rms_{name}"] = np.array([ref.rms_residual(p, q, t)])
        _, t2, mask, used = ref.ransac(p, q, kind, RansacConfig(200, 0.3, 42), 8, 5)
        g[f"ransac_{name}"] = np.array([t2.tx, t2.ty, t2.theta, t2.s])
        g[f"ransac_mask_{name}"] = mask
    # trajectory
    rng = np.random.default_rng(9)
    d = rng.normal(0, 1, size=(40, 4)) * [2, 2, 0.01, 0.005]
    g["traj_deltas"] = d
    g["traj_corr_r7"] = ref.trajectory_corrections(d, 7)
    # compose
    t = _abi.Transform(2.3, -1.7, 0.02, 1.01, _abi.SIMILARITY)
    g["compose_t"] = np.array([t.tx, t.ty, t.theta, t.s])
    g["warp"] = ref.warp_similarity(f, t)
    g["crop"] = ref.crop_resize(f, 0.04)
    oy, ob, orr = ref.compose(y[0], cb[0], cr[0], t, 0.04)
    g["cb0"], g["cr0"] = cb[0], cr[0]
    g["compose_y"], g["compose_cb"], g["compose_cr"] = oy, ob, orr
    # whole sequence (run_offline semantics) with and without RANSAC
    for ransac in (0, 100):
        cfg = _data.small_cfg(_data.MODES["hybrid"], ransac=ransac, corners=60, min_dist=6.0)
        sy, sb, sr, rec = ref.stabilize_sequence(y, cfg, cb, cr, threads=1)
        g[f"seq{ransac}_y"], g[f"seq{ransac}_cb"], g[f"seq{ransac}_cr"] = sy, sb, sr
        g[f"seq{ransac}_rec"] = rec.view(np.uint8)
    g["seq_in_y"], g["seq_in_cb"], g["seq_in_cr"] = y, cb, cr
    # inputs are regenerated from the committed seeded generator (hash-checked);
    # large images are stored as sha256 digests, small arrays verbatim
    import hashlib
    small = {}
    for k, v in g.items():
        v = np.ascontiguousarray(v)
        if v.nbytes > 4096 and k not in ("traj_deltas",):
            small[k + "__sha256"] = np.frombuffer(hashlib.sha256(v.tobytes()).digest(), np.uint8)
            small[k + "__shape"] = np.array(v.shape)
        else:
            small[k] = v
    g = small
    np.savez_compressed(os.path.join(OUT, "reference_vectors.npz"), **g)
    print("wrote", os.path.join(OUT, "reference_vectors.npz"),
          os.path.getsize(os.path.join(OUT, "reference_vectors.npz")), "bytes")


if __name__ == "__main__":
    main()
