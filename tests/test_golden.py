"""Pins the C oracle to fixtures produced by the unmodified reference
(tests/golden/make_golden.py).  Runs anywhere (no reference tree needed):
inputs come from the committed seeded generator, checked by digest."""
import hashlib
import os

import numpy as np
import pytest

from paper_1701_03572_b200 import _abi
from paper_1701_03572_b200.stab import DetectConfig, FlowConfig, RansacConfig

from . import _data, _oracle

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_vectors.npz")


@pytest.fixture(scope="module")
def G():
    return dict(np.load(GOLD))


def same(G, key, arr):
    arr = np.ascontiguousarray(arr)
    if key + "__sha256" in G:
        assert tuple(G[key + "__shape"]) == arr.shape, key
        return hashlib.sha256(arr.tobytes()).digest() == G[key + "__sha256"].tobytes()
    ref = G[key]
    return ref.shape == arr.shape and ref.tobytes() == arr.tobytes()


@pytest.fixture(scope="module")
def vid():
    return _data.video(160, 120, frames=12, objects=1, color=True, seed=3)


def test_inputs_match(G, vid):
    y, cb, cr = vid
    assert same(G, "frame", y[0]) and same(G, "frame1", y[1])
    assert same(G, "seq_in_y", y) and same(G, "seq_in_cb", cb) and same(G, "seq_in_cr", cr)


def test_image_and_features(G, vid):
    o = _oracle.oracle()
    f = vid[0][0]
    _, lv = o.build_pyramid(f, 4)
    assert all(same(G, f"pyr{i}", l) for i, l in enumerate(lv))
    gx, gy = o.gradients(f)
    assert same(G, "gx", gx) and same(G, "gy", gy)
    assert same(G, "resp3", o.min_eig_response(f, 3))
    xy, sc = o.detect_corners(f, DetectConfig(max_corners=80, min_distance=6.0))
    assert same(G, "corners_xy", xy) and same(G, "corners_score", sc)


def test_flow_and_motion(G, vid):
    o = _oracle.oracle()
    y = vid[0]
    fc = FlowConfig(window_radius=10, max_levels=3)
    p0, _ = o.build_pyramid(y[0], 3)
    p1, _ = o.build_pyramid(y[1], 3)
    pts = G["corners_xy"]
    xy, ok = o.track_lk(p0, p1, pts, fc)
    assert same(G, "lk_xy", xy) and same(G, "lk_ok", ok)
    kp, kc = o.weed_tracks(p0, p1, pts[ok], xy[ok], fc)
    assert same(G, "weed_prev", kp) and same(G, "weed_cur", kc)
    for kind, name in ((_abi.RIGID, "rigid"), (_abi.SIMILARITY, "similarity")):
        _, t = o.estimate(kp, kc, kind)
        assert same(G, f"fit_{name}", np.array([t.tx, t.ty, t.theta, t.s]))
        assert same(G, f"rms_{name}", np.array([o.rms_residual(kp, kc, t)]))
        _, t2, mask, _ = o.ransac(kp, kc, kind, RansacConfig(200, 0.3, 42), 8, 5)
        assert same(G, f"ransac_{name}", np.array([t2.tx, t2.ty, t2.theta, t2.s]))
        assert same(G, f"ransac_mask_{name}", mask)


def test_trajectory_and_compose(G, vid):
    o = _oracle.oracle()
    assert same(G, "traj_corr_r7", o.trajectory_corrections(G["traj_deltas"], 7))
    y, cb, cr = vid
    tt = G["compose_t"]
    t = _abi.Transform(tt[0], tt[1], tt[2], tt[3], _abi.SIMILARITY)
    assert same(G, "warp", o.warp_similarity(y[0], t))
    assert same(G, "crop", o.crop_resize(y[0], 0.04))
    oy, ob, orr = o.compose(y[0], cb[0], cr[0], t, 0.04)
    assert same(G, "compose_y", oy) and same(G, "compose_cb", ob) and same(G, "compose_cr", orr)


@pytest.mark.parametrize("ransac", [0, 100])
def test_sequence(G, vid, ransac):
    o = _oracle.oracle()
    y, cb, cr = vid
    cfg = _data.small_cfg(_data.MODES["hybrid"], ransac=ransac, corners=60, min_dist=6.0)
    sy, sb, sr, rec = o.stabilize_sequence(y, cfg, cb, cr)
    assert same(G, f"seq{ransac}_y", sy) and same(G, f"seq{ransac}_cb", sb) and same(G, f"seq{ransac}_cr", sr)
    ref = G[f"seq{ransac}_rec"].view(rec.dtype)
    tracked = ref["frame_kind"] == _abi.FRAME_TRACKED
    for k in ("delta", "correction", "frame_kind", "n_inliers", "decision"):
        assert ref[k].tobytes() == rec[k].tobytes(), k
    assert np.array_equal(ref["n_tracks"][tracked], rec["n_tracks"][tracked])
