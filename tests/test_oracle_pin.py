"""Pins the C oracle (oracle/stab_oracle.c) to the reference itself
(oracle/_ref/libstabref.so: the unmodified reference sources).  Everything is
compared bit for bit: both are the same arithmetic in the same order."""
import numpy as np
import pytest

from paper_1701_03572_b200 import _abi
from paper_1701_03572_b200.stab import DetectConfig, FlowConfig, RansacConfig

from . import _data, _oracle

pytestmark = pytest.mark.skipif(not _oracle.have_reference(),
                                reason="oracle/_ref not built (reference tree absent)")


@pytest.fixture(scope="module")
def impls():
    return _oracle.oracle(), _oracle.reference()


FRAMES = [(_data.noise_frame(97, 61, 1), "noise97x61"), (_data.noise_frame(160, 120, 2), "noise160"),
          (np.full((40, 50), 77, np.uint8), "flat"), (_data.video(frames=2)[0][1], "video")]


@pytest.mark.parametrize("f,name", FRAMES)
@pytest.mark.parametrize("levels", [1, 3, 6])
def test_pyramid(impls, f, name, levels):
    o, r = impls
    po, lo = o.build_pyramid(f, levels)
    pr, lr = r.build_pyramid(f, levels)
    assert po.levels == pr.levels
    for a, b in zip(lo, lr):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("f,name", FRAMES)
def test_gradients_response(impls, f, name):
    o, r = impls
    for a, b in zip(o.gradients(f), r.gradients(f)):
        assert np.array_equal(a, b)
    for block in (3, 5):
        assert np.array_equal(o.min_eig_response(f, block).view(np.uint64),
                              r.min_eig_response(f, block).view(np.uint64))


@pytest.mark.parametrize("f,name", FRAMES)
@pytest.mark.parametrize("corners,dist", [(8, 1.0), (40, 5.0), (200, 12.5)])
def test_detect(impls, f, name, corners, dist):
    o, r = impls
    cfg = DetectConfig(max_corners=corners, min_distance=dist)
    xo, so = o.detect_corners(f, cfg)
    xr, sr = r.detect_corners(f, cfg)
    assert np.array_equal(xo, xr) and np.array_equal(so.view(np.uint64), sr.view(np.uint64))


def test_detect_errors(impls):
    o, r = impls
    f = _data.noise_frame(40, 40, 3)  # ROI 32x32 ok at margin 0.1 -> 32x32
    for cfg in (DetectConfig(max_corners=4), DetectConfig(quality_level=0.0),
                DetectConfig(min_distance=0.5), DetectConfig(block_size=4),
                DetectConfig(roi_margin=0.45)):
        xy = np.empty((max(cfg.max_corners, 1), 2))
        sc = np.empty(max(cfg.max_corners, 1))
        import ctypes as C
        n = C.c_int()
        c = cfg.c()
        a = o.detect_corners_raw(_oracle._vp(f), 40, 40, C.byref(c), _oracle._vp(xy), _oracle._vp(sc), C.byref(n))
        b = r.detect_corners_raw(_oracle._vp(f), 40, 40, C.byref(c), _oracle._vp(xy), _oracle._vp(sc), C.byref(n))
        assert a == b == _abi.INVALID_CONFIG


@pytest.mark.parametrize("radius,levels", [(10, 3), (15, 4), (3, 1)])
def test_track_and_weed(impls, radius, levels):
    o, r = impls
    vid = _data.video(frames=3, jit_t=4.0)[0]
    cfg = FlowConfig(window_radius=radius, max_levels=levels)
    pyr = [(o.build_pyramid(vid[i], levels)[0], r.build_pyramid(vid[i], levels)[0]) for i in range(2)]
    pts, _ = o.detect_corners(vid[0], DetectConfig(max_corners=80, min_distance=6.0))
    rng = np.random.default_rng(5)
    pts = np.concatenate([pts, rng.uniform(-3, 200, size=(20, 2))])  # plus off-frame / edge points
    fo, oko = o.track_lk(pyr[0][0], pyr[1][0], pts, cfg)
    fr, okr = r.track_lk(pyr[0][1], pyr[1][1], pts, cfg)
    assert np.array_equal(oko, okr)
    assert np.array_equal(fo, fr)
    kpo, kco = o.weed_tracks(pyr[0][0], pyr[1][0], pts[oko], fo[oko], cfg)
    kpr, kcr = r.weed_tracks(pyr[0][1], pyr[1][1], pts[okr], fr[okr], cfg)
    assert np.array_equal(kpo, kpr) and np.array_equal(kco, kcr)


def _pairs(n, seed, outliers=0.0):
    rng = np.random.default_rng(seed)
    p = rng.uniform(0, 300, size=(n, 2))
    th, s, t = 0.03, 1.02, np.array([4.0, -2.5])
    R = s * np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])
    q = p @ R.T + t + rng.normal(0, 0.3, size=(n, 2))
    k = int(outliers * n)
    q[:k] += rng.uniform(-40, 40, size=(k, 2))
    return np.ascontiguousarray(p), np.ascontiguousarray(q)


@pytest.mark.parametrize("kind", [_abi.RIGID, _abi.SIMILARITY])
@pytest.mark.parametrize("n", [2, 3, 50, 400])
def test_estimate_rms(impls, kind, n):
    o, r = impls
    p, q = _pairs(n, n)
    rco, to = o.estimate(p, q, kind)
    rcr, tr = r.estimate(p, q, kind)
    assert rco == rcr == 0
    assert (to.tx, to.ty, to.theta, to.s, to.kind) == (tr.tx, tr.ty, tr.theta, tr.s, tr.kind)
    assert o.rms_residual(p, q, to) == r.rms_residual(p, q, tr)


def test_estimate_degenerate(impls):
    o, r = impls
    p = np.zeros((5, 2))
    q = np.ones((5, 2))
    assert o.estimate(p, q, 1)[0] == r.estimate(p, q, 1)[0] == _abi.DEGENERATE_INPUT
    assert o.estimate(p[:1], q[:1], 0)[0] == r.estimate(p[:1], q[:1], 0)[0] == _abi.DEGENERATE_INPUT


@pytest.mark.parametrize("kind", [_abi.RIGID, _abi.SIMILARITY])
@pytest.mark.parametrize("iters,outl", [(0, 0.3), (50, 0.0), (500, 0.3), (500, 0.7)])
def test_ransac_restatements_agree(impls, kind, iters, outl):
    o, r = impls
    p, q = _pairs(300, 11, outl)
    cfg = RansacConfig(iterations=iters, threshold=3.0, seed=1234)
    a = o.ransac(p, q, kind, cfg, 8, 17)
    b = r.ransac(p, q, kind, cfg, 8, 17)
    assert a[0] == b[0] == 0
    assert np.array_equal(a[2], b[2]) and a[3] == b[3]
    ta, tb = a[1], b[1]
    assert (ta.tx, ta.ty, ta.theta, ta.s) == (tb.tx, tb.ty, tb.theta, tb.s)
    if iters == 0:  # off == the reference estimator on all pairs
        _, t0 = r.estimate(p, q, kind)
        assert (t0.tx, t0.ty, t0.theta, t0.s) == (ta.tx, ta.ty, ta.theta, ta.s)


def test_trajectory(impls):
    o, r = impls
    rng = np.random.default_rng(3)
    d = rng.normal(0, 1, size=(57, 4)) * [2, 2, 0.01, 0.005]
    for radius in (1, 5, 30, 100):
        assert np.array_equal(o.trajectory_corrections(d, radius), r.trajectory_corrections(d, radius))


@pytest.mark.parametrize("t", [(0, 0, 0, 1), (3.0, -2.0, 0.0, 1.0), (2.3, 1.7, 0.02, 1.0),
                               (-5.5, 4.25, -0.05, 1.03), (0.5, 0.5, 0.3, 0.9)])
def test_warp_crop_compose(impls, t):
    o, r = impls
    y = _data.noise_frame(130, 90, 4)
    cb = _data.noise_frame(130, 90, 5)
    cr = _data.noise_frame(65, 45, 6)
    tt = _abi.Transform(t[0], t[1], t[2], t[3], _abi.SIMILARITY)
    assert np.array_equal(o.warp_similarity(y, tt), r.warp_similarity(y, tt))
    for crop in (0.0, 0.04, 0.2):
        assert np.array_equal(o.crop_resize(y, crop), r.crop_resize(y, crop))
        a = o.compose(y, cb, cb.copy(), tt, crop)
        b = r.compose(y, cb, cb.copy(), tt, crop)
        assert all(np.array_equal(u, v) for u, v in zip(a, b))
    cb2 = _data.noise_frame(65, 45, 7)  # 4:2:0-style chroma geometry
    a = o.compose(y, cb2, cr, tt, 0.04)
    b = r.compose(y, cb2, cr, tt, 0.04)
    assert all(np.array_equal(u, v) for u, v in zip(a, b))


@pytest.mark.parametrize("mode", ["rigid", "similarity", "hybrid"])
@pytest.mark.parametrize("ransac", [0, 200])
def test_sequence(impls, mode, ransac):
    o, r = impls
    y = _data.video(frames=26, objects=2, jit_t=3.0)[0]
    cfg = _data.small_cfg(_data.MODES[mode], ransac=ransac)
    a = o.stabilize_sequence(y, cfg)
    b = r.stabilize_sequence(y, cfg, threads=1)
    c = r.stabilize_sequence(y, cfg, threads=3)  # segment-parallel reference driver
    assert np.array_equal(a[0], b[0]) and np.array_equal(b[0], c[0])
    for k in ("delta", "correction", "frame_kind", "n_inliers", "decision"):
        assert np.array_equal(a[3][k], b[3][k]), k
        assert np.array_equal(b[3][k], c[3][k]), k
    tracked = a[3]["frame_kind"] == _abi.FRAME_TRACKED
    assert np.array_equal(a[3]["n_tracks"][tracked], b[3]["n_tracks"][tracked])


def test_sequence_matches_run_offline(impls):
    """The glue's driver with RANSAC off == the reference's own run_offline."""
    import ctypes as C
    _, r = impls
    y, cb, cr = _data.video(frames=20, color=True)
    cfg = _data.small_cfg(_data.MODES["hybrid"])
    oy, ob, orr, rec = r.stabilize_sequence(y, cfg, cb, cr, threads=2)
    n, h, w = y.shape
    ry, rb, rr = np.empty_like(y), np.empty_like(cb), np.empty_like(cr)
    deltas = (_abi.Delta * n)()
    corr = (_abi.Transform * n)()
    c = cfg.c()
    r.check(r.run_offline_raw(_oracle._vp(y), _oracle._vp(cb), _oracle._vp(cr), n, w, h, w, h,
                              C.byref(c), _oracle._vp(ry), _oracle._vp(rb), _oracle._vp(rr),
                              deltas, corr, None))
    assert np.array_equal(oy, ry) and np.array_equal(ob, rb) and np.array_equal(orr, rr)
    assert all(corr[i].tx == rec["correction"]["tx"][i] for i in range(n))


def test_colour_conversions_exhaustive():
    """The C restatement of BT.601 (media_io.cpp:75-89, 568-570) against the
    reference's own functions, for every RGB and every YCbCr triple."""
    o1, o2, _ = _oracle.colour_and_psnr(_oracle.ORACLE, "orc_")
    r1, r2, _ = _oracle.colour_and_psnr(_oracle.REF, "ref_")
    v = np.arange(1 << 24, dtype=np.uint32)
    trip = np.stack([(v >> 16) & 255, (v >> 8) & 255, v & 255], axis=-1).astype(np.uint8).reshape(4096, 4096, 3)
    for a, b in zip(o1(trip), r1(trip)):
        assert np.array_equal(a, b)
    assert np.array_equal(o2(trip[..., 0], trip[..., 1], trip[..., 2]), r2(trip[..., 0], trip[..., 1], trip[..., 2]))


@pytest.mark.parametrize("crop", [0.0, 0.04, 0.3])
def test_psnr_pair_matches_reference(crop):
    _, _, opsnr = _oracle.colour_and_psnr(_oracle.ORACLE, "orc_")
    _, _, rpsnr = _oracle.colour_and_psnr(_oracle.REF, "ref_")
    a, b = _data.noise_frame(97, 61, 1), _data.noise_frame(97, 61, 2)
    assert opsnr(a, b, crop) == rpsnr(a, b, crop)
    assert opsnr(a, a, crop) == rpsnr(a, a, crop) == float("inf")
