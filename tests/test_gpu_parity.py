"""GPU (libstabgpu.so) vs the C oracle, stage by stage and end to end.

Bars: integer/byte/index work bit-exact (pyramid, corner sets and scores,
crop_resize, chroma, RANSAC inlier sets); floating-point LK / fits within
north_star's tolerances (positions <= 0.01 px, transform parameters <= 1e-3)
and, in practice, ~1e-9; warped luma within +-1 with the count of +-1 pixels
bounded (the GPU evaluates the reference's row-incremental coordinate walk
in closed form)."""
import numpy as np
import pytest

from paper_1701_03572_b200 import _abi, pipeline, stab
from paper_1701_03572_b200.stab import DetectConfig, FlowConfig, RansacConfig

from . import _data, _oracle

pytestmark = pytest.mark.gpu

POS_TOL = 1e-6  # px; north_star allows 0.01
PARAM_TOL = 1e-6  # north_star allows 1e-3


@pytest.fixture(scope="module")
def orc():
    return _oracle.oracle()


FRAMES = [(_data.noise_frame(97, 61, 1), "noise97x61"), (_data.noise_frame(160, 120, 2), "noise160"),
          (np.full((40, 50), 77, np.uint8), "flat"), (_data.video(frames=2)[0][1], "video")]
# extremes of the packed 16-bit pyramid lanes (all-255, 0/255 checkerboard),
# the benchmark frame size, and a width that is a multiple of 8 but not of 16
PYR_FRAMES = FRAMES + [
    (np.full((64, 128), 255, np.uint8), "sat255"),
    (((np.indices((96, 176)).sum(axis=0) % 2) * 255).astype(np.uint8), "checker"),
    (_data.noise_frame(1920, 1080, 3), "noise1080p"),
    (_data.noise_frame(200, 72, 4), "noise200x72"),
]


@pytest.mark.parametrize("f,name", PYR_FRAMES)
@pytest.mark.parametrize("levels", [1, 3, 6])
def test_pyramid_bitexact(orc, f, name, levels):
    g = stab.build_pyramid(f, levels)
    _, ref = orc.build_pyramid(f, levels)
    assert g.level_count() == len(ref)
    for a, b in zip(g.levels, ref):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("w,h,n", [(1920, 1080, 5), (352, 291, 37), (160, 37, 300), (3840, 64, 3)])
def test_pyramid_level_batches(orc, w, h, n):
    """K1 over a frame batch (the Stage I layout): the bulk-copy kernel's
    bands, row groups, odd heights and item counts beyond the grid."""
    import ctypes as C

    import torch

    from paper_1701_03572_b200 import _lib

    rng = np.random.default_rng(w * h + n)
    frames = rng.integers(0, 256, size=(n, h, w), dtype=np.uint8)
    frames[0] = 255
    src = torch.from_numpy(frames).cuda()
    ow, oh = w // 2, h // 2
    dst = torch.empty((n, oh, ow), dtype=torch.uint8, device="cuda")
    _lib.load().stabgpu_debug_pyramid_level(C.c_void_p(src.data_ptr()), C.c_size_t(w * h), w, h,
                                            C.c_void_p(dst.data_ptr()), C.c_size_t(ow * oh), n,
                                            C.c_void_p(torch.cuda.current_stream().cuda_stream))
    got = dst.cpu().numpy()
    for i in sorted({0, 1, n // 2, n - 1}):
        _, ref = orc.build_pyramid(frames[i], 2)
        assert np.array_equal(got[i], ref[1]), i


@pytest.mark.parametrize("w,h,n,levels", [
    (640, 480, 60, 3),     # C1: 128-thread carry kernel at level 1, bulk below
    (1280, 720, 40, 4),    # C2/C5: 256-thread carry kernel
    (1920, 1080, 40, 4),   # C3: 256-thread carry kernel, then 128-thread carry (960)
    (3840, 2160, 12, 5),   # C4: 512-thread carry kernel
    (1008, 600, 50, 4),    # carry band rounding (buffer / width not a whole number of rows)
    (976, 100, 300, 3),    # many short frames: CTA runs cross frame boundaries
])
def test_pyramid_batch_every_frame(orc, w, h, n, levels):
    """Batched K1 (the Stage I launch) equals the reference pyramid on every
    frame, at the BASELINE geometries and with enough frames that a CTA's run
    of (frame, band) items carries filtered rows from band to band.  (Round 1
    sized the 128-thread carry kernel's band one row too large for 640-wide
    frames; its first band overran the staging buffer.)"""
    rng = np.random.default_rng(w + h + n)
    base = _data.noise_frame(w, h, 11)
    frames = np.stack([np.roll(base, (3 * i, 5 * i), axis=(0, 1)) ^ rng.integers(0, 4, size=(h, w), dtype=np.uint8)
                       for i in range(n)])
    frames[0, :h // 3] = 255
    got = stab.build_pyramid_batch(frames, levels)
    for i in range(n):
        _, ref = orc.build_pyramid(frames[i], levels)
        assert len(got[i]) == len(ref)
        for lev, (a, b) in enumerate(zip(got[i], ref)):
            assert np.array_equal(a, b), (i, lev)


@pytest.mark.parametrize("f,name", FRAMES)
def test_gradients_response_bitexact(orc, f, name):
    gx, gy = stab.gradients(f)
    ox, oy = orc.gradients(f)
    assert np.array_equal(gx, ox) and np.array_equal(gy, oy)
    for block in (3, 5, 7):
        assert np.array_equal(stab.min_eig_response(f, block).view(np.uint64),
                              orc.min_eig_response(f, block).view(np.uint64))


@pytest.mark.parametrize("f,name", FRAMES)
@pytest.mark.parametrize("corners,dist,block", [(8, 1.0, 3), (40, 5.0, 3), (200, 12.5, 3),
                                                (60, 4.0, 5), (30, 7.0, 7)])
def test_detect_bitexact(orc, f, name, corners, dist, block):
    cfg = DetectConfig(max_corners=corners, min_distance=dist, block_size=block)
    xg, sg = stab.detect_corners(f, cfg)
    xo, so = orc.detect_corners(f, cfg)
    assert np.array_equal(xg, xo)
    assert np.array_equal(sg.view(np.uint64), so.view(np.uint64))


def test_detect_many_ties(orc):
    """Large plateaus of identical scores exercise the tie-heavy bucket path."""
    f = np.zeros((300, 400), np.uint8)
    f[::8, :] = 255
    f[:, ::8] = 255
    for corners, dist in ((5000, 1.0), (300, 3.0)):
        cfg = DetectConfig(max_corners=corners, min_distance=dist)
        xg, sg = stab.detect_corners(f, cfg)
        xo, so = orc.detect_corners(f, cfg)
        assert np.array_equal(xg, xo) and np.array_equal(sg, so)


def test_detect_cut_redo(orc):
    """A strong textured patch holds far more candidates than the greedy can
    accept under a large min_distance, so the fp32-histogram cut prefix runs
    out before max_corners and the full-list redo path must take over
    ((100, 20), (300, 12)); (60, 40) is dense enough (exclusion discs cover
    the ROI more than twice) that selection skips the cut altogether."""
    rng = np.random.default_rng(7)
    f = (rng.integers(118, 138, size=(320, 320))).astype(np.uint8)   # weak texture
    f[100:220, 100:220] = rng.integers(0, 256, size=(120, 120))      # strong patch
    for corners, dist in ((60, 40.0), (20, 25.0), (300, 12.0), (100, 20.0)):
        cfg = DetectConfig(max_corners=corners, min_distance=dist, roi_margin=0.0)
        xg, sg = stab.detect_corners(f, cfg)
        xo, so = orc.detect_corners(f, cfg)
        assert len(xo) > 0
        assert np.array_equal(xg, xo) and np.array_equal(sg.view(np.uint64), so.view(np.uint64))


def test_detect_chunk_growth_and_retry(orc):
    """K4's adaptive chunks: a few very strong clusters (their neighbours fill
    the top of the list and are nearly all excluded, so the chunk size grows to
    its maximum) followed by tens of thousands of weak, well separated
    candidates (a maximum-size chunk whose survivors overflow the chunk buffer
    and must be retried smaller).  With and without the candidate cut, one
    round (max_corners reached in the list's head) and two (re-bucketed rest)."""
    rng = np.random.default_rng(11)
    f = rng.integers(120, 136, size=(480, 640)).astype(np.uint8)     # weak texture everywhere
    for cy, cx in ((100, 120), (240, 330), (380, 520), (110, 500)):   # strong clusters
        f[cy - 12:cy + 12, cx - 12:cx + 12] = rng.integers(0, 256, size=(24, 24))
    for corners, dist, q in ((6000, 1.5, 0.0005), (3000, 2.0, 0.001), (400, 6.0, 0.001), (150, 45.0, 0.0005)):
        cfg = DetectConfig(max_corners=corners, min_distance=dist, quality_level=q, roi_margin=0.05)
        xg, sg = stab.detect_corners(f, cfg)
        xo, so = orc.detect_corners(f, cfg)
        assert len(xo) > 50
        assert np.array_equal(xg, xo) and np.array_equal(sg.view(np.uint64), so.view(np.uint64))


@pytest.mark.parametrize("w,h", [(1920, 1080), (640, 480)])
def test_detect_full_size(orc, w, h):
    y = _data.video(w, h, frames=1, tex=2048, blobs=1600)[0][0]
    for cfg in (DetectConfig(max_corners=1000, min_distance=15.0),
                DetectConfig(max_corners=200, min_distance=30.0)):
        xg, sg = stab.detect_corners(y, cfg)
        xo, so = orc.detect_corners(y, cfg)
        assert np.array_equal(xg, xo) and np.array_equal(sg, so)


def test_detect_errors():
    f = _data.noise_frame(64, 64, 3)
    for cfg in (DetectConfig(max_corners=4), DetectConfig(quality_level=1.0),
                DetectConfig(min_distance=0.5), DetectConfig(block_size=4),
                DetectConfig(roi_margin=0.45)):
        with pytest.raises(stab.InvalidConfigError):
            stab.detect_corners(f, cfg)
    with pytest.raises(stab.InvalidInputError):
        stab.detect_corners(np.zeros((10, 40), np.uint8), DetectConfig())
    with pytest.raises(stab.InvalidConfigError):  # ROI < 32x32
        stab.detect_corners(np.zeros((36, 36), np.uint8), DetectConfig())
    xy, sc = stab.detect_corners(np.full((64, 64), 9, np.uint8), DetectConfig())
    assert len(xy) == 0  # flat frame: empty, not an error


@pytest.mark.parametrize("radius,levels,shift", [(10, 3, 4.0), (15, 5, 8.0), (3, 1, 1.0), (10, 4, 20.0)])
def test_track_lk(orc, radius, levels, shift):
    vid = _data.video(320, 240, frames=2, jit_t=shift, tex=512, blobs=200)[0]
    cfg = FlowConfig(window_radius=radius, max_levels=levels)
    pts, _ = orc.detect_corners(vid[0], DetectConfig(max_corners=150, min_distance=6.0))
    rng = np.random.default_rng(5)
    pts = np.concatenate([pts, rng.uniform(-3, 330, size=(30, 2))])
    gp = [stab.build_pyramid(vid[i], levels) for i in range(2)]
    op = [orc.build_pyramid(vid[i], levels)[0] for i in range(2)]
    pg, okg = stab.track_lk(gp[0], gp[1], pts, cfg)
    po, oko = orc.track_lk(op[0], op[1], pts, cfg)
    assert np.array_equal(okg, oko)
    assert np.abs(pg - po).max() <= POS_TOL
    ts = stab.weed_tracks(gp[0], gp[1], pts[okg], pg[okg], cfg)
    kp, kc = orc.weed_tracks(op[0], op[1], pts[oko], po[oko], cfg)
    assert ts.size() == len(kp)
    assert np.array_equal(ts.prev_points, kp)


def test_track_identical_frames_exact_zero():
    """test_flow.cpp:24-40: identical frames -> exactly zero flow."""
    f = _data.video(200, 150, frames=1, tex=256)[0][0]
    p = stab.build_pyramid(f, 3)
    pts, _ = stab.detect_corners(f, DetectConfig(max_corners=40))
    out, ok = stab.track_lk(p, p, pts, FlowConfig(max_levels=3))
    assert ok.all() and np.array_equal(out, pts)


def test_track_integer_shift():
    """test_flow.cpp:42-62: a (5,3) shift is recovered within 0.2 px for >= 90%."""
    f = _data.video(240, 180, frames=1, tex=256)[0][0]
    g = _data.integer_shift(f, 5, 3)
    pts, _ = stab.detect_corners(f, DetectConfig(max_corners=60, min_distance=8))
    out, ok = stab.track_lk(stab.build_pyramid(f, 3), stab.build_pyramid(g, 3), pts, FlowConfig(max_levels=3))
    err = np.hypot(out[:, 0] - pts[:, 0] - 5, out[:, 1] - pts[:, 1] - 3)
    assert (ok & (err < 0.2)).mean() >= 0.9


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
@pytest.mark.parametrize("n", [2, 3, 50, 1000])
def test_estimate(orc, kind, n):
    p, q = _pairs(n, n)
    ts = stab.TrackSet(p, q)
    g = stab.estimate_rigid(ts) if kind == _abi.RIGID else stab.estimate_similarity(ts)
    _, o = orc.estimate(p, q, kind)
    assert abs(g.tx - o.tx) < PARAM_TOL and abs(g.ty - o.ty) < PARAM_TOL
    assert abs(g.theta - o.theta) < 1e-12 and abs(g.s - o.s) < 1e-12 and g.kind == o.kind
    assert abs(stab.rms_residual(ts, g) - orc.rms_residual(p, q, o)) < 1e-9


def test_estimate_degenerate():
    with pytest.raises(stab.DegenerateInputError):
        stab.estimate_similarity(stab.TrackSet(np.zeros((5, 2)), np.ones((5, 2))))
    with pytest.raises(stab.DegenerateInputError):
        stab.estimate_rigid(stab.TrackSet(np.zeros((1, 2)), np.ones((1, 2))))


@pytest.mark.parametrize("kind", [_abi.RIGID, _abi.SIMILARITY])
@pytest.mark.parametrize("iters,outl", [(0, 0.3), (50, 0.0), (500, 0.3), (1000, 0.7)])
def test_ransac_inliers_bitexact(orc, kind, iters, outl):
    p, q = _pairs(700, 11, outl)
    cfg = RansacConfig(iterations=iters, threshold=3.0, seed=1234)
    t, mask = stab.ransac_estimate(stab.TrackSet(p, q), kind, cfg, 8, 17)
    _, to, mo, _ = orc.ransac(p, q, kind, cfg, 8, 17)
    assert np.array_equal(mask, mo)
    assert abs(t.tx - to.tx) < PARAM_TOL and abs(t.theta - to.theta) < 1e-12


def test_trajectory(orc):
    rng = np.random.default_rng(3)
    d = rng.normal(0, 1, size=(257, 4)) * [2, 2, 0.01, 0.005]
    for radius in (1, 5, 30):
        g = stab.trajectory_corrections(d, radius)
        o = orc.trajectory_corrections(d, radius)
        assert np.array_equal(g[:, :3], o[:, :3])  # sequential sums: bit-exact
        assert np.abs(g[:, 3] - o[:, 3]).max() <= 2e-16  # exp(): device vs glibc ulp


def _offby(a, b):
    d = np.abs(a.astype(int) - b.astype(int))
    return int(d.max()), int((d > 0).sum())


TRANSFORMS = [(0, 0, 0, 1), (3.0, -2.0, 0.0, 1.0), (2.3, 1.7, 0.02, 1.0), (-5.5, 4.25, -0.05, 1.03),
              (0.5, 0.5, 0.3, 0.9), (40.0, -30.0, 0.6, 1.4), (-3.0, 2.0, -1.2, 0.6),
              (0.25, -0.75, 0.001, 1.0), (900.0, 0.0, 0.0, 1.0)]


@pytest.mark.parametrize("t", TRANSFORMS)
@pytest.mark.parametrize("w,h", [(330, 190), (331, 77), (1920, 1080)])
def test_warp_crop_compose_bitexact(orc, t, w, h):
    """K8 reproduces warp_similarity (incl. its sequential row walk), crop_resize and
    compose_plane bit for bit; large rotations/scales exercise the unstaged path."""
    y = _data.noise_frame(w, h, 4)
    cb = _data.noise_frame(w, h, 5)
    cr = _data.noise_frame((w + 1) // 2, (h + 1) // 2, 6)
    cr2 = _data.noise_frame((w + 1) // 2, (h + 1) // 2, 8)
    tt = _abi.Transform(t[0], t[1], t[2], t[3], _abi.SIMILARITY)
    T = stab.SimilarityTransform(*t, kind=_abi.SIMILARITY)
    assert np.array_equal(stab.warp_similarity(y, T), orc.warp_similarity(y, tt))
    for crop in (0.0, 0.04, 0.2):
        assert np.array_equal(stab.crop_resize(y, crop), orc.crop_resize(y, crop))
        gy, gb, gr = stab.compose_stabilized(y, T, crop, cb, cb[::-1].copy())
        oy, ob, orr = orc.compose(y, cb, cb[::-1].copy(), tt, crop)
        assert np.array_equal(gy, oy) and np.array_equal(gb, ob) and np.array_equal(gr, orr)
    gy, gb, gr = stab.compose_stabilized(y, T, 0.04, cr, cr2)  # 4:2:0 chroma geometry
    oy, ob, orr = orc.compose(y, cr, cr2, tt, 0.04)
    assert np.array_equal(gy, oy) and np.array_equal(gb, ob) and np.array_equal(gr, orr)


def test_identity_compose_equals_crop():
    """test_pipeline.cpp:83-105: identity correction -> crop_resize(input)."""
    y = _data.noise_frame(256, 144, 9)
    I = stab.SimilarityTransform()
    assert np.array_equal(stab.compose_stabilized(y, I, 0.04), stab.crop_resize(y, 0.04))
    assert np.array_equal(stab.warp_similarity(y, I), y)


def test_transform_errors():
    y = _data.noise_frame(64, 64, 1)
    with pytest.raises(stab.InvalidTransformError):
        stab.warp_similarity(y, stab.SimilarityTransform(s=0.0))
    with pytest.raises(stab.InvalidTransformError):
        stab.warp_similarity(y, stab.SimilarityTransform(s=1.1, kind=_abi.RIGID))
    with pytest.raises(stab.InvalidConfigError):
        stab.crop_resize(y, 0.3)


def _compare_records(g, o, tracked_tol=PARAM_TOL):
    assert np.array_equal(g["frame_kind"], o["frame_kind"])
    tr = o["frame_kind"] == _abi.FRAME_TRACKED
    assert np.array_equal(g["n_tracks"][tr], o["n_tracks"][tr])
    assert np.array_equal(g["n_inliers"], o["n_inliers"])
    assert np.array_equal(g["decision"], o["decision"])
    assert np.array_equal(g["delta"]["kind"], o["delta"]["kind"])
    assert np.array_equal(g["delta"]["skipped"], o["delta"]["skipped"])
    for k in ("dx", "dy", "da", "dls"):
        assert np.abs(g["delta"][k] - o["delta"][k]).max() <= tracked_tol, k
    for k in ("tx", "ty", "theta", "s"):
        assert np.abs(g["correction"][k] - o["correction"][k]).max() <= tracked_tol, k


@pytest.mark.parametrize("mode", ["rigid", "similarity", "hybrid"])
@pytest.mark.parametrize("ransac", [0, 300])
def test_sequence(orc, mode, ransac):
    y, cb, cr = _data.video(frames=41, objects=2, jit_t=3.0, color=True)
    cfg = _data.small_cfg(_data.MODES[mode], ransac=ransac)
    gy, gb, gr, gr_rec = pipeline.stabilize_sequence(y, cfg, cb, cr)
    oy, ob, orr, o_rec = orc.stabilize_sequence(y, cfg, cb, cr)
    _compare_records(gr_rec, o_rec)
    # corrections carry device atan2/exp/cos/sin ulps, so a pixel may sit on the
    # other side of a .5 tie: +-1, rarely
    mx, cnt = _offby(gy, oy)
    assert mx <= 1 and cnt <= 0.0005 * gy.size
    for a, b in ((gb, ob), (gr, orr)):
        mx, cnt = _offby(a, b)
        assert mx <= 1 and cnt <= 0.0005 * a.size


def test_sequence_many_detection_frames(orc):
    """More detection frames than SMs: K4 runs as two 512-thread CTAs per SM
    (3072-candidate chunks) instead of one 1024-thread CTA; same corners."""
    import torch

    n = 5 * (torch.cuda.get_device_properties(0).multi_processor_count + 12) + 1
    y = _data.video(frames=n, objects=1, jit_t=3.0)[0]
    cfg = _data.small_cfg(_data.MODES["similarity"], ransac=100)
    gy, _, _, grec = pipeline.stabilize_sequence(y, cfg)
    oy, _, _, orec = orc.stabilize_sequence(y, cfg)
    _compare_records(grec, orec)
    mx, cnt = _offby(gy, oy)
    assert mx <= 1 and cnt <= 0.0005 * gy.size


@pytest.mark.parametrize("n", [2, 3, 4])
def test_short_clip_large_corner_budget(orc, n):
    """Fewer frames than the re-detect interval with a 1000-corner budget: the
    chain's per-step planes are sized min(R, n - 1), and nothing is written
    past them (run this file under compute-sanitizer to see it)."""
    from paper_1701_03572_b200 import _lib

    y = _data.video(320, 240, frames=n, jit_t=2.0, tex=512, blobs=200)[0]
    cfg = _data.small_cfg(_data.MODES["similarity"], ransac=50, corners=1000, min_dist=3.0)
    _lib.reset_contexts()  # fresh context: no scratch left over from larger runs
    gy, _, _, grec = pipeline.stabilize_sequence(y, cfg)
    oy, _, _, orec = orc.stabilize_sequence(y, cfg)
    _compare_records(grec, orec)
    mx, cnt = _offby(gy, oy)
    assert mx <= 1 and cnt <= 0.0005 * gy.size


def test_sequence_device_equals_host_path():
    import torch
    y, cb, cr = _data.video(frames=37, objects=1, color=True)
    cfg = _data.small_cfg(_data.MODES["similarity"], ransac=100)
    hy, hb, hr, hrec = pipeline.stabilize_sequence(y, cfg, cb, cr)
    dev = [torch.from_numpy(a).cuda() for a in (y, cb, cr)]
    dy, db, dr, drec = pipeline.stabilize_sequence_device(dev[0], cfg, dev[1], dev[2])
    torch.cuda.synchronize()
    assert np.array_equal(dy.cpu().numpy(), hy) and np.array_equal(db.cpu().numpy(), hb)
    assert np.array_equal(dr.cpu().numpy(), hr)
    assert hrec.tobytes() == drec.tobytes()


def test_sharded_equals_single():
    """The per-rank split (motion chunks + gathered plan + own compose), run
    for every rank in one process, reproduces the one-GPU run bitwise."""
    import torch
    y = _data.video(frames=53, objects=1)[0]
    cfg = _data.small_cfg(_data.MODES["hybrid"], ransac=100)
    dy = torch.from_numpy(y).cuda()
    ref_y, _, _, ref_rec = pipeline.stabilize_sequence_device(dy, cfg)
    for world in (2, 3, 4, 11):
        shards = pipeline.shard_ranges(len(y), cfg.flow.redetect_interval, world)
        parts = []
        for sh in shards:
            if sh.count:
                parts.append((sh, pipeline.motion_chunk(dy[sh.first: sh.first + sh.count + 1], sh.first, sh.count, cfg)))
            else:
                parts.append((sh, np.zeros(1, pipeline.MOTION_DT)))
        motion = pipeline.assemble_motion(len(y), parts)
        rec = pipeline.plan_corrections(motion, cfg)
        assert rec.tobytes() == ref_rec.tobytes()
        out = torch.empty_like(dy)
        for sh in shards:
            if sh.own_end > sh.own_begin:
                oy, _, _ = pipeline.compose_frames(dy[sh.own_begin: sh.own_end],
                                                   rec["correction"][sh.own_begin: sh.own_end], cfg.crop_ratio)
                out[sh.own_begin: sh.own_end] = oy
        torch.cuda.synchronize()
        assert torch.equal(out, ref_y)


def test_sequence_errors():
    y = _data.video(frames=12)[0]
    cfg = _data.small_cfg()
    cfg.smooth_radius = 40  # queue_capacity 64 < 2*40+4
    with pytest.raises(stab.InvalidConfigError):
        pipeline.stabilize_sequence(y, cfg)
    with pytest.raises(stab.InvalidInputError):
        pipeline.stabilize_sequence(y[:1], _data.small_cfg())


def _release_schedule(n, r):
    """CompensationPlanner::release (pipeline.cpp:137-150): frames released
    after each push (0-based) and at finish."""
    out, nxt = [], 0
    for k in range(n):
        size = k + 1
        rel = []
        if size >= 2 * r:
            while nxt < size and nxt + r < size:
                rel.append(nxt)
                nxt += 1
        out.append(rel)
    return out, list(range(nxt, n))


@pytest.mark.parametrize("mode,ransac,smooth,graphs", [("similarity", 0, 5, True), ("hybrid", 200, 4, True),
                                                         ("rigid", 100, 9, True), ("hybrid", 200, 4, False),
                                                         ("similarity", 0, 1, True), ("similarity", 0, 1, False)])
def test_stream_equals_stage1(mode, ransac, smooth, graphs):
    """Stage II (push one frame at a time) releases frames on the reference's
    schedule (latency r, first emission at 2r) and each released frame and
    record is bit-identical to Stage I, with the per-frame CUDA graphs and
    with one launch per kernel."""
    y, cb, cr = _data.video(frames=41, objects=2, jit_t=3.0, color=True)
    cfg = _data.small_cfg(_data.MODES[mode], ransac=ransac, smooth=smooth)
    sy, sb, sr, srec = pipeline.stabilize_sequence(y, cfg, cb, cr)
    n, (h, w) = len(y), y.shape[1:]
    s = pipeline.StreamStabilizer(cfg, w, h, cb.shape[2], cb.shape[1], graphs=graphs)
    sched, tail = _release_schedule(n, cfg.smooth_radius)
    got = []
    for k in range(n):
        rel = s.push(y[k], cb[k], cr[k])
        assert [r[0] for r in rel] == sched[k], k
        got += rel
    rel = s.finish()
    assert [r[0] for r in rel] == tail
    got += rel
    s.close()
    assert [g[0] for g in got] == list(range(n))
    for i, gy, gb, gr, grec in got:
        assert np.array_equal(gy, sy[i]) and np.array_equal(gb, sb[i]) and np.array_equal(gr, sr[i]), i
        assert grec.tobytes() == srec[i].tobytes(), i


@pytest.mark.parametrize("interval", [1, 2, 3, 7])
def test_redetect_intervals(orc, interval):
    """Other re-detection cadences than the default 5 (flow.cpp:326-330):
    Stage I against the oracle (segment map, carried points), and Stage II with
    the device several frames ahead of the host (re-detections start as soon as
    their frame has landed; interval 1 re-detects every frame, so the point
    buffers rotate every push) bitwise against Stage I."""
    import dataclasses

    y = _data.video(frames=33, objects=1, jit_t=2.5)[0]
    cfg = _data.small_cfg(_data.MODES["hybrid"], ransac=60, smooth=4)
    cfg = dataclasses.replace(cfg, flow=dataclasses.replace(cfg.flow, redetect_interval=interval))
    sy, _, _, srec = pipeline.stabilize_sequence(y, cfg)
    oy, _, _, orec = orc.stabilize_sequence(y, cfg)
    assert np.array_equal(srec["frame_kind"], orec["frame_kind"])
    tr = srec["frame_kind"] == 2
    assert np.array_equal(srec["n_tracks"][tr], orec["n_tracks"][tr])
    assert np.array_equal(srec["n_inliers"][tr], orec["n_inliers"][tr])
    for k in ("dx", "dy", "da", "dls"):
        assert np.abs(srec["delta"][k] - orec["delta"][k]).max() < 1e-6, k
    d = np.abs(sy.astype(int) - oy.astype(int))
    assert d.max() <= 1 and (d > 0).mean() < 1e-3
    for depth in (1, 6):
        s = pipeline.StreamStabilizer(cfg, y.shape[2], y.shape[1], overlap_pops=True, async_push=True, depth=depth)
        got = []
        for k in range(len(y)):
            got += s.push(y[k].copy())
        got += s.finish()
        s.close()
        assert [g[0] for g in got] == list(range(len(y)))
        for i, gy, _, _, grec in got:
            assert np.array_equal(gy, sy[i]), (depth, i)
            assert grec.tobytes() == srec[i].tobytes(), (depth, i)


@pytest.mark.parametrize("overlap", [False, True])
def test_stream_async_push_equals_stage1(overlap):
    """stabgpu_stream_push_async (push returns before the upload has landed;
    a fresh host array per frame, kept alive until the next push) releases the
    same frames, bit for bit, as the blocking push and as Stage I."""
    y, cb, cr = _data.video(frames=37, objects=2, jit_t=3.0, color=True)
    cfg = _data.small_cfg(_data.MODES["hybrid"], ransac=100, smooth=4)
    sy, sb, sr, srec = pipeline.stabilize_sequence(y, cfg, cb, cr)
    n, (h, w) = len(y), y.shape[1:]
    s = pipeline.StreamStabilizer(cfg, w, h, cb.shape[2], cb.shape[1], async_push=True, overlap_pops=overlap)
    got = []
    for k in range(n):
        got += s.push(y[k].copy(), cb[k].copy(), cr[k].copy())
    got += s.finish()
    s.close()
    assert [g[0] for g in got] == list(range(n))
    for i, gy, gb, gr, grec in got:
        assert np.array_equal(gy, sy[i]) and np.array_equal(gb, sb[i]) and np.array_equal(gr, sr[i]), i
        assert grec.tobytes() == srec[i].tobytes(), i


@pytest.mark.parametrize("name,frames", [("c1", 90), ("c3", 40)])
def test_stream_equals_oracle_config(name, frames):
    """Stage II against the CPU reference path directly (not through Stage
    I): the first frames of a BASELINE config pushed one at a time, every
    released frame and record compared with the reference's run_offline
    semantics on the same frames (oracle/_ref when built, else the C
    restatement); pixels bit-identical, parameters to 1e-9."""
    from paper_1701_03572_b200.synth import CONFIGS, Video

    from . import _parity

    cfg = CONFIGS[name]
    planes = Video(cfg.video).render(0, frames)
    y = planes[0]
    cb, cr = (planes[1], planes[2]) if len(planes) == 3 else (None, None)
    ref = _oracle.reference() if _oracle.have_reference() else orc_checker()
    kw = {"threads": 8} if ref.prefix == "ref_" else {}
    oy, ob, orr, orec = ref.stabilize_sequence(y, cfg.stab, cb, cr, **kw)
    h, w = y.shape[1:]
    s = pipeline.StreamStabilizer(cfg.stab, w, h, 0 if cb is None else cb.shape[2], 0 if cb is None else cb.shape[1])
    got = []
    for k in range(frames):
        got += s.push(y[k], None if cb is None else cb[k], None if cr is None else cr[k])
    got += s.finish()
    s.close()
    assert [g[0] for g in got] == list(range(frames))
    gy = np.stack([g[1] for g in got])
    grec = np.stack([g[4] for g in got]).reshape(-1)
    gp = [gy] + ([np.stack([g[2] for g in got]), np.stack([g[3] for g in got])] if cb is not None else [])
    op = [oy] + ([ob, orr] if cb is not None else [])
    summ = _parity.summarize(grec, orec, gp, op)
    assert summ["ok"], summ
    assert summ["max_delta_err"] <= 1e-9 and summ["max_pixel_diff"] == 0, summ


def orc_checker():
    return _oracle.oracle()


@pytest.mark.parametrize("graphs,depth", [(True, 1), (False, 1), (True, 4)])
def test_stream_overlapped_pops_long(graphs, depth):
    """pop_async / wait_pops (downloads of the frames released by the previous
    push overlap the next upload) over a stream long enough to grow the
    frame-indexed arrays (256 frames) and wrap the input ring many times, with
    the motion, release and detect chains on their three streams: frames come
    back `depth` pushes late (the device ahead of the host: re-detections start
    as soon as their frame has landed) and are bitwise Stage I."""
    y = _data.video(w=128, h=96, frames=300, jit_t=1.5)[0]
    cfg = _data.small_cfg(_data.MODES["hybrid"], ransac=50, smooth=3, corners=40, levels=2, radius=7)
    sy, _, _, srec = pipeline.stabilize_sequence(y, cfg)
    s = pipeline.StreamStabilizer(cfg, y.shape[2], y.shape[1], graphs=graphs, overlap_pops=True, depth=depth)
    sched, tail = _release_schedule(len(y), cfg.smooth_radius)
    got = []
    for k in range(len(y)):
        rel = s.push(y[k])
        assert [r[0] for r in rel] == (sched[k - depth] if k >= depth else []), k
        got += rel
    rel = s.finish()
    assert [r[0] for r in rel] == sum(sched[len(y) - depth:], []) + tail
    got += rel
    s.close()
    assert [g[0] for g in got] == list(range(len(y)))
    for i, gy, _, _, grec in got:
        assert np.array_equal(gy, sy[i]), i
        assert grec.tobytes() == srec[i].tobytes(), i


def test_stream_device_pointers():
    """push/pop take device pointers too (unified addressing): frames already
    in HBM stream through the same path with the same results."""
    import ctypes as C

    import torch

    y = _data.video(frames=16)[0]
    cfg = _data.small_cfg(smooth=3)
    sy, _, _, _ = pipeline.stabilize_sequence(y, cfg)
    h, w = y.shape[1:]
    s = pipeline.StreamStabilizer(cfg, w, h)
    dy = torch.from_numpy(y).cuda()
    out = torch.empty_like(dy)
    lib, hs = s._lib, s._h
    n = C.c_int()
    popped = []

    def pop(k):
        for _ in range(k):
            idx = C.c_int64()
            j = len(popped)
            assert lib.stabgpu_stream_pop(hs, C.byref(idx), C.c_void_p(out[j].data_ptr()), None, None, None) == 0
            popped.append(idx.value)

    for k in range(len(y)):
        assert lib.stabgpu_stream_push(hs, C.c_void_p(dy[k].data_ptr()), None, None, C.byref(n)) == 0
        pop(n.value)
    assert lib.stabgpu_stream_finish(hs, C.byref(n)) == 0
    pop(n.value)
    s.close()
    assert popped == list(range(len(y)))
    assert np.array_equal(out.cpu().numpy(), sy)


@pytest.mark.gpu
@pytest.mark.parametrize("w,h", [(256, 192), (200, 150)])
def test_stream_packed_frames(w, h):
    """A caller whose frame is one contiguous planar buffer (Y | Cb | Cr) on
    both sides: push and pop move it in one copy when the planes tile the ring
    slot exactly (plane sizes multiples of 256 B: 256x192), and plane by plane
    otherwise (200x150); both equal Stage I bit for bit, and so does the same
    stream fed from three separate arrays."""
    import ctypes as C

    y, cb, cr = _data.video(w=w, h=h, frames=18, color=True)
    cfg = _data.small_cfg(smooth=3)
    sy, sb, sr, _ = pipeline.stabilize_sequence(y, cfg, cb, cr)
    n, fl = len(y), w * h
    packed_in = np.concatenate([p.reshape(n, -1) for p in (y, cb, cr)], axis=1)
    packed_in = np.ascontiguousarray(packed_in)
    packed_out = np.zeros_like(packed_in)
    s = pipeline.StreamStabilizer(cfg, w, h, w, h)
    lib, hs = s._lib, s._h
    nr = C.c_int()
    popped = []

    def ptr(a, k, plane):
        return C.c_void_p(a.ctypes.data + k * a.strides[0] + plane * fl)

    def pop(k):
        for _ in range(k):
            idx = C.c_int64()
            j = len(popped)
            assert lib.stabgpu_stream_pop(hs, C.byref(idx), ptr(packed_out, j, 0), ptr(packed_out, j, 1),
                                          ptr(packed_out, j, 2), None) == 0
            popped.append(idx.value)

    for k in range(n):
        assert lib.stabgpu_stream_push(hs, ptr(packed_in, k, 0), ptr(packed_in, k, 1), ptr(packed_in, k, 2),
                                       C.byref(nr)) == 0
        pop(nr.value)
    assert lib.stabgpu_stream_finish(hs, C.byref(nr)) == 0
    pop(nr.value)
    s.close()
    assert popped == list(range(n))
    got = packed_out.reshape(n, 3, h, w)
    assert np.array_equal(got[:, 0], sy) and np.array_equal(got[:, 1], sb) and np.array_equal(got[:, 2], sr)


def test_stream_gray_and_errors():
    y = _data.video(frames=14)[0]
    cfg = _data.small_cfg(smooth=3)
    sy, _, _, srec = pipeline.stabilize_sequence(y, cfg)
    s = pipeline.StreamStabilizer(cfg, y.shape[2], y.shape[1])
    got = []
    for f in y:
        got += s.push(f)
    got += s.finish()
    assert [g[0] for g in got] == list(range(len(y)))
    assert all(np.array_equal(g[1], sy[g[0]]) for g in got)
    with pytest.raises(stab.SequencingError):
        s.push(y[0])  # push after finish
    s.close()
    one = pipeline.StreamStabilizer(cfg, y.shape[2], y.shape[1])
    assert one.push(y[0]) == []
    with pytest.raises(stab.InvalidInputError):
        one.finish()  # fewer than 2 frames
    one.close()


# ------------------------------------------------ colour I/O + evaluation ----
def test_colour_conversions_exhaustive_gpu():
    """Device BT.601 conversions (k_eval.cu) against the pinned C restatement,
    for every RGB and every YCbCr triple."""
    import torch
    from paper_1701_03572_b200 import evaluate
    o1, o2, _ = _oracle.colour_and_psnr(_oracle.ORACLE, "orc_")
    v = np.arange(1 << 24, dtype=np.uint32)
    trip = np.stack([(v >> 16) & 255, (v >> 8) & 255, v & 255], axis=-1).astype(np.uint8).reshape(16, 1024, 1024, 3)
    gy, gb, gr = evaluate.rgb_to_ycbcr(trip)
    oy, ob, orr = o1(trip)
    assert np.array_equal(gy.cpu().numpy(), oy) and np.array_equal(gb.cpu().numpy(), ob)
    assert np.array_equal(gr.cpu().numpy(), orr)
    g = evaluate.ycbcr_to_rgb(trip[..., 0], trip[..., 1], trip[..., 2])
    torch.cuda.synchronize()
    assert np.array_equal(g.cpu().numpy(), o2(trip[..., 0], trip[..., 1], trip[..., 2]))


@pytest.mark.parametrize("pinned,crop,zero_copy", [(False, 0.04, False), (True, 0.04, False), (True, 0.04, True),
                                                    (True, 0.0, True), (False, 0.001, False)])
def test_stabilize_rgb_equals_planes(pinned, crop, zero_copy, monkeypatch):
    """RGB in / RGB out (media_io load -> run_offline -> save) equals the
    plane path with the reference conversions around it: the staged upload
    (copy engine + conversion per chunk) and the zero-copy one (pinned input
    read by the conversion kernel over PCIe), the RGB store fused into K8
    (crop margins >= 1 px) and the planes + conversion fallback (crop 0, or a
    margin rounding to 0 px on one axis)."""
    import dataclasses

    if zero_copy:
        monkeypatch.setenv("STABGPU_RGB_ZEROCOPY", "1")
    else:
        monkeypatch.delenv("STABGPU_RGB_ZEROCOPY", raising=False)

    import torch

    from paper_1701_03572_b200._lib import check, context, load
    import ctypes as C
    o1, o2, _ = _oracle.colour_and_psnr(_oracle.ORACLE, "orc_")
    y, cb, cr = _data.video(frames=23, objects=1, color=True)
    rgb = o2(y, cb, cr)  # a plausible RGB source
    cfg = dataclasses.replace(_data.small_cfg(_data.MODES["similarity"], ransac=100), crop_ratio=crop)
    py, pb, pr = o1(rgb)
    sy, sb, sr, srec = pipeline.stabilize_sequence(py, cfg, pb, pr)
    want = o2(sy, sb, sr)
    src = torch.from_numpy(rgb).pin_memory() if pinned else torch.from_numpy(rgb)
    out = torch.empty_like(src).pin_memory() if pinned else torch.empty_like(src)
    rec = np.zeros(len(rgb), pipeline.RECORD_DT)
    c = cfg.c()
    n, h, w = y.shape
    check(load().stabgpu_stabilize_sequence_rgb(context(0).handle, C.c_void_p(src.data_ptr()), n, w, h, C.byref(c),
                                                C.c_void_p(out.data_ptr()), C.c_void_p(rec.ctypes.data)))
    assert np.array_equal(out.numpy(), want)
    assert rec.tobytes() == srec.tobytes()


def test_stabilize_rgb_config_c3():
    """BASELINE C3 (1920x1080 RGB, first 30 frames) through the RGB entry
    point with pinned buffers (fused upload + fused RGB store) against the
    reference: its own BT.601 load conversion, run_offline semantics, and its
    yuv_to_rgb at save (oracle/_ref when built, else the C restatement)."""
    import ctypes as C

    import torch

    from paper_1701_03572_b200._lib import check, context, load
    from paper_1701_03572_b200.synth import CONFIGS, Video

    cfg = CONFIGS["c3"]
    y, cb, cr = Video(cfg.video).render(0, 30)
    ref = _oracle.reference() if _oracle.have_reference() else _oracle.oracle()
    lib, pre = (_oracle.REF, "ref_") if _oracle.have_reference() else (_oracle.ORACLE, "orc_")
    _, to_rgb, _ = _oracle.colour_and_psnr(lib, pre)
    rgb = to_rgb(y, cb, cr)  # an RGB source whose conversion gives these planes back (checked below)
    r2y, _, _ = _oracle.colour_and_psnr(lib, pre)
    py, pb, pr = r2y(rgb)
    kw = {"threads": 8} if ref.prefix == "ref_" else {}
    oy, ob, orr, orec = ref.stabilize_sequence(py, cfg.stab, pb, pr, **kw)
    want = to_rgb(oy, ob, orr)
    src = torch.from_numpy(rgb).pin_memory()
    out = torch.empty_like(src).pin_memory()
    rec = np.zeros(len(rgb), pipeline.RECORD_DT)
    c = cfg.stab.c()
    n, h, w = py.shape
    check(load().stabgpu_stabilize_sequence_rgb(context(0).handle, C.c_void_p(src.data_ptr()), n, w, h, C.byref(c),
                                                C.c_void_p(out.data_ptr()), C.c_void_p(rec.ctypes.data)))
    assert np.array_equal(rec["frame_kind"], orec["frame_kind"])
    assert np.array_equal(out.numpy(), want)


@pytest.mark.parametrize("crop", [0.0, 0.04])
def test_interframe_psnr_bitexact(crop):
    from paper_1701_03572_b200 import evaluate
    _, _, opsnr = _oracle.colour_and_psnr(_oracle.ORACLE, "orc_")
    y = _data.video(frames=9, jit_t=3.0)[0]
    y[4] = y[3]  # an identical pair: infinite PSNR
    g = evaluate.interframe_psnr(y, crop)
    want = [opsnr(y[i - 1], y[i], crop) for i in range(1, len(y))]
    assert g == want


@pytest.mark.skipif(not _oracle.have_reference(), reason="reference library not built")
def test_score_matches_reference():
    """evaluate.score (synth_eval.cpp:303-349) against the reference's own
    score(): PSNRs bit-identical, jitter energies within tracking tolerance."""
    from paper_1701_03572_b200 import evaluate
    reest, rscore = _oracle.ref_eval()
    y = _data.video(w=192, h=144, frames=21, jit_t=3.0)[0]
    cfg = _data.small_cfg(_data.MODES["similarity"])
    sy, _, _, rec = pipeline.stabilize_sequence(y, cfg)
    truth = rec["delta"].copy()
    truth["dx"] += 0.01  # any truth vector exercises the recovery RMSE
    est = rec["delta"]
    g = evaluate.score(y, sy, truth, est, crop_ratio=0.04)
    r = rscore(y, sy, truth, est, 0.04)
    assert g.mean_psnr_before == r[0] and g.mean_psnr_after == r[1]
    assert np.allclose(g.jitter_energy_before, r[2:6], rtol=0, atol=1e-6)
    assert np.allclose(g.jitter_energy_after, r[6:10], rtol=0, atol=1e-6)
    assert np.allclose(g.truth_recovery_rmse, r[10:14], rtol=0, atol=1e-12)
    assert g.has_truth == bool(r[14]) and g.frames_skipped == int(r[15])
    d = evaluate.reestimate_deltas(y)
    rd = reest(y)
    for k in ("dx", "dy", "da", "dls"):
        assert np.abs(d[k] - rd[k]).max() <= 1e-6, k
    assert np.array_equal(d["skipped"], rd["skipped"])


@pytest.mark.parametrize("w,h", [(192, 144), (193, 145)])
def test_sequence_420_chroma(orc, w, h):
    """Y4M 4:2:0 chroma geometry ((w+1)/2 x (h+1)/2, media_io.cpp:139-145)
    through the whole Stage I: compose_plane's chroma scaling
    (image_ops.cpp:165-202) on every frame."""
    y, cb, cr = _data.video(w=w, h=h, frames=17, objects=1, jit_t=3.0, color=True)
    cb2 = np.ascontiguousarray(cb[:, ::2, ::2])
    cr2 = np.ascontiguousarray(cr[:, ::2, ::2])
    assert cb2.shape[1:] == ((h + 1) // 2, (w + 1) // 2)
    cfg = _data.small_cfg(_data.MODES["similarity"], ransac=100)
    gy, gb, gr, grec = pipeline.stabilize_sequence(y, cfg, cb2, cr2)
    oy, ob, orr, orec = orc.stabilize_sequence(y, cfg, cb2, cr2)
    _compare_records(grec, orec)
    for a, b in ((gy, oy), (gb, ob), (gr, orr)):
        mx, cnt = _offby(a, b)
        assert mx <= 1 and cnt <= 0.0005 * a.size


@pytest.mark.parametrize("radius", [3, 15, 20])
def test_sequence_lk_windows(orc, radius):
    """Stage I with the chain kernel at its window extremes (3, 15: the
    33-column template path) and the generic kernel above 31x31 (r = 20)."""
    y = _data.video(w=256, h=192, frames=16, jit_t=3.0, tex=512, blobs=200)[0]
    cfg = _data.small_cfg(_data.MODES["similarity"], radius=radius, levels=3)
    gy, _, _, grec = pipeline.stabilize_sequence(y, cfg)
    oy, _, _, orec = orc.stabilize_sequence(y, cfg)
    _compare_records(grec, orec)
    mx, cnt = _offby(gy, oy)
    assert mx <= 1 and cnt <= 0.0005 * gy.size


# ---- multi-stream Stage I (BASELINE configs[4]) ------------------------------
def _streams(S, frames, color=True, seed=20):
    vids = [_data.video(frames=frames, objects=1, color=color, seed=seed + k, jit_t=2.0 + k)
            for k in range(S)]
    y = np.stack([v[0] for v in vids])
    if not color:
        return y, None, None
    return y, np.stack([v[1] for v in vids]), np.stack([v[2] for v in vids])


@pytest.mark.parametrize("frames,mode,ransac", [(25, "hybrid", 200), (23, "rigid", 100),
                                                (21, "similarity", 0), (2, "similarity", 0)])
def test_streams_equal_each_stream_alone(orc, frames, mode, ransac):
    """Every stream of a batched call is bitwise the one-sequence run of that
    stream (records and planes), and matches the CPU oracle.  frames=25 takes
    the strided detection batch (F % R == 0), 23 and 21 the per-stream one."""
    S = 4
    y, cb, cr = _streams(S, frames)
    cfg = _data.small_cfg(_data.MODES[mode], ransac=ransac)
    gy, gb, gr, rec = pipeline.stabilize_streams(y, cfg, cb, cr)
    assert rec.shape == (S, frames)
    for k in range(S):
        sy, sb, sr, srec = pipeline.stabilize_sequence(y[k], cfg, cb[k], cr[k])
        assert rec[k].tobytes() == srec.tobytes(), k
        assert np.array_equal(gy[k], sy) and np.array_equal(gb[k], sb) and np.array_equal(gr[k], sr), k
    for k in (0, S - 1):
        oy, ob, orr, o_rec = orc.stabilize_sequence(y[k], cfg, cb[k], cr[k])
        _compare_records(rec[k], o_rec)
        mx, cnt = _offby(gy[k], oy)
        assert mx <= 1 and cnt <= 0.0005 * oy.size


def test_streams_grouped_host_path_and_device(monkeypatch):
    """The host entry point moves groups of streams through two device slots;
    forcing 2 streams per group (3 groups) must not change a byte, and the
    device-resident entry point agrees."""
    import torch
    S, F = 5, 16
    y, _, _ = _streams(S, F, color=False, seed=40)
    cfg = _data.small_cfg(_data.MODES["hybrid"], ransac=50)
    ay, _, _, arec = pipeline.stabilize_streams(y, cfg)
    monkeypatch.setenv("STABGPU_STREAMS_PER_GROUP", "2")
    by, _, _, brec = pipeline.stabilize_streams(y, cfg)
    assert np.array_equal(ay, by) and arec.tobytes() == brec.tobytes()
    dy, _, _, drec = pipeline.stabilize_streams_device(torch.from_numpy(y).cuda(), cfg)
    torch.cuda.synchronize()
    assert np.array_equal(dy.cpu().numpy(), ay) and drec.tobytes() == arec.tobytes()
    for k in range(S):
        sy, _, _, srec = pipeline.stabilize_sequence(y[k], cfg)
        assert np.array_equal(ay[k], sy) and arec[k].tobytes() == srec.tobytes()


def test_streams_errors():
    y, _, _ = _streams(2, 8, color=False)
    cfg = _data.small_cfg()
    with pytest.raises(stab.InvalidInputError):
        pipeline.stabilize_streams(y[:, :1], cfg)
    with pytest.raises(stab.InvalidInputError):
        pipeline.stabilize_streams(y[:0], cfg)
    bad = _data.small_cfg()
    bad.smooth_radius = 40
    with pytest.raises(stab.InvalidConfigError):
        pipeline.stabilize_streams(y, bad)


@pytest.mark.parametrize("color", [False, True])
def test_sharded_entry_points_equal_single(color):
    """The C-ABI sharded Stage I: the host split (shard_motion -> host
    all-gather -> shard_compose) for 2, 3, 4 and 11 ranks emulated in one
    process (one context per rank, as one rank per GPU would have), the
    one-call host entry point, and the device entry point over a 1-rank NCCL
    communicator, all bitwise equal to the one-GPU run."""
    import ctypes as C

    import torch

    from paper_1701_03572_b200 import _lib

    y, cb, cr = _data.video(frames=53, objects=1, color=True)
    if not color:
        cb = cr = None
    cfg = _data.small_cfg(_data.MODES["hybrid"], ransac=100)
    n, h, w = y.shape
    ch, cw = (0, 0) if cb is None else cb.shape[1:]
    ref_y, ref_b, ref_r, ref_rec = pipeline.stabilize_sequence(y, cfg, cb, cr)
    R = cfg.flow.redetect_interval
    for world in (2, 3, 4, 11):
        shards = [pipeline.shard_range_c(n, R, world, g) for g in range(world)]
        assert shards == pipeline.shard_ranges(n, R, world)
        ctxs = [_lib.Context(0) for _ in range(world)]
        parts = []
        for sh, ctx in zip(shards, ctxs):
            sl = slice(sh.first, sh.first + sh.count + 1)
            parts.append((sh, pipeline.shard_motion(ctx, n, world, sh.rank, y[sl], cfg,
                                                    None if cb is None else cb[sl], None if cr is None else cr[sl])))
        motion = pipeline.assemble_motion(n, parts)
        out = [np.zeros_like(a) if a is not None else None for a in (y, cb, cr)]
        for sh, ctx in zip(shards, ctxs):
            a, b = sh.own_begin, sh.own_end
            oy = np.zeros((max(b - a, 1), h, w), np.uint8)
            ob = orr = None
            if cb is not None:
                ob, orr = (np.zeros((max(b - a, 1), ch, cw), np.uint8) for _ in range(2))
            rec = pipeline.shard_compose(ctx, n, world, sh.rank, motion, cfg, w, h, cw, ch, oy, ob, orr)
            assert rec.tobytes() == ref_rec.tobytes(), (world, sh.rank)
            if b > a:
                out[0][a:b] = oy[: b - a]
                if cb is not None:
                    out[1][a:b], out[2][a:b] = ob[: b - a], orr[: b - a]
        for c in ctxs:
            c.close()
        assert np.array_equal(out[0], ref_y), world
        if cb is not None:
            assert np.array_equal(out[1], ref_b) and np.array_equal(out[2], ref_r)
    # one-call entry points, world 1 (no communicator, then a 1-rank NCCL one)
    ctx = _lib.Context(0)
    oy, ob, orr = np.zeros_like(y), None if cb is None else np.zeros_like(cb), None if cr is None else np.zeros_like(cr)
    rec = pipeline.stabilize_sharded_host(ctx, n, y, cfg, cb, cr, oy, ob, orr)
    assert rec.tobytes() == ref_rec.tobytes() and np.array_equal(oy, ref_y)
    uid = np.zeros(128, np.uint8)
    _lib.check(_lib.load().stabgpu_nccl_unique_id(C.c_void_p(uid.ctypes.data)))
    _lib.check(_lib.load().stabgpu_comm_init(ctx.handle, C.c_void_p(uid.ctypes.data), 1, 0))
    oy2 = np.zeros_like(y)
    rec2 = pipeline.stabilize_sharded_host(ctx, n, y, cfg, cb, cr, oy2, ob, orr)
    assert rec2.tobytes() == ref_rec.tobytes() and np.array_equal(oy2, ref_y)
    if cb is not None:
        assert np.array_equal(ob, ref_b) and np.array_equal(orr, ref_r)
    dev = [None if a is None else torch.from_numpy(a).cuda() for a in (y, cb, cr)]
    outs = [None if a is None else torch.empty_like(a) for a in dev]
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    rec3 = pipeline.stabilize_sharded_device(ctx, n, dev[0], cfg, dev[1], dev[2], *outs)
    torch.cuda.synchronize()
    assert rec3.tobytes() == ref_rec.tobytes() and np.array_equal(outs[0].cpu().numpy(), ref_y)
    ctx.close()


def test_device_tracker_matches_reference_tracker(orc):
    """stabgpu_tracker_* (Tracker::advance with device-resident state, the
    drop-in's Tracker) against the reference Tracker's semantics restated
    with the oracle's stage functions (flow.cpp:297-337): same kinds, same
    TrackSets (positions to 1e-9 px), same active point counts."""
    import ctypes as C

    from paper_1701_03572_b200 import _lib

    y = _data.video(320, 240, frames=23, jit_t=3.0, tex=512, blobs=200)[0]
    fc, dc = FlowConfig(max_levels=3), DetectConfig(max_corners=80, min_distance=6.0)
    lib = _lib.load()
    ctx = _lib.Context(0)
    h = C.c_void_p()
    f_c, d_c = fc.c(), dc.c()
    _lib.check(lib.stabgpu_tracker_create(ctx.handle, C.byref(f_c), C.byref(d_c), 320, 240, C.byref(h)))
    pts, prev_pyr = None, None
    since = 0
    for i in range(len(y)):
        p = np.zeros((dc.max_corners, 2))
        q = np.zeros((dc.max_corners, 2))
        kind, n, act = C.c_int(), C.c_int(), C.c_int()
        _lib.check(lib.stabgpu_tracker_advance(h, C.c_void_p(np.ascontiguousarray(y[i]).ctypes.data), i, C.byref(kind),
                                               C.c_void_p(p.ctypes.data), C.c_void_p(q.ctypes.data), C.byref(n),
                                               C.byref(act)))
        pyr = orc.build_pyramid(y[i], fc.max_levels)[0]
        if prev_pyr is None:
            pts, _ = orc.detect_corners(y[i], dc)
            assert kind.value == _abi.FRAME_FIRST and act.value == len(pts)
        else:
            fwd, ok = orc.track_lk(prev_pyr, pyr, pts, fc)
            kp, kc = orc.weed_tracks(prev_pyr, pyr, pts[ok], fwd[ok], fc)
            assert n.value == len(kp), i
            assert np.abs(p[: n.value] - kp).max(initial=0) <= 1e-9 and np.abs(q[: n.value] - kc).max(initial=0) <= 1e-9
            want = _abi.FRAME_SKIPPED if len(kp) < fc.min_tracks else _abi.FRAME_TRACKED
            assert kind.value == want
            pts = kc
            since += 1
            if since >= fc.redetect_interval:
                pts, _ = orc.detect_corners(y[i], dc)
                since = 0
            assert act.value == len(pts), i
        prev_pyr = pyr
    with pytest.raises(stab.SequencingError):
        _lib.check(lib.stabgpu_tracker_advance(h, C.c_void_p(np.ascontiguousarray(y[0]).ctypes.data), 3, C.byref(kind),
                                               C.c_void_p(p.ctypes.data), C.c_void_p(q.ctypes.data), C.byref(n), None))
    lib.stabgpu_tracker_destroy(h)
    ctx.close()
