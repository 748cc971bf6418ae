"""Python mirror of the reference stage API (namespace ``stab``,
/root/reference/proj/include/stab/*.hpp), executed on the B200 through the
C ABI in include/stabgpu.h.

Same names, same argument meaning, same error classes (raised where the
reference throws).  Frames are 2-D ``uint8`` arrays (GrayFrame); points are
``(n, 2)`` float64 arrays of (x, y) (Point2); pyramids are :class:`Pyramid`
objects (a packed host buffer plus level views).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from ._lib import (CudaError, DegenerateInputError, InvalidConfigError, InvalidInputError,  # noqa: F401
                   InvalidTransformError, IoError, SequencingError, StabError, check, context,
                   load)

RIGID, SIMILARITY = _abi.RIGID, _abi.SIMILARITY
HYBRID, FORCE_RIGID, FORCE_SIMILARITY = _abi.HYBRID, _abi.FORCE_RIGID, _abi.FORCE_SIMILARITY
K_MIN_FRAME_DIM = 16  # frame.hpp:12


def _ptr(a: np.ndarray | None) -> C.c_void_p:
    return C.c_void_p(0 if a is None else a.ctypes.data)


def _frame(f) -> np.ndarray:
    a = np.ascontiguousarray(f, dtype=np.uint8)
    if a.ndim != 2:
        raise InvalidInputError("frame must be a 2-D uint8 array")
    return a


def _points(p) -> np.ndarray:
    a = np.ascontiguousarray(p, dtype=np.float64).reshape(-1, 2)
    return a


# ---------------------------------------------------------------- configs ----
@dataclass
class DetectConfig:  # features.hpp:15-21
    max_corners: int = 50
    quality_level: float = 0.01
    min_distance: float = 10.0
    block_size: int = 3
    roi_margin: float = 0.1

    def c(self) -> _abi.DetectCfg:
        return _abi.DetectCfg(self.max_corners, self.quality_level, self.min_distance,
                              self.block_size, self.roi_margin)


@dataclass
class FlowConfig:  # flow.hpp:13-21
    window_radius: int = 10
    max_levels: int = 4
    max_iterations: int = 30
    epsilon: float = 0.01
    fb_threshold: float = 0.5
    redetect_interval: int = 5
    min_tracks: int = 8

    def c(self) -> _abi.FlowCfg:
        return _abi.FlowCfg(self.window_radius, self.max_levels, self.max_iterations, self.epsilon,
                            self.fb_threshold, self.redetect_interval, self.min_tracks)


@dataclass
class RansacConfig:
    """Robust wrapper (new; the reference has none)."""
    iterations: int = 0
    threshold: float = 3.0
    seed: int = 0

    def c(self) -> _abi.RansacCfg:
        return _abi.RansacCfg(self.iterations, self.threshold, self.seed)


@dataclass
class SelectorConfig:  # motion.hpp:29-33
    dwell: int = 20
    margin: float = 0.05
    mode: int = HYBRID


@dataclass
class StabConfig:  # pipeline.hpp:15-22
    detect: DetectConfig = field(default_factory=DetectConfig)
    flow: FlowConfig = field(default_factory=FlowConfig)
    smooth_radius: int = 10  # SmoothConfig.radius, smoothing.hpp:11-13
    selector: SelectorConfig = field(default_factory=SelectorConfig)
    ransac: RansacConfig = field(default_factory=RansacConfig)
    crop_ratio: float = 0.04
    queue_capacity: int = 64

    def c(self) -> _abi.Config:
        return _abi.Config(self.detect.c(), self.flow.c(), self.smooth_radius,
                           _abi.SelectorCfg(self.selector.dwell, self.selector.margin,
                                            self.selector.mode),
                           self.ransac.c(), self.crop_ratio, self.queue_capacity)


def validate(cfg: StabConfig) -> None:
    """validate(StabConfig), pipeline.cpp:17-28 (raises InvalidConfigError)."""
    c = cfg.c()
    check(load().stabgpu_validate_config(C.byref(c)))


# ---------------------------------------------------------------- values -----
@dataclass
class SimilarityTransform:  # transform.hpp:13-32
    tx: float = 0.0
    ty: float = 0.0
    theta: float = 0.0
    s: float = 1.0
    kind: int = SIMILARITY

    def c(self) -> _abi.Transform:
        return _abi.Transform(self.tx, self.ty, self.theta, self.s, self.kind)

    @staticmethod
    def of(t: _abi.Transform) -> "SimilarityTransform":
        return SimilarityTransform(t.tx, t.ty, t.theta, t.s, t.kind)


@dataclass
class DeltaParams:  # transform.hpp:42-49
    dx: float = 0.0
    dy: float = 0.0
    da: float = 0.0
    dls: float = 0.0
    kind: int = RIGID
    skipped: bool = False


@dataclass
class RoiRect:  # features.hpp:27-36
    x0: int
    y0: int
    x1: int
    y1: int

    def width(self) -> int:
        return self.x1 - self.x0

    def height(self) -> int:
        return self.y1 - self.y0


@dataclass
class TrackSet:  # flow.hpp:43-50
    prev_points: np.ndarray
    cur_points: np.ndarray
    frame_index: int = 0

    def size(self) -> int:
        return len(self.prev_points)


class Pyramid:
    """Pyramid (frame.hpp:43-49): packed levels in one host buffer."""

    def __init__(self, w: int, h: int, max_levels: int):
        nbytes = load().stabgpu_pyramid_bytes(w, h, max_levels)
        self.buf = np.zeros(max(nbytes, 1), np.uint8)
        self.c = _abi.Pyramid()
        self.c.data = self.buf.ctypes.data_as(_abi.c_u8p)

    @property
    def levels(self) -> list[np.ndarray]:
        out = []
        for i in range(self.c.levels):
            w, h, o = self.c.width[i], self.c.height[i], self.c.offset[i]
            out.append(self.buf[o:o + w * h].reshape(h, w))
        return out

    def level_count(self) -> int:
        return self.c.levels

    @staticmethod
    def from_levels(levels: list[np.ndarray]) -> "Pyramid":
        p = Pyramid.__new__(Pyramid)
        p.buf = np.concatenate([np.ascontiguousarray(l, np.uint8).ravel() for l in levels])
        p.c = _abi.Pyramid()
        p.c.levels = len(levels)
        off = 0
        for i, l in enumerate(levels):
            p.c.height[i], p.c.width[i] = l.shape
            p.c.offset[i] = off
            off += l.size
        p.c.data = p.buf.ctypes.data_as(_abi.c_u8p)
        return p


# ------------------------------------------------------------- image_ops -----
def build_pyramid(frame, max_levels: int, device: int = 0) -> Pyramid:
    """build_pyramid, image_ops.hpp:12 / image_ops.cpp:62-77."""
    f = _frame(frame)
    h, w = f.shape
    if w < K_MIN_FRAME_DIM or h < K_MIN_FRAME_DIM:
        raise InvalidInputError("frame smaller than 16x16")
    if max_levels < 1:
        raise InvalidInputError("max_levels must be >= 1")
    p = Pyramid(w, h, max_levels)
    check(load().stabgpu_build_pyramid(context(device).handle, _ptr(f), w, h, max_levels,
                                       C.byref(p.c)))
    return p


def build_pyramid_batch(frames, max_levels: int, device: int = 0) -> list[list[np.ndarray]]:
    """build_pyramid of every frame of an (n, h, w) stack in the batched
    per-level launches Stage I uses -> per frame, its list of levels."""
    f = np.ascontiguousarray(frames, np.uint8)
    if f.ndim != 3:
        raise InvalidInputError("frames must be (n, h, w)")
    n, h, w = f.shape
    if w < K_MIN_FRAME_DIM or h < K_MIN_FRAME_DIM:
        raise InvalidInputError("frame smaller than 16x16")
    if max_levels < 1:
        raise InvalidInputError("max_levels must be >= 1")
    lib = load()
    per = lib.stabgpu_pyramid_bytes(w, h, max_levels)
    out = np.empty((n, per), np.uint8)
    check(lib.stabgpu_build_pyramid_batch(context(device).handle, _ptr(f), n, w, h, max_levels, _ptr(out)))
    dims = []
    lw, lh = w, h
    for lev in range(max_levels):  # image_ops.cpp:71
        if lev > 0:
            if lw // 2 < K_MIN_FRAME_DIM or lh // 2 < K_MIN_FRAME_DIM:
                break
            lw, lh = lw // 2, lh // 2
        dims.append((lh, lw))
    res = []
    for i in range(n):
        off, lv = 0, []
        for (hh, ww) in dims:
            lv.append(out[i, off:off + hh * ww].reshape(hh, ww))
            off += hh * ww
        res.append(lv)
    return res


def gradients(frame, device: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """gradients, image_ops.hpp:15 / image_ops.cpp:79-96."""
    f = _frame(frame)
    gx = np.empty(f.shape, np.float64)
    gy = np.empty(f.shape, np.float64)
    check(load().stabgpu_gradients(context(device).handle, _ptr(f), f.shape[1], f.shape[0],
                                   _ptr(gx), _ptr(gy)))
    return gx, gy


def warp_similarity(frame, t: SimilarityTransform, device: int = 0) -> np.ndarray:
    """warp_similarity, image_ops.hpp:23 / image_ops.cpp:115-134."""
    f = _frame(frame)
    out = np.empty_like(f)
    tc = t.c()
    check(load().stabgpu_warp_similarity(context(device).handle, _ptr(f), f.shape[1], f.shape[0],
                                         C.byref(tc), _ptr(out)))
    return out


def crop_resize(frame, crop_ratio: float, device: int = 0) -> np.ndarray:
    """crop_resize, image_ops.hpp:27 / image_ops.cpp:136-159."""
    f = _frame(frame)
    out = np.empty_like(f)
    check(load().stabgpu_crop_resize(context(device).handle, _ptr(f), f.shape[1], f.shape[0],
                                     crop_ratio, _ptr(out)))
    return out


def compose_stabilized(luma, correction: SimilarityTransform, crop_ratio: float, cb=None, cr=None,
                       device: int = 0):
    """compose_stabilized, image_ops.hpp:32-33 / image_ops.cpp:206-219.

    Returns the output luma, or (luma, cb, cr) when chroma planes are given."""
    y = _frame(luma)
    h, w = y.shape
    oy = np.empty_like(y)
    tc = correction.c()
    if cb is None:
        check(load().stabgpu_compose_stabilized(context(device).handle, _ptr(y), None, None, w, h,
                                                0, 0, C.byref(tc), crop_ratio, _ptr(oy), None, None))
        return oy
    b, r = _frame(cb), _frame(cr)
    ob, orr = np.empty_like(b), np.empty_like(r)
    check(load().stabgpu_compose_stabilized(context(device).handle, _ptr(y), _ptr(b), _ptr(r), w, h,
                                            b.shape[1], b.shape[0], C.byref(tc), crop_ratio,
                                            _ptr(oy), _ptr(ob), _ptr(orr)))
    return oy, ob, orr


# -------------------------------------------------------------- features -----
def detection_roi(frame_or_shape, roi_margin: float) -> RoiRect:
    """detection_roi, features.hpp:40 / features.cpp:28-36."""
    h, w = frame_or_shape.shape if hasattr(frame_or_shape, "shape") else frame_or_shape
    r = _abi.Roi()
    check(load().stabgpu_detection_roi(w, h, roi_margin, C.byref(r)))
    return RoiRect(r.x0, r.y0, r.x1, r.y1)


def min_eig_response(frame, block_size: int, device: int = 0) -> np.ndarray:
    """min_eig_response, features.hpp:44 / features.cpp:78-87."""
    f = _frame(frame)
    out = np.empty(f.shape, np.float64)
    check(load().stabgpu_min_eig_response(context(device).handle, _ptr(f), f.shape[1], f.shape[0],
                                          block_size, _ptr(out)))
    return out


def detect_corners(frame, cfg: DetectConfig, device: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """detect_corners, features.hpp:49 / features.cpp:89-141.

    Returns (positions (n,2), scores (n,)) in selection order."""
    f = _frame(frame)
    xy = np.empty((max(cfg.max_corners, 1), 2), np.float64)
    sc = np.empty(max(cfg.max_corners, 1), np.float64)
    n = C.c_int(0)
    cc = cfg.c()
    check(load().stabgpu_detect_corners(context(device).handle, _ptr(f), f.shape[1], f.shape[0],
                                        C.byref(cc), _ptr(xy), _ptr(sc), C.byref(n)))
    return xy[:n.value].copy(), sc[:n.value].copy()


def detect_corners_batch(frames, cfg: DetectConfig, device: int = 0) -> list[tuple[np.ndarray, np.ndarray]]:
    """detect_corners on every frame of an (n, h, w) stack in one batched
    launch (the K2-K4 batch Stage I runs); frame f's result equals
    detect_corners(frames[f])."""
    f = np.ascontiguousarray(frames, np.uint8)
    if f.ndim != 3:
        raise InvalidInputError("frames must be (n, h, w)")
    nb, h, w = f.shape
    m = max(cfg.max_corners, 1)
    xy = np.empty((nb, m, 2), np.float64)
    sc = np.empty((nb, m), np.float64)
    nn = np.zeros(nb, np.int32)
    cc = cfg.c()
    check(load().stabgpu_detect_corners_batch(context(device).handle, _ptr(f), nb, w, h, C.byref(cc),
                                              _ptr(xy), _ptr(sc), nn.ctypes.data_as(C.POINTER(C.c_int))))
    return [(xy[i, :nn[i]].copy(), sc[i, :nn[i]].copy()) for i in range(nb)]


# ------------------------------------------------------------------ flow -----
def track_lk(prev: Pyramid, cur: Pyramid, points, cfg: FlowConfig, device: int = 0):
    """track_lk, flow.hpp:35-36 / flow.cpp:243-256 -> (positions (n,2), ok (n,) bool)."""
    pts = _points(points)
    n = len(pts)
    out = np.empty_like(pts)
    ok = np.zeros(n, np.uint8)
    fc = cfg.c()
    check(load().stabgpu_track_lk(context(device).handle, C.byref(prev.c), C.byref(cur.c),
                                  _ptr(pts), n, C.byref(fc), _ptr(out), _ptr(ok)))
    return out, ok.astype(bool)


def weed_tracks(prev: Pyramid, cur: Pyramid, prev_points, cur_points, cfg: FlowConfig,
                device: int = 0) -> TrackSet:
    """weed_tracks, flow.hpp:51-52 / flow.cpp:258-280."""
    p, q = _points(prev_points), _points(cur_points)
    if len(p) != len(q):
        raise InvalidInputError("prev/cur point lists must be index-aligned")
    n = len(p)
    kp, kc = np.empty_like(p), np.empty_like(q)
    m = C.c_int(0)
    fc = cfg.c()
    check(load().stabgpu_weed_tracks(context(device).handle, C.byref(prev.c), C.byref(cur.c),
                                     _ptr(p), _ptr(q), n, C.byref(fc), _ptr(kp), _ptr(kc),
                                     C.byref(m)))
    return TrackSet(kp[:m.value].copy(), kc[:m.value].copy())


# ---------------------------------------------------------------- motion -----
def _estimate(ts: TrackSet, kind: int, device: int) -> SimilarityTransform:
    p, q = _points(ts.prev_points), _points(ts.cur_points)
    t = _abi.Transform()
    check(load().stabgpu_estimate(context(device).handle, _ptr(p), _ptr(q), len(p), kind,
                                  C.byref(t)))
    return SimilarityTransform.of(t)


def estimate_similarity(ts: TrackSet, device: int = 0) -> SimilarityTransform:
    """estimate_similarity, motion.hpp:13 / motion.cpp:62-70."""
    return _estimate(ts, SIMILARITY, device)


def estimate_rigid(ts: TrackSet, device: int = 0) -> SimilarityTransform:
    """estimate_rigid, motion.hpp:16 / motion.cpp:72-76."""
    return _estimate(ts, RIGID, device)


def ransac_estimate(ts: TrackSet, kind: int, cfg: RansacConfig, min_tracks: int = 8,
                    frame_index: int = 0, device: int = 0):
    """Robust fit -> (transform, inlier mask)."""
    p, q = _points(ts.prev_points), _points(ts.cur_points)
    t = _abi.Transform()
    mask = np.zeros(len(p), np.uint8)
    used = C.c_int(0)
    rc = cfg.c()
    check(load().stabgpu_ransac_estimate(context(device).handle, _ptr(p), _ptr(q), len(p), kind,
                                         C.byref(rc), min_tracks, frame_index, C.byref(t),
                                         _ptr(mask), C.byref(used)))
    return SimilarityTransform.of(t), mask.astype(bool)


def rms_residual(ts: TrackSet, t: SimilarityTransform, device: int = 0) -> float:
    """rms_residual, motion.hpp:19 / motion.cpp:78-90."""
    p, q = _points(ts.prev_points), _points(ts.cur_points)
    out = C.c_double(0.0)
    tc = t.c()
    check(load().stabgpu_rms_residual(context(device).handle, _ptr(p), _ptr(q), len(p),
                                      C.byref(tc), C.byref(out)))
    return out.value


def extract_delta(t: SimilarityTransform) -> DeltaParams:
    """extract_delta, motion.cpp:92-101."""
    d = _abi.Delta()
    tc = t.c()
    load().stabgpu_extract_delta(C.byref(tc), C.byref(d))
    return DeltaParams(d.dx, d.dy, d.da, d.dls, d.kind, bool(d.skipped))


def delta_to_transform(dx: float, dy: float, da: float, dls: float) -> SimilarityTransform:
    """delta_to_transform, motion.cpp:103-111."""
    t = _abi.Transform()
    load().stabgpu_delta_to_transform(dx, dy, da, dls, C.byref(t))
    return SimilarityTransform.of(t)


def trajectory_corrections(deltas, radius: int, device: int = 0) -> np.ndarray:
    """Trajectory::append + correction over a complete trajectory
    (smoothing.cpp:16-57).  deltas: (n,4) [dx,dy,da,dls] -> (n,4) [tx,ty,theta,s]."""
    d = np.ascontiguousarray(deltas, np.float64).reshape(-1, 4)
    n = len(d)
    arr = (_abi.Delta * max(n, 1))()
    for i in range(n):
        arr[i].dx, arr[i].dy, arr[i].da, arr[i].dls = d[i]
    out = (_abi.Transform * max(n, 1))()
    check(load().stabgpu_trajectory_corrections(context(device).handle, arr, n, radius, out))
    return np.array([[o.tx, o.ty, o.theta, o.s] for o in out[:n]], np.float64).reshape(-1, 4)
