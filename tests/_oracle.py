"""Test-side loaders for the CPU checkers (TEST INFRASTRUCTURE ONLY).

liboracle.so  : the C restatement in oracle/stab_oracle.c (orc_* symbols)
libstabref.so : the unmodified reference compiled from its own sources plus
                oracle/ref_glue.cpp (ref_* symbols); built only where
                /root/reference exists, shipped prebuilt to the GPU box.
Both share the struct layouts of include/stabgpu.h (paper_1701_03572_b200/_abi.py).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_1701_03572_b200 import _abi
from paper_1701_03572_b200.pipeline import MOTION_DT, RECORD_DT

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE = os.path.join(ROOT, "oracle", "liboracle.so")
REF = os.path.join(ROOT, "oracle", "_ref", "libstabref.so")

P, V, I, D = C.POINTER, C.c_void_p, C.c_int, C.c_double
A = _abi
PROTO = {
    "last_error": (C.c_char_p, []),
    "pyramid_bytes": (C.c_size_t, [I, I, I]),
    "build_pyramid": (I, [V, I, I, I, P(A.Pyramid)]),
    "gradients": (I, [V, I, I, V, V]),
    "min_eig_response": (I, [V, I, I, I, V]),
    "detection_roi": (I, [I, I, D, P(A.Roi)]),
    "detect_corners": (I, [V, I, I, P(A.DetectCfg), V, V, P(I)]),
    "track_lk": (I, [P(A.Pyramid), P(A.Pyramid), V, I, P(A.FlowCfg), V, V]),
    "weed_tracks": (I, [P(A.Pyramid), P(A.Pyramid), V, V, I, P(A.FlowCfg), V, V, P(I)]),
    "estimate": (I, [V, V, I, I, P(A.Transform)]),
    "rms_residual": (I, [V, V, I, P(A.Transform), P(D)]),
    "ransac_estimate": (I, [V, V, I, I, P(A.RansacCfg), I, C.c_int64, P(A.Transform), V, P(I)]),
    "extract_delta": (None, [P(A.Transform), P(A.Delta)]),
    "delta_to_transform": (None, [D, D, D, D, P(A.Transform)]),
    "trajectory_corrections": (I, [V, I, I, V]),
    "warp_similarity": (I, [V, I, I, P(A.Transform), V]),
    "crop_resize": (I, [V, I, I, D, V]),
    "compose_stabilized": (I, [V, V, V, I, I, I, I, P(A.Transform), D, V, V, V]),
}
ORC_ONLY = {"stabilize_sequence": (I, [V, V, V, I, I, I, I, I, P(A.Config), V, V, V, V])}
REF_ONLY = {
    "stabilize_sequence": (I, [V, V, V, I, I, I, I, I, P(A.Config), V, V, V, V, I]),
    "run_offline": (I, [V, V, V, I, I, I, I, I, P(A.Config), V, V, V, V, V, P(D)]),
    "motion_chunk": (I, [V, C.c_longlong, I, I, I, P(A.Config), V]),
    "plan_corrections": (I, [V, I, P(A.Config), V]),
}


def _vp(a):
    return C.c_void_p(0) if a is None else C.c_void_p(a.ctypes.data)


class CpuImpl:
    """The same call surface over liboracle (prefix orc_) or libstabref (ref_)."""

    def __init__(self, path: str, prefix: str, extra: dict):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        self.prefix = prefix
        for name, (res, args) in {**PROTO, **extra}.items():
            fn = getattr(self.lib, prefix + name)
            fn.restype, fn.argtypes = res, args
            setattr(self, name + "_raw", fn)

    def err(self):
        return self.last_error_raw().decode()

    def check(self, rc):
        if rc != 0:
            raise RuntimeError(f"{self.prefix} rc={rc}: {self.err()}")

    # -- wrappers returning numpy ------------------------------------------
    def build_pyramid(self, f, levels):
        f = np.ascontiguousarray(f, np.uint8)
        h, w = f.shape
        buf = np.zeros(max(self.pyramid_bytes_raw(w, h, levels), 1), np.uint8)
        p = A.Pyramid()
        p.data = buf.ctypes.data_as(A.c_u8p)
        rc = self.build_pyramid_raw(_vp(f), w, h, levels, C.byref(p))
        self.check(rc)
        p._keep = buf
        return p, [buf[p.offset[i]: p.offset[i] + p.width[i] * p.height[i]].reshape(p.height[i], p.width[i])
                   for i in range(p.levels)]

    def gradients(self, f):
        f = np.ascontiguousarray(f, np.uint8)
        gx = np.empty(f.shape, np.float64)
        gy = np.empty(f.shape, np.float64)
        self.check(self.gradients_raw(_vp(f), f.shape[1], f.shape[0], _vp(gx), _vp(gy)))
        return gx, gy

    def min_eig_response(self, f, block):
        f = np.ascontiguousarray(f, np.uint8)
        out = np.empty(f.shape, np.float64)
        self.check(self.min_eig_response_raw(_vp(f), f.shape[1], f.shape[0], block, _vp(out)))
        return out

    def detect_corners(self, f, cfg):
        f = np.ascontiguousarray(f, np.uint8)
        xy = np.empty((cfg.max_corners, 2), np.float64)
        sc = np.empty(cfg.max_corners, np.float64)
        n = C.c_int(0)
        c = cfg.c()
        self.check(self.detect_corners_raw(_vp(f), f.shape[1], f.shape[0], C.byref(c), _vp(xy),
                                           _vp(sc), C.byref(n)))
        return xy[: n.value].copy(), sc[: n.value].copy()

    def track_lk(self, prev, cur, pts, cfg):
        pts = np.ascontiguousarray(pts, np.float64).reshape(-1, 2)
        out = np.empty_like(pts)
        ok = np.zeros(len(pts), np.uint8)
        c = cfg.c()
        self.check(self.track_lk_raw(C.byref(prev), C.byref(cur), _vp(pts), len(pts), C.byref(c),
                                     _vp(out), _vp(ok)))
        return out, ok.astype(bool)

    def weed_tracks(self, prev, cur, p, q, cfg):
        p = np.ascontiguousarray(p, np.float64).reshape(-1, 2)
        q = np.ascontiguousarray(q, np.float64).reshape(-1, 2)
        kp, kc = np.empty_like(p), np.empty_like(q)
        m = C.c_int(0)
        c = cfg.c()
        self.check(self.weed_tracks_raw(C.byref(prev), C.byref(cur), _vp(p), _vp(q), len(p),
                                        C.byref(c), _vp(kp), _vp(kc), C.byref(m)))
        return kp[: m.value].copy(), kc[: m.value].copy()

    def estimate(self, p, q, kind):
        p, q = np.ascontiguousarray(p, np.float64), np.ascontiguousarray(q, np.float64)
        t = A.Transform()
        rc = self.estimate_raw(_vp(p), _vp(q), len(p), kind, C.byref(t))
        return rc, t

    def ransac(self, p, q, kind, rcfg, min_tracks, frame):
        p, q = np.ascontiguousarray(p, np.float64), np.ascontiguousarray(q, np.float64)
        t = A.Transform()
        mask = np.zeros(len(p), np.uint8)
        used = C.c_int(0)
        r = rcfg.c()
        rc = self.ransac_estimate_raw(_vp(p), _vp(q), len(p), kind, C.byref(r), min_tracks, frame,
                                      C.byref(t), _vp(mask), C.byref(used))
        return rc, t, mask.astype(bool), used.value

    def rms_residual(self, p, q, t):
        p, q = np.ascontiguousarray(p, np.float64), np.ascontiguousarray(q, np.float64)
        out = C.c_double()
        self.check(self.rms_residual_raw(_vp(p), _vp(q), len(p), C.byref(t), C.byref(out)))
        return out.value

    def trajectory_corrections(self, deltas, radius):
        n = len(deltas)
        arr = (A.Delta * n)()
        for i in range(n):
            arr[i].dx, arr[i].dy, arr[i].da, arr[i].dls = deltas[i]
        out = (A.Transform * n)()
        self.check(self.trajectory_corrections_raw(arr, n, radius, out))
        return np.array([[o.tx, o.ty, o.theta, o.s] for o in out])

    def warp_similarity(self, f, t):
        f = np.ascontiguousarray(f, np.uint8)
        out = np.empty_like(f)
        self.check(self.warp_similarity_raw(_vp(f), f.shape[1], f.shape[0], C.byref(t), _vp(out)))
        return out

    def crop_resize(self, f, crop):
        f = np.ascontiguousarray(f, np.uint8)
        out = np.empty_like(f)
        self.check(self.crop_resize_raw(_vp(f), f.shape[1], f.shape[0], crop, _vp(out)))
        return out

    def compose(self, y, cb, cr, t, crop):
        y = np.ascontiguousarray(y, np.uint8)
        cb = None if cb is None else np.ascontiguousarray(cb, np.uint8)
        cr = None if cr is None else np.ascontiguousarray(cr, np.uint8)
        oy = np.empty_like(y)
        ob = None if cb is None else np.empty_like(cb)
        orr = None if cr is None else np.empty_like(cr)
        ch, cw = (0, 0) if cb is None else cb.shape
        self.check(self.compose_stabilized_raw(_vp(y), _vp(cb), _vp(cr), y.shape[1], y.shape[0],
                                               cw, ch, C.byref(t), crop, _vp(oy), _vp(ob), _vp(orr)))
        return oy, ob, orr

    def stabilize_sequence(self, y, cfg, cb=None, cr=None, compose=True, threads=1):
        y = np.ascontiguousarray(y, np.uint8)
        cb = None if cb is None else np.ascontiguousarray(cb, np.uint8)
        cr = None if cr is None else np.ascontiguousarray(cr, np.uint8)
        n, h, w = y.shape
        ch, cw = (0, 0) if cb is None else cb.shape[1:]
        oy = np.empty_like(y) if compose else None
        ob = None if (cb is None or not compose) else np.empty_like(cb)
        orr = None if (cr is None or not compose) else np.empty_like(cr)
        rec = np.zeros(n, RECORD_DT)
        c = cfg.c()
        args = [_vp(y), _vp(cb), _vp(cr), n, w, h, cw, ch, C.byref(c), _vp(oy), _vp(ob), _vp(orr),
                _vp(rec)]
        if self.prefix == "ref_":
            args.append(threads)
        self.check(self.stabilize_sequence_raw(*args))
        return oy, ob, orr, rec


_cache: dict = {}


def oracle() -> CpuImpl:
    if "orc" not in _cache:
        _cache["orc"] = CpuImpl(ORACLE, "orc_", ORC_ONLY)
    return _cache["orc"]


def reference() -> CpuImpl:
    if "ref" not in _cache:
        _cache["ref"] = CpuImpl(REF, "ref_", REF_ONLY)
    return _cache["ref"]


def have_reference() -> bool:
    return os.path.exists(REF)


def colour_and_psnr(lib_path: str, prefix: str):
    """(rgb_to_ycbcr, ycbcr_to_rgb, psnr_pair) of liboracle / libstabref."""
    lib = C.CDLL(lib_path)
    f1 = getattr(lib, prefix + "rgb_to_ycbcr")
    f1.argtypes, f1.restype = [V, C.c_size_t, V, V, V], None
    f2 = getattr(lib, prefix + "ycbcr_to_rgb")
    f2.argtypes, f2.restype = [V, V, V, C.c_size_t, V], None
    f3 = getattr(lib, prefix + "psnr_pair")
    f3.argtypes, f3.restype = [V, V, I, I, D, P(D)], I

    def rgb_to_ycbcr(rgb):
        rgb = np.ascontiguousarray(rgb, np.uint8)
        npx = rgb.size // 3
        y, cb, cr = (np.empty(rgb.shape[:-1], np.uint8) for _ in range(3))
        f1(_vp(rgb), npx, _vp(y), _vp(cb), _vp(cr))
        return y, cb, cr

    def ycbcr_to_rgb(y, cb, cr):
        y, cb, cr = (np.ascontiguousarray(a, np.uint8) for a in (y, cb, cr))
        out = np.empty(y.shape + (3,), np.uint8)
        f2(_vp(y), _vp(cb), _vp(cr), y.size, _vp(out))
        return out

    def psnr_pair(a, b, crop):
        a, b = np.ascontiguousarray(a, np.uint8), np.ascontiguousarray(b, np.uint8)
        out = C.c_double()
        rc = f3(_vp(a), _vp(b), a.shape[1], a.shape[0], crop, C.byref(out))
        if rc:
            raise ValueError(rc)
        return out.value

    return rgb_to_ycbcr, ycbcr_to_rgb, psnr_pair


def ref_eval():
    """libstabref's reestimate_deltas / score (synth_eval.cpp)."""
    lib = C.CDLL(REF)
    re_ = lib.ref_reestimate_deltas
    re_.argtypes, re_.restype = [V, I, I, I, V], I
    sc = lib.ref_score
    sc.argtypes, sc.restype = [V, V, I, I, I, V, V, I, D, V], I
    from paper_1701_03572_b200.pipeline import DELTA_DT

    def reestimate(y):
        y = np.ascontiguousarray(y, np.uint8)
        out = np.zeros(len(y), DELTA_DT)
        assert re_(_vp(y), y.shape[0], y.shape[2], y.shape[1], _vp(out)) == 0
        return out

    def score(orig, stab, truth, est, crop):
        orig, stab = np.ascontiguousarray(orig, np.uint8), np.ascontiguousarray(stab, np.uint8)
        out = np.zeros(16)
        truth = None if truth is None else np.ascontiguousarray(truth)  # record views are strided
        est = None if est is None else np.ascontiguousarray(est)
        nt = 0 if truth is None else len(truth)
        assert sc(_vp(orig), _vp(stab), orig.shape[0], orig.shape[2], orig.shape[1], _vp(truth), _vp(est), nt,
                  crop, _vp(out)) == 0
        return out

    return reestimate, score
