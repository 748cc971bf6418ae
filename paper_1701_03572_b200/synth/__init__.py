"""Seeded synthetic videos for the BASELINE.json configs (bench/test input).

The generator is host C (videogen.c, OpenMP, counter-based RNG): the same
bytes feed the GPU path and every CPU checker.  ``CONFIGS`` maps the five
BASELINE.json configs to generator settings and to the StabConfig the
stabilizer runs with (SURVEY §8 config mapping).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from ..stab import (FORCE_RIGID, FORCE_SIMILARITY, DetectConfig, FlowConfig, RansacConfig,
                    SelectorConfig, StabConfig)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(_HERE, "libvideogen.so")


class _VG(C.Structure):
    _fields_ = [("width", C.c_int), ("height", C.c_int), ("frames", C.c_int),
                ("tex_size", C.c_int), ("blobs", C.c_int), ("objects", C.c_int), ("color", C.c_int),
                ("drift", C.c_double), ("jit_t", C.c_double), ("jit_rot_deg", C.c_double),
                ("jit_scale", C.c_double), ("noise_sigma", C.c_double), ("seed", C.c_uint64)]


_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise ImportError(f"{LIB} missing: run `make` / __graft_entry__.build()")
        _lib = C.CDLL(LIB)
        _lib.vg_create.restype = C.c_void_p
        _lib.vg_create.argtypes = [C.POINTER(_VG)]
        _lib.vg_destroy.argtypes = [C.c_void_p]
        _lib.vg_render.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.vg_pose.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
        _lib.vg_set_threads.argtypes = [C.c_int]
    return _lib


@dataclass
class VideoSpec:
    width: int
    height: int
    frames: int
    tex_size: int
    blobs: int
    objects: int = 0
    color: bool = False
    drift: float = 0.5
    jit_t: float = 3.0
    jit_rot_deg: float = 0.5
    jit_scale: float = 0.005
    noise_sigma: float = 2.0
    seed: int = 0x5EED0000
    streams: int = 1  # config 5: independent streams, seeds seed ^ stream


@dataclass
class BenchConfig:
    name: str
    video: VideoSpec
    stab: StabConfig = field(default_factory=StabConfig)


def _stab(mode, corners, min_dist, levels, radius=10, ransac_iters=500) -> StabConfig:
    return StabConfig(
        detect=DetectConfig(max_corners=corners, quality_level=0.01, min_distance=min_dist,
                            block_size=3, roi_margin=0.1),
        flow=FlowConfig(window_radius=radius, max_levels=levels, max_iterations=30, epsilon=0.01),
        smooth_radius=30,
        selector=SelectorConfig(mode=mode),
        ransac=RansacConfig(iterations=ransac_iters, threshold=3.0, seed=0x5EED),
        crop_ratio=0.04,
        queue_capacity=64,
    )


# BASELINE.json configs[0..4]
CONFIGS = {
    "c1": BenchConfig("640x480 gray, 300 frames, rigid, 200 corners",
                      VideoSpec(640, 480, 300, 1024, 400, 0, False, 0.5, 3.0, 0.5, 0.005, 2.0,
                                0x5EED0000 + 1),
                      _stab(FORCE_RIGID, 200, 30.0, 3)),
    "c2": BenchConfig("1280x720 gray, 600 frames, similarity, 500 corners, 8 outlier objects",
                      VideoSpec(1280, 720, 600, 2048, 1600, 8, False, 0.5, 6.0, 1.0, 0.01, 2.0,
                                0x5EED0000 + 2),
                      _stab(FORCE_SIMILARITY, 500, 20.0, 4)),
    "c3": BenchConfig("1920x1080 RGB (Y/Cb/Cr 4:4:4), 1000 frames, similarity, 1000 corners, "
                      "12 outlier objects",
                      VideoSpec(1920, 1080, 1000, 2048, 1600, 12, True, 0.5, 8.0, 1.0, 0.01, 2.0,
                                0x5EED0000 + 3),
                      _stab(FORCE_SIMILARITY, 1000, 15.0, 4)),
    "c4": BenchConfig("3840x2160 gray, 500 frames, similarity, 2000 corners, LK 31x31, 5 levels",
                      VideoSpec(3840, 2160, 500, 4096, 1600, 0, False, 0.5, 16.0, 1.5, 0.015, 2.0,
                                0x5EED0000 + 4),
                      _stab(FORCE_SIMILARITY, 2000, 20.0, 5, radius=15, ransac_iters=1000)),
    "c5": BenchConfig("256 streams x 240 frames 1280x720 gray, rigid, 300 corners, 3 levels",
                      VideoSpec(1280, 720, 240, 2048, 1600, 0, False, 0.5, 6.0, 1.0, 0.01, 2.0,
                                0x5EED0000 + 5, streams=256),
                      _stab(FORCE_RIGID, 300, 20.0, 3)),
}


class Video:
    """A generator handle (texture built once) that renders frame ranges."""

    def __init__(self, spec: VideoSpec, stream: int = 0, threads: int = 0):
        lib = _load()
        if threads:
            lib.vg_set_threads(threads)
        self.spec = spec
        seed = spec.seed ^ stream if spec.streams > 1 else spec.seed
        c = _VG(spec.width, spec.height, spec.frames, spec.tex_size, spec.blobs, spec.objects,
                1 if spec.color else 0, spec.drift, spec.jit_t, spec.jit_rot_deg, spec.jit_scale,
                spec.noise_sigma, seed)
        self.h = lib.vg_create(C.byref(c))
        if not self.h:
            raise ValueError("bad video spec")

    def __del__(self):
        if getattr(self, "h", None):
            _load().vg_destroy(self.h)
            self.h = None

    def render(self, first: int = 0, count: int | None = None, out=None):
        """-> y (count,h,w) [, cb, cr] uint8 (colour: Y/Cb/Cr 4:4:4)."""
        s = self.spec
        count = s.frames - first if count is None else count
        shape = (count, s.height, s.width)
        if out is None:
            out = [np.empty(shape, np.uint8) for _ in range(3 if s.color else 1)]
        ptrs = [C.c_void_p(a.ctypes.data) if isinstance(a, np.ndarray) else C.c_void_p(a.data_ptr())
                for a in out]
        while len(ptrs) < 3:
            ptrs.append(C.c_void_p(0))
        _load().vg_render(self.h, first, count, ptrs[0], ptrs[1], ptrs[2])
        return out

    def pose(self, i: int) -> np.ndarray:
        o = np.zeros(4, np.float64)
        _load().vg_pose(self.h, i, C.c_void_p(o.ctypes.data))
        return o
