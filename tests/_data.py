"""Seeded test inputs (small sizes the CPU checkers finish in seconds)."""
from __future__ import annotations

import numpy as np

from paper_1701_03572_b200.stab import (FORCE_RIGID, FORCE_SIMILARITY, HYBRID, DetectConfig,
                                        FlowConfig, RansacConfig, SelectorConfig, StabConfig)
from paper_1701_03572_b200.synth import Video, VideoSpec


def video(w=192, h=144, frames=24, objects=0, color=False, seed=7, jit_t=2.0, jit_rot=0.5,
          jit_scale=0.005, tex=256, blobs=60):
    spec = VideoSpec(w, h, frames, tex, blobs, objects, color, 0.5, jit_t, jit_rot, jit_scale, 2.0,
                     0x5EED1000 + seed)
    return Video(spec).render()


def small_cfg(mode=FORCE_SIMILARITY, ransac=0, corners=60, min_dist=8.0, levels=3, radius=10,
              smooth=5):
    return StabConfig(
        detect=DetectConfig(max_corners=corners, quality_level=0.01, min_distance=min_dist),
        flow=FlowConfig(window_radius=radius, max_levels=levels),
        smooth_radius=smooth,
        selector=SelectorConfig(mode=mode),
        ransac=RansacConfig(iterations=ransac, threshold=3.0, seed=99),
        crop_ratio=0.04,
        queue_capacity=64,
    )


def noise_frame(w, h, seed, smooth=True):
    rng = np.random.default_rng(seed)
    a = rng.integers(0, 256, size=(h, w)).astype(np.float64)
    if smooth:  # cheap separable box blur -> corner-rich but not white noise
        k = np.ones(5) / 5
        a = np.apply_along_axis(lambda r: np.convolve(r, k, "same"), 1, a)
        a = np.apply_along_axis(lambda c: np.convolve(c, k, "same"), 0, a)
        a = (a - a.mean()) * 3 + 128
    return np.ascontiguousarray(np.clip(np.rint(a), 0, 255).astype(np.uint8))


def integer_shift(f, dx, dy):
    """out(x, y) = f(x - dx, y - dy) with edge replication."""
    h, w = f.shape
    ys = np.clip(np.arange(h) - dy, 0, h - 1)
    xs = np.clip(np.arange(w) - dx, 0, w - 1)
    return f[ys][:, xs].copy()


MODES = {"hybrid": HYBRID, "rigid": FORCE_RIGID, "similarity": FORCE_SIMILARITY}
