"""B200-native (sm_100a) hot path of the arXiv 1701.03572 optical-flow video
stabilizer: Shi-Tomasi corners, Gaussian pyramid, pyramidal LK with
forward-backward weeding, RANSAC rigid/similarity fit, trajectory smoothing
and warp + crop composition, behind the C ABI in include/stabgpu.h.

``stab`` mirrors the reference stage API (namespace stab); ``pipeline``
holds the whole-sequence (Stage I) driver and the multi-GPU sharding.
"""
from . import stab  # noqa: F401

__all__ = ["stab"]
