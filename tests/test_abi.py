"""The C-ABI library loads and exports every symbol include/stabgpu.h
declares (no compute calls: this runs without a GPU)."""
import ctypes
import os
import re

from paper_1701_03572_b200 import _abi, _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "stabgpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(stabgpu_[a-z_0-9]+)\s*\(", src)))


def test_header_symbols_exported():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = declared_symbols()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_python_prototypes_cover_header():
    assert set(declared_symbols()) == set(_abi.PROTOTYPES)


def test_struct_sizes():
    assert ctypes.sizeof(_abi.Transform) == 40
    assert ctypes.sizeof(_abi.Delta) == 40
    assert ctypes.sizeof(_abi.FrameRecord) == 96
    assert ctypes.sizeof(_abi.MotionRecord) == 120


def test_defaults_match_reference():
    lib = _lib.load()
    c = _abi.Config()
    lib.stabgpu_default_config(ctypes.byref(c))
    # features.hpp:16-20, flow.hpp:14-20, smoothing.hpp:12, motion.hpp:30-32, pipeline.hpp:20-21
    assert (c.detect.max_corners, c.detect.quality_level, c.detect.min_distance,
            c.detect.block_size, c.detect.roi_margin) == (50, 0.01, 10.0, 3, 0.1)
    assert (c.flow.window_radius, c.flow.max_levels, c.flow.max_iterations, c.flow.epsilon,
            c.flow.fb_threshold, c.flow.redetect_interval, c.flow.min_tracks) == (10, 4, 30, 0.01, 0.5, 5, 8)
    assert c.smooth_radius == 10 and (c.selector.dwell, c.selector.margin, c.selector.mode) == (20, 0.05, 0)
    assert c.crop_ratio == 0.04 and c.queue_capacity == 64
    assert lib.stabgpu_validate_config(ctypes.byref(c)) == 0
    c.queue_capacity = 20
    assert lib.stabgpu_validate_config(ctypes.byref(c)) == _abi.INVALID_CONFIG


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        return
    lib = _lib.load()
    h = ctypes.c_void_p()
    assert lib.stabgpu_create(0, ctypes.byref(h)) == _abi.CUDA
    assert b"no CPU fallback" in lib.stabgpu_last_error()
