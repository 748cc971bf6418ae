"""ctypes mirror of include/stabgpu.h (struct layouts and prototypes).

Only layouts and signatures live here; libstabgpu.so is loaded by
``_lib.load()``.  The same structs describe the C oracle's entry points,
which the tests load separately (oracle/stab_oracle.h shares this ABI).
"""
from __future__ import annotations

import ctypes as C

c_u8p = C.POINTER(C.c_uint8)
c_dp = C.POINTER(C.c_double)
c_ip = C.POINTER(C.c_int)

STABGPU_MAX_LEVELS = 16

OK, INVALID_INPUT, INVALID_CONFIG, INVALID_TRANSFORM, DEGENERATE_INPUT, SEQUENCING, IO, CUDA = range(8)
HYBRID, FORCE_RIGID, FORCE_SIMILARITY = range(3)
RIGID, SIMILARITY = 0, 1
FRAME_FIRST, FRAME_SKIPPED, FRAME_TRACKED = range(3)


class DetectCfg(C.Structure):  # DetectConfig, features.hpp:15-21
    _fields_ = [("max_corners", C.c_int), ("quality_level", C.c_double),
                ("min_distance", C.c_double), ("block_size", C.c_int), ("roi_margin", C.c_double)]


class FlowCfg(C.Structure):  # FlowConfig, flow.hpp:13-21
    _fields_ = [("window_radius", C.c_int), ("max_levels", C.c_int), ("max_iterations", C.c_int),
                ("epsilon", C.c_double), ("fb_threshold", C.c_double),
                ("redetect_interval", C.c_int), ("min_tracks", C.c_int)]


class RansacCfg(C.Structure):
    _fields_ = [("iterations", C.c_int), ("threshold", C.c_double), ("seed", C.c_uint64)]


class SelectorCfg(C.Structure):  # SelectorConfig, motion.hpp:29-33
    _fields_ = [("dwell", C.c_int), ("margin", C.c_double), ("mode", C.c_int)]


class Config(C.Structure):  # StabConfig, pipeline.hpp:15-22
    _fields_ = [("detect", DetectCfg), ("flow", FlowCfg), ("smooth_radius", C.c_int),
                ("selector", SelectorCfg), ("ransac", RansacCfg), ("crop_ratio", C.c_double),
                ("queue_capacity", C.c_size_t)]


class Transform(C.Structure):  # SimilarityTransform, transform.hpp:13-32
    _fields_ = [("tx", C.c_double), ("ty", C.c_double), ("theta", C.c_double), ("s", C.c_double),
                ("kind", C.c_int)]


class Delta(C.Structure):  # DeltaParams, transform.hpp:42-49
    _fields_ = [("dx", C.c_double), ("dy", C.c_double), ("da", C.c_double), ("dls", C.c_double),
                ("kind", C.c_int), ("skipped", C.c_int)]


class Roi(C.Structure):  # RoiRect, features.hpp:27-36
    _fields_ = [("x0", C.c_int), ("y0", C.c_int), ("x1", C.c_int), ("y1", C.c_int)]


class Pyramid(C.Structure):  # Pyramid, frame.hpp:43-49
    _fields_ = [("levels", C.c_int), ("width", C.c_int * STABGPU_MAX_LEVELS),
                ("height", C.c_int * STABGPU_MAX_LEVELS),
                ("offset", C.c_size_t * STABGPU_MAX_LEVELS), ("data", c_u8p)]


class FrameRecord(C.Structure):
    _fields_ = [("delta", Delta), ("correction", Transform), ("frame_kind", C.c_int),
                ("n_tracks", C.c_int), ("n_inliers", C.c_int), ("decision", C.c_int)]


class MotionRecord(C.Structure):
    _fields_ = [("rigid", Delta), ("similarity", Delta), ("e_rigid", C.c_double),
                ("e_similarity", C.c_double), ("frame_kind", C.c_int), ("n_tracks", C.c_int),
                ("n_inliers_rigid", C.c_int), ("n_inliers_similarity", C.c_int),
                ("status", C.c_int), ("pad", C.c_int)]


class Stats(C.Structure):
    _fields_ = [("ms_pyramid", C.c_double), ("ms_detect", C.c_double), ("ms_track", C.c_double),
                ("ms_fit", C.c_double), ("ms_plan", C.c_double), ("ms_compose", C.c_double),
                ("ms_total", C.c_double), ("launches", C.c_longlong), ("lk_level_builds", C.c_longlong),
                ("lk_iterations", C.c_longlong)]


P = C.POINTER
V = C.c_void_p
I = C.c_int

# name -> (restype, argtypes): the entry points include/stabgpu.h declares
PROTOTYPES = {
    "stabgpu_last_error": (C.c_char_p, []),
    "stabgpu_version": (C.c_char_p, []),
    "stabgpu_default_config": (None, [P(Config)]),
    "stabgpu_validate_config": (I, [P(Config)]),
    "stabgpu_create": (I, [I, P(V)]),
    "stabgpu_destroy": (I, [V]),
    "stabgpu_set_stream": (I, [V, V]),
    "stabgpu_synchronize": (I, [V]),
    "stabgpu_pyramid_bytes": (C.c_size_t, [I, I, I]),
    "stabgpu_build_pyramid": (I, [V, V, I, I, I, P(Pyramid)]),
    "stabgpu_build_pyramid_batch": (I, [V, V, I, I, I, I, V]),
    "stabgpu_gradients": (I, [V, V, I, I, V, V]),
    "stabgpu_warp_similarity": (I, [V, V, I, I, P(Transform), V]),
    "stabgpu_crop_resize": (I, [V, V, I, I, C.c_double, V]),
    "stabgpu_compose_stabilized": (I, [V, V, V, V, I, I, I, I, P(Transform), C.c_double, V, V, V]),
    "stabgpu_detection_roi": (I, [I, I, C.c_double, P(Roi)]),
    "stabgpu_min_eig_response": (I, [V, V, I, I, I, V]),
    "stabgpu_detect_corners": (I, [V, V, I, I, P(DetectCfg), V, V, c_ip]),
    "stabgpu_detect_corners_batch": (I, [V, V, I, I, I, P(DetectCfg), V, V, c_ip]),
    "stabgpu_track_lk": (I, [V, P(Pyramid), P(Pyramid), V, I, P(FlowCfg), V, V]),
    "stabgpu_weed_tracks": (I, [V, P(Pyramid), P(Pyramid), V, V, I, P(FlowCfg), V, V, c_ip]),
    "stabgpu_estimate": (I, [V, V, V, I, I, P(Transform)]),
    "stabgpu_rms_residual": (I, [V, V, V, I, P(Transform), c_dp]),
    "stabgpu_ransac_estimate": (I, [V, V, V, I, I, P(RansacCfg), I, C.c_int64, P(Transform), V, c_ip]),
    "stabgpu_extract_delta": (None, [P(Transform), P(Delta)]),
    "stabgpu_delta_to_transform": (None, [C.c_double, C.c_double, C.c_double, C.c_double, P(Transform)]),
    "stabgpu_trajectory_corrections": (I, [V, V, I, I, V]),
    "stabgpu_stabilize_sequence": (I, [V, V, V, V, I, I, I, I, I, P(Config), V, V, V, V]),
    "stabgpu_stabilize_sequence_device": (I, [V, V, V, V, I, I, I, I, I, P(Config), V, V, V, V]),
    "stabgpu_stabilize_streams": (I, [V, V, V, V, I, I, I, I, I, I, P(Config), V, V, V, V]),
    "stabgpu_stabilize_streams_device": (I, [V, V, V, V, I, I, I, I, I, I, P(Config), V, V, V, V]),
    "stabgpu_motion_chunk": (I, [V, V, C.c_int64, I, I, I, P(Config), V]),
    "stabgpu_plan_corrections": (I, [V, V, I, P(Config), V]),
    "stabgpu_compose_frames": (I, [V, V, V, V, I, I, I, I, I, V, C.c_double, V, V, V]),
    "stabgpu_shard_range": (I, [C.c_int64, I, I, I, P(C.c_int64), c_ip, P(C.c_int64), P(C.c_int64)]),
    "stabgpu_nccl_unique_id": (I, [V]),
    "stabgpu_comm_init": (I, [V, V, I, I]),
    "stabgpu_stabilize_sharded": (I, [V, V, V, V, C.c_int64, I, I, I, I, P(Config), V, V, V, V]),
    "stabgpu_stabilize_sharded_device": (I, [V, V, V, V, C.c_int64, I, I, I, I, P(Config), V, V, V, V]),
    "stabgpu_shard_motion": (I, [V, V, V, V, C.c_int64, I, I, I, I, I, I, P(Config), V]),
    "stabgpu_shard_compose": (I, [V, V, C.c_int64, I, I, I, I, I, I, P(Config), V, V, V, V]),
    "stabgpu_tracker_create": (I, [V, P(FlowCfg), P(DetectCfg), I, I, P(V)]),
    "stabgpu_tracker_advance": (I, [V, V, C.c_int64, c_ip, V, V, c_ip, c_ip]),
    "stabgpu_tracker_points": (I, [V, c_ip]),
    "stabgpu_tracker_destroy": (I, [V]),
    "stabgpu_stream_create": (I, [V, P(Config), I, I, I, I, P(V)]),
    "stabgpu_stream_push": (I, [V, V, V, V, c_ip]),
    "stabgpu_stream_push_async": (I, [V, V, V, V, c_ip]),
    "stabgpu_stream_wait_inputs": (I, [V]),
    "stabgpu_host_alloc": (I, [C.POINTER(V), C.c_size_t]),
    "stabgpu_host_free": (I, [V]),
    "stabgpu_stream_finish": (I, [V, c_ip]),
    "stabgpu_stream_pop": (I, [V, P(C.c_int64), V, V, V, V]),
    "stabgpu_stream_pop_async": (I, [V, P(C.c_int64), V, V, V, V]),
    "stabgpu_stream_wait_pops": (I, [V]),
    "stabgpu_stream_destroy": (I, [V]),
    "stabgpu_stream_set_graphs": (I, [V, I]),
    "stabgpu_rgb_to_ycbcr": (I, [V, V, I, I, I, V, V, V]),
    "stabgpu_ycbcr_to_rgb": (I, [V, V, V, V, I, I, I, V]),
    "stabgpu_stabilize_sequence_rgb": (I, [V, V, I, I, I, P(Config), V, V]),
    "stabgpu_interframe_sse": (I, [V, V, I, I, I, C.c_double, V, P(C.c_int64)]),
    "stabgpu_get_stats": (I, [V, P(Stats)]),
    "stabgpu_debug_read_scratch": (I, [V, C.c_char_p, V, C.c_size_t, C.POINTER(C.c_size_t)]),
    "stabgpu_enable_timing": (I, [V, I]),
}


def bind(lib: C.CDLL, prototypes: dict, rename=lambda n: n) -> C.CDLL:
    for name, (res, args) in prototypes.items():
        fn = getattr(lib, rename(name))
        fn.restype = res
        fn.argtypes = args
    return lib
