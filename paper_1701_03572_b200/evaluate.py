"""Evaluation of a stabilized stream: the reference's
synth_eval.cpp:214-349 (interframe_psnr, reestimate_deltas, score) on the GPU.

- Inter-frame PSNR: the exact integer sum of squared differences comes from
  the device (stabgpu_interframe_sse); mse and 10*log10(255^2/mse) are formed
  on the host exactly as psnr_pair does, so the values are bit-identical.
- Re-estimated deltas: Stage I motion with the reference's default detector and
  flow configs, similarity model, no RANSAC (Tracker::advance +
  estimate_similarity + extract_delta, synth_eval.cpp:243-263).
- Jitter energy: the population std of each delta component over frames 1..n-1
  (delta_std / std_of), computed in the reference's summation order.

Inputs are (n, h, w) uint8 luma arrays (numpy or torch CUDA tensors)."""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from ._abi import FORCE_SIMILARITY
from ._lib import check, context, load
from .stab import DetectConfig, FlowConfig, SelectorConfig, StabConfig


def _dev(y):
    import torch

    if isinstance(y, np.ndarray):
        return torch.from_numpy(np.ascontiguousarray(y, np.uint8)).cuda()
    return y.contiguous()


def interframe_psnr(y, crop_ratio: float = 0.0, device: int = 0) -> list[float]:
    """psnr_pair(frames[i-1], frames[i]) for i = 1 .. n-1 (synth_eval.cpp:242-252)."""
    d = _dev(y)
    n, h, w = d.shape
    sse = np.zeros(max(n - 1, 1), np.uint64)
    cnt = C.c_int64()
    check(load().stabgpu_interframe_sse(context(device).handle, C.c_void_p(d.data_ptr()), n, w, h, crop_ratio,
                                        C.c_void_p(sse.ctypes.data), C.byref(cnt)))
    out = []
    for k in range(n - 1):
        mse = float(int(sse[k])) / float(cnt.value)  # the reference's double acc is exact here
        out.append(math.inf if mse == 0.0 else 10.0 * math.log10(255.0 * 255.0 / mse))
    return out


def reestimate_config() -> StabConfig:
    """The shared estimator of reestimate_deltas: default DetectConfig and
    FlowConfig, similarity fits without RANSAC."""
    return StabConfig(detect=DetectConfig(), flow=FlowConfig(),
                      selector=SelectorConfig(mode=FORCE_SIMILARITY))


def reestimate_deltas(y, device: int = 0) -> np.ndarray:
    """Per-frame deltas re-estimated from pixels (synth_eval.cpp:254-272)."""
    from .pipeline import stabilize_sequence_device

    d = _dev(y)
    _, _, _, rec = stabilize_sequence_device(d, reestimate_config(), device=device)
    return rec["delta"]


def _mean(v):
    acc = 0.0
    for x in v:
        acc += x
    return acc / len(v)


def _std(v):  # std_of, synth_eval.cpp:74-80
    if len(v) < 2:
        return 0.0
    m = _mean(v)
    acc = 0.0
    for x in v:
        acc += (x - m) * (x - m)
    return math.sqrt(acc / len(v))


def _delta_std(d):
    return tuple(_std([float(d[k][i]) for i in range(1, len(d))]) for k in ("dx", "dy", "da", "dls"))


def _mean_finite(v):
    acc, n = 0.0, 0
    for x in v:
        if math.isfinite(x):
            acc += x
            n += 1
    return acc / n if n else math.inf


@dataclass
class EvalReport:  # synth_eval.hpp:74-82
    mean_psnr_before: float = 0.0
    mean_psnr_after: float = 0.0
    jitter_energy_before: tuple = (0.0, 0.0, 0.0, 0.0)
    jitter_energy_after: tuple = (0.0, 0.0, 0.0, 0.0)
    truth_recovery_rmse: tuple = (0.0, 0.0, 0.0, 0.0)
    has_truth: bool = False
    frames_skipped: int = 0
    extra: dict = field(default_factory=dict)


def score(original, stabilized, truth=None, estimated=None, crop_ratio: float = 0.0,
          device: int = 0) -> EvalReport:
    """score(), synth_eval.cpp:303-349.  truth / estimated are delta arrays
    (pipeline.DELTA_DT) or None."""
    if len(original) != len(stabilized):
        raise ValueError("original and stabilized streams differ in length")
    r = EvalReport()
    r.mean_psnr_before = _mean_finite(interframe_psnr(original, crop_ratio, device))
    r.mean_psnr_after = _mean_finite(interframe_psnr(stabilized, crop_ratio, device))
    r.jitter_energy_before = _delta_std(reestimate_deltas(original, device))
    r.jitter_energy_after = _delta_std(reestimate_deltas(stabilized, device))
    if estimated is not None:
        r.frames_skipped = int(sum(1 for d in estimated if d["skipped"]))
    if truth is not None and estimated is not None and len(truth) and len(estimated):
        r.has_truth = True
        s = [0.0, 0.0, 0.0, 0.0]
        n = 0
        for i in range(1, len(truth)):
            if estimated[i]["skipped"]:
                continue
            for j, k in enumerate(("dx", "dy", "da", "dls")):
                e = float(estimated[i][k]) - float(truth[i][k])
                s[j] += e * e
            n += 1
        if n:
            r.truth_recovery_rmse = tuple(math.sqrt(x / n) for x in s)
    return r


def rgb_to_ycbcr(rgb, device: int = 0):
    """(n, h, w, 3) uint8 RGB (device or host) -> Y, Cb, Cr device planes."""
    import torch

    d = _dev(rgb)
    n, h, w, _ = d.shape
    y, cb, cr = (torch.empty((n, h, w), dtype=torch.uint8, device=d.device) for _ in range(3))
    check(load().stabgpu_rgb_to_ycbcr(context(device).handle, C.c_void_p(d.data_ptr()), n, w, h,
                                      C.c_void_p(y.data_ptr()), C.c_void_p(cb.data_ptr()), C.c_void_p(cr.data_ptr())))
    return y, cb, cr


def ycbcr_to_rgb(y, cb, cr, device: int = 0):
    import torch

    y, cb, cr = _dev(y), _dev(cb), _dev(cr)
    n, h, w = y.shape
    out = torch.empty((n, h, w, 3), dtype=torch.uint8, device=y.device)
    check(load().stabgpu_ycbcr_to_rgb(context(device).handle, C.c_void_p(y.data_ptr()), C.c_void_p(cb.data_ptr()),
                                      C.c_void_p(cr.data_ptr()), n, w, h, C.c_void_p(out.data_ptr())))
    return out
