"""Whole-sequence comparison of the GPU Stage I output with a CPU checker
(TEST INFRASTRUCTURE: used by tests/ and by bench.py's cpu_baseline leg).

north_star tolerances: transform parameters within 1e-3 (translation px,
rotation rad, scale relative), warped 8-bit pixels within +-1; the GPU is in
practice ~1e-9 on parameters and off by one on a handful of pixels (a value
that lands on the other side of an lround .5 tie when an upstream double
differs in its last bits).  The summary reports every count so a run at
config scale can be read off, not just pass/fail."""
from __future__ import annotations

import numpy as np

from paper_1701_03572_b200 import _abi

PARAM_TOL = 1e-3  # north_star
PIXEL_TOL = 1  # north_star


def _max_abs(a, b):
    if a.size == 0:
        return 0.0
    return float(np.abs(a.astype(np.float64) - b.astype(np.float64)).max())


def compare_records(g, o) -> dict:
    """Per-frame records (pipeline.RECORD_DT) -> summary dict."""
    g, o = g.reshape(-1), o.reshape(-1)
    tr = o["frame_kind"] == _abi.FRAME_TRACKED
    out = {
        "frames": int(len(o)),
        "tracked_frames": int(tr.sum()),
        "frame_kind_equal": bool(np.array_equal(g["frame_kind"], o["frame_kind"])),
        "n_tracks_equal": bool(np.array_equal(g["n_tracks"][tr], o["n_tracks"][tr])),
        "n_tracks_mismatch_frames": int((g["n_tracks"][tr] != o["n_tracks"][tr]).sum()),
        "n_inliers_equal": bool(np.array_equal(g["n_inliers"], o["n_inliers"])),
        "decision_equal": bool(np.array_equal(g["decision"], o["decision"])),
        "kind_equal": bool(np.array_equal(g["delta"]["kind"], o["delta"]["kind"])
                           and np.array_equal(g["delta"]["skipped"], o["delta"]["skipped"])),
    }
    out["max_delta_err"] = max(_max_abs(g["delta"][k], o["delta"][k]) for k in ("dx", "dy", "da", "dls"))
    out["max_correction_err"] = max(
        max(_max_abs(g["correction"][k], o["correction"][k]) for k in ("tx", "ty", "theta")),
        _max_abs(np.log(g["correction"]["s"]), np.log(o["correction"]["s"])))
    return out


def compare_planes(gs, os_) -> dict:
    """Lists of uint8 planes (None entries skipped) -> max |diff| and the
    count of differing pixels."""
    mx, cnt, tot = 0, 0, 0
    for a, b in zip(gs, os_):
        if a is None or b is None:
            continue
        a = np.asarray(a)
        b = np.asarray(b)
        # chunked: full-length 4K sequences are GBs
        flat_a, flat_b = a.reshape(-1), b.reshape(-1)
        step = 1 << 26
        for i in range(0, flat_a.size, step):
            d = np.abs(flat_a[i:i + step].astype(np.int16) - flat_b[i:i + step].astype(np.int16))
            mx = max(mx, int(d.max()) if d.size else 0)
            cnt += int(np.count_nonzero(d))
        tot += flat_a.size
    return {"pixels": int(tot), "max_pixel_diff": mx, "pixels_off": cnt,
            "pixels_off_frac": (cnt / tot) if tot else 0.0}


def summarize(g_rec, o_rec, g_planes, o_planes) -> dict:
    s = compare_records(g_rec, o_rec)
    s.update(compare_planes(g_planes, o_planes))
    s["ok"] = bool(s["frame_kind_equal"] and s["n_tracks_equal"] and s["n_inliers_equal"]
                   and s["decision_equal"] and s["kind_equal"] and s["max_delta_err"] <= PARAM_TOL
                   and s["max_correction_err"] <= PARAM_TOL and s["max_pixel_diff"] <= PIXEL_TOL)
    return s
