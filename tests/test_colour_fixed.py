"""The fixed-point BT.601 rule of csrc/colour.cuh against the reference's fp64
formulas (media_io.cpp:75-89, 568-570) on every one of the 2^24 inputs of
each conversion.  numpy float64 ops are correctly rounded IEEE operations in
the reference's order (no fma), i.e. what the reference computes; the numpy
formulas are in turn pinned to the reference's own functions by
test_oracle_pin.py::test_colour_conversions_exhaustive (through the C
restatement) — checked here against the oracle as well."""
import re
from pathlib import Path

import numpy as np

from . import _oracle

CUH = Path(__file__).resolve().parents[1] / "paper_1701_03572_b200" / "csrc" / "colour.cuh"


def _consts():
    src = CUH.read_text()
    get = lambda n: int(re.search(rf"constexpr int {n} = (0x[0-9a-f]+);", src).group(1), 16)
    fb = int(re.search(r"constexpr int FB = (\d+);", src).group(1))
    tie = int(re.search(r"constexpr unsigned TIE = (\d+);", src).group(1))
    return fb, tie, get


def _lround_clamp(s):
    r = np.where(s >= 0, np.floor(s + 0.5), np.ceil(s - 0.5))  # std::lround: half away from zero
    return np.clip(r, 0, 255).astype(np.int64)


def _fx(v, fb, tie):
    """(byte, near) of a fixed-point value, as fx_byte."""
    s = 1 << fb
    near = ((v + tie) & (s - 1)) <= 2 * tie
    return np.clip(v >> fb, 0, 255), near


def test_coefficients_are_rounded_products():
    fb, _, get = _consts()
    for name, c in [("K_R_V", 1.402), ("K_G_U", 0.344136), ("K_G_V", 0.714136), ("K_B_U", 1.772),
                    ("K_CB_R", 0.168736), ("K_CB_G", 0.331264), ("K_CR_G", 0.418688), ("K_CR_B", 0.081312)]:
        assert get(name) == int(round(c * (1 << fb))), name


def test_ycc_to_rgb_rule_exhaustive():
    fb, tie, get = _consts()
    v = np.arange(256, dtype=np.float64)
    y, cb, cr = v[:, None, None], v[None, :, None], v[None, None, :]
    du, dv = cb - 128.0, cr - 128.0
    ref = [_lround_clamp(y + 1.402 * dv), _lround_clamp((y - 0.344136 * du) - 0.714136 * dv),
           _lround_clamp(y + 1.772 * du)]
    i = np.arange(256, dtype=np.int64)
    yv = (i[:, None, None] << fb) + (1 << (fb - 1))
    ku, kv = (i - 128)[None, :, None], (i - 128)[None, None, :]
    r, n1 = _fx(yv + kv * get("K_R_V"), fb, tie)
    g, n2 = _fx(yv - ku * get("K_G_U") - kv * get("K_G_V"), fb, tie)
    b, n3 = _fx(yv + ku * get("K_B_U"), fb, tie)
    near = n1 | n2 | n3
    for fast, want in zip((r, g, b), ref):
        assert int(((fast != want) & ~near).sum()) == 0
    assert near.mean() < 1e-2  # the fp64 fallback is rare (B: the exact ties 1.772*du = k + 1/2)
    # int32 range of every intermediate
    for t in (yv + kv * get("K_R_V"), yv - ku * get("K_G_U") - kv * get("K_G_V"), yv + ku * get("K_B_U")):
        assert np.abs(t).max() < 2 ** 31


def test_rgb_to_ycc_rule_exhaustive():
    fb, tie, get = _consts()
    v = np.arange(256, dtype=np.float64)
    r, g, b = v[:, None, None], v[None, :, None], v[None, None, :]
    ref_cb = _lround_clamp(((128.0 - 0.168736 * r) - 0.331264 * g) + 0.5 * b)
    ref_cr = _lround_clamp(((128.0 + 0.5 * r) - 0.418688 * g) - 0.081312 * b)
    i = np.arange(256, dtype=np.int64)
    base = (128 << fb) + (1 << (fb - 1))
    tcb = base - i[:, None, None] * get("K_CB_R") - i[None, :, None] * get("K_CB_G") + (i[None, None, :] << (fb - 1))
    tcr = base + (i[:, None, None] << (fb - 1)) - i[None, :, None] * get("K_CR_G") - i[None, None, :] * get("K_CR_B")
    cb, n1 = _fx(tcb, fb, tie)
    cr, n2 = _fx(tcr, fb, tie)
    near = n1 | n2
    assert int(((cb != ref_cb) & ~near).sum()) == 0
    assert int(((cr != ref_cr) & ~near).sum()) == 0
    assert near.mean() < 5e-3
    assert max(np.abs(tcb).max(), np.abs(tcr).max()) < 2 ** 31


def test_numpy_formulas_match_the_oracle():
    """The fp64 numpy formulas above are the reference's: compared with the C
    restatement (pinned to the reference's media_io.cpp) on all triples."""
    o_rgb2ycc, o_ycc2rgb, _ = _oracle.colour_and_psnr(_oracle.ORACLE, "orc_")
    t = np.arange(1 << 24, dtype=np.uint32)
    trip = np.stack([(t >> 16) & 255, (t >> 8) & 255, t & 255], -1).astype(np.uint8)
    y, cb, cr = o_rgb2ycc(trip)
    v = trip.astype(np.float64)
    assert np.array_equal(cb, _lround_clamp(((128.0 - 0.168736 * v[:, 0]) - 0.331264 * v[:, 1]) + 0.5 * v[:, 2]))
    assert np.array_equal(cr, _lround_clamp(((128.0 + 0.5 * v[:, 0]) - 0.418688 * v[:, 1]) - 0.081312 * v[:, 2]))
    rgb = o_ycc2rgb(trip[:, 0], trip[:, 1], trip[:, 2])
    du, dv = v[:, 1] - 128.0, v[:, 2] - 128.0
    assert np.array_equal(rgb[:, 0], _lround_clamp(v[:, 0] + 1.402 * dv))
    assert np.array_equal(rgb[:, 1], _lround_clamp((v[:, 0] - 0.344136 * du) - 0.714136 * dv))
    assert np.array_equal(rgb[:, 2], _lround_clamp(v[:, 0] + 1.772 * du))
