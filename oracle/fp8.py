"""FP8 (e4m3) KV quantisation, written from the format's definition (S8(f) F4).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

SURVEY.md Sec. 8(f) F4 names "FP8 (e4m3) KV pages with per-page scales (halves B_alg)" as
a variant of the decode step; the paper itself keeps the engine's KV precision implicit
(vLLM).  DESIGN.md reading F4-a: scales are static per (layer, KV head)
(k_scale, v_scale), supplied by the caller, because an append-only decode stream cannot
fix a page's scale before the page has filled.  So, for a bf16 value x of K (or V) of
layer l, head g:

    code = E4M3_RNE_SATFINITE( fp32(x) / fp32(scale[l, g]) )      (fp32 IEEE division)
    K    = scale[l, g] * value(code)                               (exact)

and the attention oracle (oracle/attention.py) runs on the dequantised K, V in fp64.

E4M3 ("fn" flavour): 1 sign, 4 exponent bits (bias 7), 3 mantissa bits; exponent field 0
is subnormal (value m/8 * 2^-6), fields 1..15 normal ((1 + m/8) * 2^(e-7)); the single
NaN pattern S.1111.111 has no infinity beside it, so the largest finite is 1.75 * 2^8 =
448.  Round to nearest, ties to the even code (mantissa LSB 0); SATFINITE clamps
magnitudes beyond 448 to 448 (the same decision the device's cvt.rn.satfinite makes, in
the same fp32 precision).
"""
from __future__ import annotations

import numpy as np

E4M3_MAX = 448.0


def e4m3_value(code: int) -> float:
    """The real value of one e4m3 code (NaN for the NaN patterns)."""
    code = int(code) & 0xFF
    s = -1.0 if code & 0x80 else 1.0
    e = (code >> 3) & 0xF
    m = code & 0x7
    if e == 0xF and m == 0x7:
        return float("nan")
    if e == 0:
        return s * (m / 8.0) * 2.0 ** -6
    return s * (1.0 + m / 8.0) * 2.0 ** (e - 7)


def _positive_table():
    """Finite non-negative codes 0x00..0x7E and their values, increasing."""
    codes = np.arange(0x7F, dtype=np.int64)
    vals = np.array([e4m3_value(c) for c in codes], dtype=np.float64)
    assert np.all(np.diff(vals) > 0)
    return codes, vals


_CODES, _VALS = _positive_table()


def quantize_e4m3(x: np.ndarray) -> np.ndarray:
    """Round fp32 values to e4m3 codes (uint8): nearest, ties to even, saturate at 448.

    Elementwise from the definition: find the two representable neighbours of |x| and pick
    the nearer; on an exact tie pick the one whose code (= mantissa LSB) is even."""
    x = np.asarray(x, dtype=np.float32).astype(np.float64)
    if np.isnan(x).any():
        raise ValueError("NaN inputs are undefined (reading #16)")
    a = np.minimum(np.abs(x), E4M3_MAX)
    hi = np.searchsorted(_VALS, a, side="left")          # first value >= a
    hi = np.minimum(hi, len(_VALS) - 1)
    lo = np.maximum(hi - 1, 0)
    d_hi = _VALS[hi] - a
    d_lo = a - _VALS[lo]
    exact = d_hi == 0
    pick_hi = exact | (d_hi < d_lo) | ((d_hi == d_lo) & (_CODES[hi] % 2 == 0))
    mag = np.where(pick_hi, _CODES[hi], _CODES[lo]).astype(np.uint8)
    neg = np.signbit(x)          # the sign survives rounding to zero (-0 -> 0x80), as in IEEE conversions
    return (mag | np.where(neg, 0x80, 0)).astype(np.uint8)


def dequantize_e4m3(codes: np.ndarray, scale) -> np.ndarray:
    """scale * value(code), fp64 (exact)."""
    lut = np.array([e4m3_value(c) for c in range(256)], dtype=np.float64)
    return lut[np.asarray(codes, dtype=np.uint8)] * np.asarray(scale, dtype=np.float64)


def quantize_kv(x_f32: np.ndarray, scale: np.ndarray) -> np.ndarray:
    """Codes of x / scale with the division in fp32 (IEEE, round to nearest), as defined
    above.  x_f32: fp32 values (bf16 inputs upcast exactly); scale broadcast against x."""
    q = np.asarray(x_f32, dtype=np.float32) / np.asarray(scale, dtype=np.float32)
    return quantize_e4m3(q.astype(np.float32))
