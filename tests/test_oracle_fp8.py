"""Pins of the e4m3 quantiser oracle (oracle/fp8.py) against the format's definition, exact
round trips, tie and saturation cases, brute force and torch's float8_e4m3fn conversion."""
import numpy as np
import torch

from oracle.fp8 import E4M3_MAX, dequantize_e4m3, e4m3_value, quantize_e4m3, quantize_kv


def test_known_codes():
    assert e4m3_value(0x38) == 1.0
    assert e4m3_value(0x7E) == 448.0 == E4M3_MAX
    assert e4m3_value(0x01) == 2.0 ** -9            # smallest subnormal
    assert e4m3_value(0x08) == 2.0 ** -6            # smallest normal
    assert e4m3_value(0x07) == 7 / 8 * 2.0 ** -6    # largest subnormal
    assert e4m3_value(0xB8) == -1.0
    assert np.isnan(e4m3_value(0x7F)) and np.isnan(e4m3_value(0xFF))
    assert e4m3_value(0x80) == 0.0 and np.signbit(e4m3_value(0x80))


def test_every_finite_code_round_trips():
    codes = np.array([c for c in range(256) if c not in (0x7F, 0xFF)], dtype=np.uint8)
    vals = np.array([e4m3_value(c) for c in codes], dtype=np.float32)
    assert np.array_equal(quantize_e4m3(vals), codes)


def test_ties_go_to_even_and_neighbours_to_nearest():
    pos = [c for c in range(0x7F)]
    for c in pos[:-1]:
        a, b = e4m3_value(c), e4m3_value(c + 1)
        mid = np.float32((a + b) / 2)
        assert float(mid) == (a + b) / 2          # every midpoint is an fp32 number
        even = c if c % 2 == 0 else c + 1
        assert quantize_e4m3(np.array([mid]))[0] == even
        assert quantize_e4m3(np.array([-mid]))[0] == even | 0x80
        up = np.nextafter(mid, np.float32(np.inf))
        dn = np.nextafter(mid, np.float32(-np.inf))
        assert quantize_e4m3(np.array([up]))[0] == c + 1
        assert quantize_e4m3(np.array([dn]))[0] == c


def test_saturation_and_signed_zero():
    x = np.array([449.0, 464.0, 1e6, -1e6, 3.0e38, -0.0, -1e-30, 1e-30], dtype=np.float32)
    assert quantize_e4m3(x).tolist() == [0x7E, 0x7E, 0x7E, 0xFE, 0x7E, 0x80, 0x80, 0x00]


def test_brute_force_nearest():
    rng = np.random.default_rng(7)
    x = (rng.standard_normal(4000) * np.exp(rng.uniform(-9, 6, 4000))).astype(np.float32)
    x = x[np.abs(x) <= E4M3_MAX]
    codes = quantize_e4m3(x)
    allv = np.array([e4m3_value(c) for c in range(256)])
    finite = ~np.isnan(allv)
    for xi, ci in zip(x.astype(np.float64), codes):
        d = np.abs(allv[finite] - xi)
        assert abs(e4m3_value(ci) - xi) == d.min()


def test_matches_torch_float8_e4m3fn_in_range():
    rng = np.random.default_rng(8)
    x = (rng.standard_normal(20000) * np.exp(rng.uniform(-10, 6, 20000))).astype(np.float32)
    x = np.clip(x, -E4M3_MAX, E4M3_MAX)
    ref = torch.from_numpy(x).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    assert np.array_equal(quantize_e4m3(x), ref)


def test_quantize_kv_divides_in_fp32_and_dequantizes_exactly():
    x = np.array([0.3, -1.7, 2.5, 7.9], dtype=np.float32)
    s = np.float32(8.0 / 448.0)
    codes = quantize_kv(x, s)
    assert np.array_equal(codes, quantize_e4m3((x / s).astype(np.float32)))
    back = dequantize_e4m3(codes, s)
    assert np.all(np.abs(back - x) <= np.abs(x) * 2.0 ** -4 + 1e-12)   # half an ulp of 3 mantissa bits
