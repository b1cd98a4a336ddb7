"""Pins for oracle/attention.py against things other than itself (CPU only).

Pins: hand-derived golden fixtures (tests/golden/attention_hand.json), a library routine
(torch scaled_dot_product_attention / logsumexp in fp64), brute-force pure-Python loops,
and closed-form invariants of attention (single key, identical keys, one-hot dominance,
permutation, key shift, V-affine, window limits, split merge).
"""
import json
import math
import os

import numpy as np
import pytest
import torch

from oracle.attention import decode_attention, decode_attention_keys, merge_partials

GOLD = os.path.join(os.path.dirname(__file__), "golden", "attention_hand.json")


def _f(x):
    return -np.inf if x == "-inf" else x


def _rand(rng, n, hq, hkv, d):
    return rng.standard_normal((hq, d)), rng.standard_normal((n, hkv, d)), rng.standard_normal((n, hkv, d))


@pytest.mark.parametrize("case", json.load(open(GOLD))["cases"], ids=lambda c: c["name"])
def test_golden_hand_cases(case):
    O, LSE = decode_attention(np.array(case["q"]), np.array(case["K"]), np.array(case["V"]),
                              case["scale"], case["window"])
    np.testing.assert_allclose(O, np.array(case["O"]), rtol=0, atol=1e-14)
    np.testing.assert_allclose(LSE, np.array(case["LSE"]), rtol=0, atol=1e-14)


@pytest.mark.parametrize("case", json.load(open(GOLD))["merge_cases"], ids=lambda c: c["name"])
def test_golden_merge_cases(case):
    lse_in = np.array([_f(x) for x in case["part_lse"]], dtype=np.float64)
    O, LSE = merge_partials(np.array(case["part_o"]), lse_in)
    np.testing.assert_allclose(O, np.array(case["O"]), rtol=0, atol=1e-14)
    want = _f(case["LSE"])
    if want == -np.inf:
        assert LSE == -np.inf
    else:
        assert abs(LSE - want) < 1e-14


@pytest.mark.parametrize("seed", range(12))
def test_matches_torch_sdpa_fp64(seed):
    """Library routine: torch SDPA (fp64, CPU) with K/V repeat_interleaved G times."""
    rng = np.random.default_rng(seed)
    hkv = int(rng.choice([1, 2, 4]))
    g = int(rng.choice([1, 2, 3, 5]))
    hq, d, n = hkv * g, int(rng.choice([4, 16, 64])), int(rng.integers(1, 65))
    window = int(rng.choice([0, 0, 1, 3, 17, 100]))
    scale = float(rng.uniform(0.05, 0.7))
    q, K, V = _rand(rng, n, hq, hkv, d)
    O, LSE = decode_attention(q, K, V, scale, window)

    tq = torch.from_numpy(q)[:, None, :]                                   # [Hq, 1, d]
    tk = torch.from_numpy(K).permute(1, 0, 2).repeat_interleave(g, dim=0)  # [Hq, n, d]
    tv = torch.from_numpy(V).permute(1, 0, 2).repeat_interleave(g, dim=0)
    lo = max(0, n - window) if window > 0 else 0
    mask = torch.zeros(1, n, dtype=torch.bool)
    mask[:, lo:] = True
    ref = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv, attn_mask=mask, scale=scale)
    logits = (tq @ tk.transpose(1, 2))[:, 0, :] * scale
    ref_lse = torch.logsumexp(logits[:, lo:], dim=-1)
    np.testing.assert_allclose(O, ref[:, 0, :].numpy(), rtol=0, atol=1e-12)
    np.testing.assert_allclose(LSE, ref_lse.numpy(), rtol=0, atol=1e-12)


def _brute(q, K, V, scale, window):
    """Per-head pure-Python loops (math.exp), the textbook definition, tiny sizes only."""
    hq, d = len(q), len(q[0])
    n, hkv = len(K), len(K[0])
    G = hq // hkv
    lo = max(0, n - window) if window > 0 else 0
    O = [[0.0] * d for _ in range(hq)]
    L = [0.0] * hq
    for h in range(hq):
        g = h // G
        z = [scale * sum(q[h][c] * K[j][g][c] for c in range(d)) for j in range(lo, n)]
        m = max(z)
        s = sum(math.exp(x - m) for x in z)
        L[h] = m + math.log(s)
        for jj, j in enumerate(range(lo, n)):
            w = math.exp(z[jj] - L[h])
            for c in range(d):
                O[h][c] += w * V[j][g][c]
    return np.array(O), np.array(L)


@pytest.mark.parametrize("hq,hkv", [(4, 4), (4, 1), (6, 2), (1, 1)])
@pytest.mark.parametrize("window", [0, 2])
def test_gqa_reductions_brute_force(hq, hkv, window):
    """MHA (Hkv = Hq), MQA (Hkv = 1) and GQA agree with per-head textbook loops."""
    rng = np.random.default_rng(hq * 10 + hkv + window)
    q, K, V = _rand(rng, 7, hq, hkv, 5)
    O, LSE = decode_attention(q, K, V, 0.4, window)
    Ob, Lb = _brute(q.tolist(), K.tolist(), V.tolist(), 0.4, window)
    np.testing.assert_allclose(O, Ob, rtol=0, atol=1e-13)
    np.testing.assert_allclose(LSE, Lb, rtol=0, atol=1e-13)


def test_single_key_returns_its_value():
    rng = np.random.default_rng(1)
    q, K, V = _rand(rng, 1, 6, 3, 16)
    O, LSE = decode_attention(q, K, V, 0.25, 0)
    G = 2
    for h in range(6):
        assert np.array_equal(O[h], V[0, h // G])           # weight exp(0) = 1 exactly
        assert abs(LSE[h] - 0.25 * q[h] @ K[0, h // G]) < 1e-15


def test_identical_keys_give_mean_of_values():
    rng = np.random.default_rng(2)
    n = 37
    q, K, V = _rand(rng, n, 4, 2, 8)
    K[:] = K[0]
    O, LSE = decode_attention(q, K, V, 0.3, 0)
    for h in range(4):
        np.testing.assert_allclose(O[h], V[:, h // 2].mean(axis=0), rtol=0, atol=1e-13)
        assert abs(LSE[h] - (0.3 * q[h] @ K[0, h // 2] + math.log(n))) < 1e-12


def test_one_hot_dominance():
    rng = np.random.default_rng(3)
    n = 50
    q, K, V = _rand(rng, n, 2, 1, 8)
    j = 17
    K[j, 0] = 60.0 * q[0] / np.linalg.norm(q[0])
    O, _ = decode_attention(q[:1], K, V, 1.0, 0)
    z = K[:, 0] @ q[0]
    gap = z[j] - np.delete(z, j).max()
    assert gap > 40
    np.testing.assert_allclose(O[0], V[j, 0], rtol=0, atol=n * math.exp(-gap) * np.abs(V).max() * 2)


def test_permutation_invariance():
    rng = np.random.default_rng(4)
    q, K, V = _rand(rng, 29, 4, 2, 16)
    perm = rng.permutation(29)
    O1, L1 = decode_attention(q, K, V, 0.2, 0)
    O2, L2 = decode_attention(q, K[perm], V[perm], 0.2, 0)
    np.testing.assert_allclose(O1, O2, rtol=0, atol=1e-13)
    np.testing.assert_allclose(L1, L2, rtol=0, atol=1e-13)


def test_key_shift():
    """k_j -> k_j + u for all j: O unchanged, LSE += scale * q.u (softmax shift invariance)."""
    rng = np.random.default_rng(5)
    q, K, V = _rand(rng, 23, 3, 1, 16)
    u = rng.standard_normal(16)
    O1, L1 = decode_attention(q, K, V, 0.3, 0)
    O2, L2 = decode_attention(q, K + u, V, 0.3, 0)
    np.testing.assert_allclose(O1, O2, rtol=0, atol=1e-12)
    np.testing.assert_allclose(L2, L1 + 0.3 * q @ u, rtol=0, atol=1e-12)


def test_v_affine():
    """V -> V A + b: O -> O A + b, because the weights sum to one."""
    rng = np.random.default_rng(6)
    q, K, V = _rand(rng, 19, 4, 2, 8)
    A = rng.standard_normal((8, 8))
    b = rng.standard_normal(8)
    O1, _ = decode_attention(q, K, V, 0.3, 0)
    O2, _ = decode_attention(q, K, V @ A + b, 0.3, 0)
    np.testing.assert_allclose(O2, O1 @ A + b, rtol=0, atol=1e-12)


def test_window_limits():
    rng = np.random.default_rng(7)
    n = 40
    q, K, V = _rand(rng, n, 4, 2, 8)
    full = decode_attention(q, K, V, 0.3, 0)
    for W in (n, n + 5, 10_000):
        w = decode_attention(q, K, V, 0.3, W)
        np.testing.assert_array_equal(full[0], w[0])
    O1, L1 = decode_attention(q, K, V, 0.3, 1)
    for h in range(4):
        assert np.array_equal(O1[h], V[n - 1, h // 2])
        assert abs(L1[h] - 0.3 * q[h] @ K[n - 1, h // 2]) < 1e-15
    W = 9
    Ow, Lw = decode_attention(q, K, V, 0.3, W)
    Ok, Lk = decode_attention_keys(q, K, V, 0.3, range(n - W, n))
    np.testing.assert_allclose(Ow, Ok, rtol=0, atol=1e-14)
    np.testing.assert_allclose(Lw, Lk, rtol=0, atol=1e-14)


@pytest.mark.parametrize("seed", range(6))
def test_split_merge_equals_unsplit(seed):
    """merge(split(x)) == unsplit(x) for random split points, empty splits included."""
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(1, 80))
    q, K, V = _rand(rng, n, 6, 3, 16)
    q *= 3.0
    O, LSE = decode_attention(q, K, V, 0.5, 0)
    cuts = sorted(rng.integers(0, n + 1, size=int(rng.integers(1, 6))).tolist())
    bounds = [0] + cuts + [n]
    parts = [decode_attention_keys(q, K, V, 0.5, range(a, b)) for a, b in zip(bounds[:-1], bounds[1:])]
    for h in range(6):
        o, l = merge_partials(np.stack([p[0][h] for p in parts]), np.array([p[1][h] for p in parts]))
        np.testing.assert_allclose(o, O[h], rtol=0, atol=1e-12)
        assert abs(l - LSE[h]) < 1e-12


def test_empty_request_rejected():
    with pytest.raises(ValueError):
        decode_attention(np.zeros((2, 4)), np.zeros((0, 1, 4)), np.zeros((0, 1, 4)), 1.0)
