"""Pins for oracle.attention.extend_attention (the F2 extend/prefill step) against things
other than itself (CPU only): torch SDPA in fp64 with an explicitly built causal +
sliding-window mask (HF semantics: key k is visible to query position p iff
p - W < k <= p), per-token brute force, the T = 1 reduction to decode attention, and
invariance of earlier tokens' outputs to later keys (causality)."""
import math

import numpy as np
import pytest
import torch

from oracle.attention import decode_attention, extend_attention


def _rand(rng, T, n, hq, hkv, d):
    return rng.standard_normal((T, hq, d)), rng.standard_normal((n, hkv, d)), rng.standard_normal((n, hkv, d))


@pytest.mark.parametrize("seed", range(10))
def test_matches_torch_sdpa_causal_window_fp64(seed):
    rng = np.random.default_rng(100 + seed)
    hkv = int(rng.choice([1, 2, 4]))
    g = int(rng.choice([1, 2, 5]))
    hq, d = hkv * g, int(rng.choice([8, 16, 64]))
    n = int(rng.integers(1, 60))
    T = int(rng.integers(1, n + 1))
    window = int(rng.choice([0, 0, 1, 4, 13, 100]))
    scale = float(rng.uniform(0.05, 0.5))
    Q, K, V = _rand(rng, T, n, hq, hkv, d)
    O, LSE = extend_attention(Q, K, V, scale, window)

    tq = torch.from_numpy(Q).permute(1, 0, 2)                               # [Hq, T, d]
    tk = torch.from_numpy(K).permute(1, 0, 2).repeat_interleave(g, dim=0)   # [Hq, n, d]
    tv = torch.from_numpy(V).permute(1, 0, 2).repeat_interleave(g, dim=0)
    pos = torch.arange(n - T, n)[:, None]                                   # query positions
    kidx = torch.arange(n)[None, :]
    mask = kidx <= pos
    if window > 0:
        mask &= kidx > pos - window
    ref = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv, attn_mask=mask, scale=scale)
    logits = (tq @ tk.transpose(1, 2)) * scale
    ref_lse = torch.logsumexp(logits.masked_fill(~mask, -math.inf), dim=-1)  # [Hq, T]
    np.testing.assert_allclose(O, ref.permute(1, 0, 2).numpy(), rtol=0, atol=1e-12)
    np.testing.assert_allclose(LSE, ref_lse.T.numpy(), rtol=0, atol=1e-12)


def test_brute_force_tiny():
    rng = np.random.default_rng(7)
    T, n, hq, hkv, d, scale = 3, 5, 2, 1, 3, 0.4
    Q, K, V = _rand(rng, T, n, hq, hkv, d)
    O, LSE = extend_attention(Q, K, V, scale)
    for t in range(T):
        p = n - T + t
        for h in range(hq):
            z = [scale * sum(Q[t, h, c] * K[j, 0, c] for c in range(d)) for j in range(p + 1)]
            m = max(z)
            lse = m + math.log(sum(math.exp(x - m) for x in z))
            o = [sum(math.exp(z[j] - lse) * V[j, 0, c] for j in range(p + 1)) for c in range(d)]
            assert abs(LSE[t, h] - lse) < 1e-12
            assert np.max(np.abs(O[t, h] - np.array(o))) < 1e-12


def test_single_token_is_decode():
    rng = np.random.default_rng(8)
    Q, K, V = _rand(rng, 1, 9, 4, 2, 8)
    for w in (0, 3):
        O, L = extend_attention(Q, K, V, 0.3, w)
        Od, Ld = decode_attention(Q[0], K, V, 0.3, w)
        assert np.array_equal(O[0], Od) and np.array_equal(L[0], Ld)


def test_causal_later_keys_do_not_matter():
    rng = np.random.default_rng(9)
    Q, K, V = _rand(rng, 4, 10, 2, 2, 8)
    O, L = extend_attention(Q, K, V, 0.3)
    K2, V2 = K.copy(), V.copy()
    K2[-1] += 5.0                                 # the last token's key and value
    V2[-1] -= 3.0
    O2, L2 = extend_attention(Q, K2, V2, 0.3)
    np.testing.assert_array_equal(O[:3], O2[:3])  # only the last query sees them
    np.testing.assert_array_equal(L[:3], L2[:3])
    assert np.abs(O[3] - O2[3]).max() > 1e-3


def test_first_query_of_full_prefill_sees_one_key():
    rng = np.random.default_rng(10)
    Q, K, V = _rand(rng, 5, 5, 2, 1, 4)
    O, L = extend_attention(Q, K, V, 0.5)
    np.testing.assert_array_equal(O[0], np.repeat(V[0], 2, axis=0))
    np.testing.assert_allclose(L[0], 0.5 * (Q[0] @ K[0, 0]), rtol=0, atol=1e-14)


def test_bad_token_count():
    rng = np.random.default_rng(11)
    Q, K, V = _rand(rng, 3, 2, 1, 1, 4)
    with pytest.raises(ValueError):
        extend_attention(Q, K, V, 0.5)
