"""Decode attention and split-KV merge, fp64, written from the definition.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper (arXiv 2511.20048) never writes attention down; the decode step it costs is
"T_h(emptyset, N)", the time of a batch of N decode requests (Eq. 3,
Sec. IV-A), with N = N_m + N_s + N_a (Table I).  What one decode request
computes in each layer is textbook scaled-dot-product attention of its single new query
token against every key of its context, which for a grouped-query model reads:

    G = Hq / Hkv,  g(h) = floor(h / G)                          (reading #5)
    lo = max(0, n - W) if W > 0 else 0                          (reading #9)
    z_j   = scale * sum_c q[h, c] * K[j, g(h), c],   lo <= j < n  (reading #6, #8)
    LSE_h = m + ln sum_j exp(z_j - m),  m = max_j z_j           (reading #7: natural log)
    O[h]  = sum_j exp(z_j - LSE_h) * V[j, g(h), :]

The extend step (F2) is the same definition per query token t of a request's last T
tokens: the context is cut after the token's own position (causal).

The split-KV merge (north_star "split-KV partial-LSE merge"): for partials (O_s, LSE_s)
computed over disjoint key subsets,

    LSE = m + ln sum_{s: LSE_s > -inf} exp(LSE_s - m),   m = max_s LSE_s
    O   = sum_s exp(LSE_s - LSE) * O_s
    all partials -inf (or none)  ->  LSE = -inf, O = 0          (reading #11)
"""
from __future__ import annotations

import numpy as np


def decode_attention(q: np.ndarray, K: np.ndarray, V: np.ndarray, scale: float, window: int = 0):
    """One decode request, one layer.

    q: [Hq, d] fp64 query of the new token.
    K, V: [n, Hkv, d] fp64 logical keys/values of the request (n >= 1), in logical order;
          the query attends to all n of them, its own just-appended key included (#8).
    Returns (O [Hq, d] fp64, LSE [Hq] fp64).
    """
    q = np.asarray(q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    Hq, d = q.shape
    n, Hkv, _ = K.shape
    if n == 0:
        raise ValueError("decode over an empty request (reading #11)")
    if Hq % Hkv:
        raise ValueError("Hq must be a multiple of Hkv")
    G = Hq // Hkv
    lo = max(0, n - window) if window > 0 else 0
    O = np.zeros((Hq, d))
    LSE = np.zeros(Hq)
    for g in range(Hkv):
        Qg = q[g * G:(g + 1) * G]              # [G, d]
        Kg = K[lo:n, g, :]                     # [n', d]
        Vg = V[lo:n, g, :]
        Z = scale * (Qg @ Kg.T)                # [G, n']  (BLAS dgemm)
        m = Z.max(axis=1, keepdims=True)
        lse = m + np.log(np.exp(Z - m).sum(axis=1, keepdims=True))
        P = np.exp(Z - lse)
        O[g * G:(g + 1) * G] = P @ Vg
        LSE[g * G:(g + 1) * G] = lse[:, 0]
    return O, LSE


def extend_attention(Q: np.ndarray, K: np.ndarray, V: np.ndarray, scale: float, window: int = 0):
    """The last T tokens of one request as queries: the prefill of an extension (the
    speculative prompt appended to a fork of c_i, "prefill overhead is added
    once per speculative request"), causal.

    Q: [T, Hq, d] fp64 queries of the request's last T tokens, in order.
    K, V: [n, Hkv, d] fp64 logical keys/values of the request, n >= T, the T new tokens
          included (appended before attention, reading #8).
    Token t sits at position p = n - T + t and attends to keys [max(0, p + 1 - W), p + 1)
    (window W > 0, reading #9) or [0, p + 1): that is, by definition, the decode attention
    of the request's context cut after position p -- which is what is computed here.
    Returns (O [T, Hq, d] fp64, LSE [T, Hq] fp64).
    """
    Q = np.asarray(Q, dtype=np.float64)
    T = Q.shape[0]
    n = K.shape[0]
    if T < 1 or T > n:
        raise ValueError("need 1 <= T <= n query tokens")
    O = np.zeros(Q.shape)
    LSE = np.zeros(Q.shape[:2])
    for t in range(T):
        p = n - T + t
        O[t], LSE[t] = decode_attention(Q[t], K[:p + 1], V[:p + 1], scale, window)
    return O, LSE


def decode_attention_keys(q: np.ndarray, K: np.ndarray, V: np.ndarray, scale: float, keys):
    """Attention of every query head over an explicit subset of logical key indices.

    Used to form split partials: an empty subset returns (O = 0, LSE = -inf) (#11).
    """
    keys = np.asarray(list(keys), dtype=np.int64)
    Hq, d = q.shape
    if keys.size == 0:
        return np.zeros((Hq, d)), np.full(Hq, -np.inf)
    Hkv = K.shape[1]
    G = Hq // Hkv
    O = np.zeros((Hq, d))
    LSE = np.zeros(Hq)
    for g in range(Hkv):
        Qg = np.asarray(q[g * G:(g + 1) * G], dtype=np.float64)
        Kg = np.asarray(K[keys, g, :], dtype=np.float64)
        Vg = np.asarray(V[keys, g, :], dtype=np.float64)
        Z = scale * (Qg @ Kg.T)
        m = Z.max(axis=1, keepdims=True)
        lse = m + np.log(np.exp(Z - m).sum(axis=1, keepdims=True))
        O[g * G:(g + 1) * G] = np.exp(Z - lse) @ Vg
        LSE[g * G:(g + 1) * G] = lse[:, 0]
    return O, LSE


def merge_partials(part_o: np.ndarray, part_lse: np.ndarray):
    """Merge S split partials of one (request, head).

    part_o: [S, d], part_lse: [S].  Returns (O [d], LSE scalar).
    """
    part_o = np.asarray(part_o, dtype=np.float64)
    part_lse = np.asarray(part_lse, dtype=np.float64)
    live = part_lse > -np.inf
    if not np.any(live):
        return np.zeros(part_o.shape[-1]), -np.inf
    m = part_lse[live].max()
    lse = m + np.log(np.exp(part_lse[live] - m).sum())
    w = np.exp(part_lse[live] - lse)
    return (w[:, None] * part_o[live]).sum(axis=0), lse
