"""Seeded synthetic input generators shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no attention, no softmax, no paging).
It only turns integer counters into bf16 bit patterns, identically in NumPy (host,
for the oracle) and in PyTorch integer ops (device, for filling the KV pool at bench
scale), so that neither side ever has to take an input from the other.

Generator: a counter-based 32-bit hash (lowbias32 finaliser) applied to a key built
from (seed, stream kind, origin request, layer, position, head, channel).  Every
32-bit hash h yields one value

    v = (b0 + b1 + b2 + b3 - 126) / 32,   b_i = (h >> 6i) & 63   (Irwin-Hall of 4)

so v is an integer multiple of 1/32 in [-3.9375, 3.9375], std ~= 1.155, and is
*exactly* representable in bf16 (|32 v| <= 126 < 2^8).  The bf16 bit pattern is
therefore obtained without any rounding step, bit-identically on both sides.

Only integer ops whose results stay below 2^63 are used (32x16-bit split multiply),
so NumPy int64 and torch int64 (CPU or CUDA) agree bit for bit.
"""
from __future__ import annotations

import numpy as np

MASK32 = 0xFFFFFFFF

KIND_K = 1
KIND_V = 2
KIND_Q = 3


def _mul32(x, c: int):
    """(x * c) mod 2^32 for x in [0, 2^32), without int64 overflow."""
    lo = c & 0xFFFF
    hi = c >> 16
    return (x * lo + (((x * hi) & 0xFFFF) << 16)) & MASK32


def hash32(x):
    """lowbias32 finaliser on int64 arrays holding values in [0, 2^32)."""
    x = x ^ (x >> 16)
    x = _mul32(x, 0x7FEB352D)
    x = x ^ (x >> 15)
    x = _mul32(x, 0x846CA68B)
    x = x ^ (x >> 16)
    return x


def _combine(a, b):
    return hash32((a ^ b) & MASK32)


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _h2v_np(h):
    s = (h & 63) + ((h >> 6) & 63) + ((h >> 12) & 63) + ((h >> 18) & 63) - 126
    f = s.astype(np.float32) / np.float32(32.0)
    return (f.view(np.uint32) >> 16).astype(np.uint16)


def stream_key_np(seed: int, kind: int, origin: int, layers, positions):
    """32-bit keys for (layer, position) pairs of one appended stream, shape [L, T]."""
    layers = np.asarray(layers, dtype=np.int64)
    positions = np.asarray(positions, dtype=np.int64)
    base = hash32(np.int64((seed * 8 + kind) & MASK32))
    base = _combine(base, np.int64(origin & MASK32))
    kl = _combine(base, layers & MASK32)  # [L]
    return _combine(kl[:, None], (positions[None, :] * 0x9E3779B1) & MASK32)


def channel_key_np(n_heads: int, head_dim: int):
    hc = np.arange(n_heads * head_dim, dtype=np.int64)
    return hash32((hc + 0x6A09E667) & MASK32)


def kv_bits_np(seed: int, kind: int, origin: int, layers, positions, n_heads: int, head_dim: int):
    """bf16 bit patterns (uint16) of shape [L, T, H, d] for one stream of tokens.

    `origin` identifies the request that appended these tokens; `positions` are the
    logical token positions inside that request.  A forked child reads its parent's
    tokens, so the logical KV of a child is the parent's stream followed by its own.
    """
    kl = stream_key_np(seed, kind, origin, layers, positions)
    hc = channel_key_np(n_heads, head_dim)
    h = _combine(kl[:, :, None], hc[None, None, :])
    L, T = kl.shape
    return _h2v_np(h).reshape(L, T, n_heads, head_dim)


def q_bits_np(seed: int, step: int, layers, n_req: int, n_heads: int, head_dim: int):
    """bf16 bits [L, N, Hq, d] of queries for one decode step (origin = step)."""
    return kv_bits_np(seed, KIND_Q, step, layers, np.arange(n_req), n_heads, head_dim)


# ----------------------------------------------------------------------------- full-precision values
# The counter-hash values above sit on a 7-bit grid (multiples of 1/32, |32 v| <= 126), so
# they never set the bf16 mantissa LSB and keep every q.k product exact in fp32.  These
# generators fill the whole bf16 format (parity inputs too narrow):
#
#   normal(sigma)   v = RNE_bf16(fp32(sigma * z)), z ~ N(0, 1) by Box-Muller from two
#                   counter hashes (float64 NumPy; host only);
#   wide(emin, emax) random sign, exponent uniform in [emin, emax], all 7 mantissa bits from
#                   the hash: integer ops only, bit-identical in NumPy and torch.


def _bf16_rne_bits(f32):
    """bf16 bits of float32 values, round to nearest even (finite inputs)."""
    u = np.asarray(f32, np.float32).view(np.uint32).astype(np.int64)
    return (((u + 0x7FFF + ((u >> 16) & 1)) >> 16) & 0xFFFF).astype(np.uint16)


def _hash_grid_np(seed, kind, origin, layers, positions, n_heads, head_dim, salt=0):
    kl = stream_key_np(seed, kind, origin, layers, positions)
    hc = channel_key_np(n_heads, head_dim)
    if salt:
        hc = _combine(hc, np.int64(salt))
    L, T = kl.shape
    return _combine(kl[:, :, None], hc[None, None, :]).reshape(L, T, n_heads, head_dim)


def normal_bits_np(sigma: float, seed, kind, origin, layers, positions, n_heads, head_dim):
    """bf16 bits [L, T, H, d] of RNE_bf16(fp32(sigma * z)), z ~ N(0, 1) (Box-Muller)."""
    h1 = _hash_grid_np(seed, kind, origin, layers, positions, n_heads, head_dim)
    h2 = hash32((h1 ^ 0x9E3779B9) & MASK32)
    u1 = (h1.astype(np.float64) + 0.5) / 4294967296.0
    u2 = h2.astype(np.float64) / 4294967296.0
    z = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
    return _bf16_rne_bits((sigma * z).astype(np.float32))


def _wide_from_hash(h, emin: int, emax: int):
    sign = (h >> 31) & 1
    e = emin + (h & 0xFFFF) % (emax - emin + 1)
    mant = (h >> 16) & 0x7F
    return (sign << 15) | ((e + 127) << 7) | mant


def wide_bits_np(emin: int, emax: int, seed, kind, origin, layers, positions, n_heads, head_dim):
    """bf16 bits [L, T, H, d]: random sign, exponent uniform in [emin, emax] (|v| in
    [2^emin, 2^(emax+1))), random 7-bit mantissa."""
    h = _hash_grid_np(seed, kind, origin, layers, positions, n_heads, head_dim, salt=0x5bd1e995)
    return _wide_from_hash(h, emin, emax).astype(np.uint16)


# ----------------------------------------------------------------------------- torch
def _torch():
    import torch  # noqa: WPS433 (lazy: the oracle side never needs torch)

    return torch


def kv_bits_torch(seed: int, kind: int, origin: int, layers, positions, n_heads: int, head_dim: int,
                  device="cuda"):
    """Same values as kv_bits_np, produced with torch int64 ops on `device`.

    Returns a torch.bfloat16 tensor [L, T, H, d] whose bit patterns equal kv_bits_np(...).
    """
    torch = _torch()
    kl = torch.from_numpy(stream_key_np(seed, kind, origin, layers, positions)).to(device)
    hc = torch.from_numpy(channel_key_np(n_heads, head_dim)).to(device)
    h = hash32((kl[:, :, None] ^ hc[None, None, :]) & MASK32)
    s = (h & 63) + ((h >> 6) & 63) + ((h >> 12) & 63) + ((h >> 18) & 63) - 126
    v = (s.to(torch.float32) / 32.0).to(torch.bfloat16)
    L, T = kl.shape
    return v.reshape(L, T, n_heads, head_dim)


def wide_bits_torch(emin: int, emax: int, seed, kind, origin, layers, positions, n_heads, head_dim, device="cuda"):
    """wide_bits_np on `device` with torch int64 ops (bit-identical); returns torch.bfloat16."""
    torch = _torch()
    kl = torch.from_numpy(stream_key_np(seed, kind, origin, layers, positions)).to(device)
    hc = torch.from_numpy(_combine(channel_key_np(n_heads, head_dim), np.int64(0x5bd1e995))).to(device)
    h = hash32((kl[:, :, None] ^ hc[None, None, :]) & MASK32)
    b = _wide_from_hash(h, emin, emax)
    b = torch.where(b >= 32768, b - 65536, b).to(torch.int16)
    L, T = kl.shape
    return b.view(torch.bfloat16).reshape(L, T, n_heads, head_dim)


def bits_to_f64(bits) -> np.ndarray:
    """Exact decode of bf16 bit patterns (uint16 / int16 array) to float64."""
    u = np.asarray(bits).astype(np.uint16).astype(np.uint32) << 16
    return u.view(np.float32).astype(np.float64)


def f32_to_bf16_bits_exact(x: np.ndarray) -> np.ndarray:
    """bf16 bits of float values that are exactly representable in bf16 (asserted)."""
    f = np.asarray(x, dtype=np.float32)
    u = f.view(np.uint32)
    if np.any(u & 0xFFFF):
        raise ValueError("value not exactly representable in bf16")
    return (u >> 16).astype(np.uint16)
