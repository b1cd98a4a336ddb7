"""Replay a batch's allocator call log on the oracle models and compute expected outputs.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Inputs arrive as bf16 bit patterns from `spa_inputs` (never from the CUDA path); they are
decoded exactly to fp64 and fed to `attention.decode_attention`, request by request.
"""
from __future__ import annotations

import numpy as np

from .attention import decode_attention, extend_attention
from .fp8 import dequantize_e4m3, quantize_kv
from .kvmodel import OK, LogicalKV, PagingModel


def bits_to_f64(bits) -> np.ndarray:
    u = np.asarray(bits).astype(np.uint16).astype(np.uint32) << 16
    return u.view(np.float32).astype(np.float64)


class Replay:
    """Dense logical KV (+ optional paging model) built from a call log."""

    def __init__(self, inputs, num_pages: int | None = None, page_size: int = 16, names=None, kv_fp8_scale=None):
        """inputs: spa_inputs.families.BatchInputs.  names: restrict data to these
        request names (and whatever they fork from) -- everything else is metadata only.
        kv_fp8_scale: [L_stored, Hkv, 2] (k_scale, v_scale) -> the pool stores e4m3 codes
        (S8(f) F4): attention runs on scale * e4m3(fp32(x) / scale) (oracle/fp8.py)."""
        m = inputs.recipe.model
        self.inputs = inputs
        self.fp8 = None if kv_fp8_scale is None else np.asarray(kv_fp8_scale, dtype=np.float32)
        self.kv = LogicalKV(len(inputs.layers), m.num_kv_heads, m.head_dim)
        self.paging = PagingModel(num_pages, page_size) if num_pages else None
        self.rid = {}
        for oi, op in enumerate(inputs.ops):
            kind = op[0]
            if kind == "alloc":
                self.kv.alloc(op[1])
                if self.paging:
                    st, r = self.paging.alloc()
                    self.rid[op[1]] = r
            elif kind == "append":
                _, name, origin, start, n = op
                assert self.kv.length(name) == start
                self.kv.append(name, inputs.append_k[oi], inputs.append_v[oi])
                if self.paging:
                    assert self.paging.append([self.rid[name]], [n]) == OK
            elif kind == "fork":
                _, child, parent, plen = op
                self.kv.fork(child, parent, plen)
                if self.paging:
                    st, r = self.paging.fork(self.rid[parent], plen)
                    assert st == OK
                    self.rid[child] = r

    def append_step(self, names, k_bits, v_bits):
        """One decode step: append one token per request. k_bits: [L, N, Hkv, d]."""
        for i, nm in enumerate(names):
            self.kv.append(nm, k_bits[:, i:i + 1], v_bits[:, i:i + 1])
        if self.paging:
            assert self.paging.append([self.rid[n] for n in names], [1] * len(names)) == OK

    def kv_f64(self, name, layer_pos: int):
        """fp64 (K, V) [n, Hkv, d] of a request at stored-layer index layer_pos, as the pool holds them."""
        K = bits_to_f64(self.kv.K[name][layer_pos])
        V = bits_to_f64(self.kv.V[name][layer_pos])
        if self.fp8 is not None:
            ks = self.fp8[layer_pos, :, 0][None, :, None]
            vs = self.fp8[layer_pos, :, 1][None, :, None]
            K = dequantize_e4m3(quantize_kv(K.astype(np.float32), ks), ks)
            V = dequantize_e4m3(quantize_kv(V.astype(np.float32), vs), vs)
        return K, V

    def expected(self, layer_pos: int, q_bits, names=None, window: int = 0, scale=None):
        """fp64 (O [N, Hq, d], LSE [N, Hq]) for the batch at stored-layer index layer_pos."""
        m = self.inputs.recipe.model
        scale = m.softmax_scale if scale is None else scale
        names = self.inputs.batch if names is None else names
        O = np.zeros((len(names), m.num_q_heads, m.head_dim))
        LSE = np.zeros((len(names), m.num_q_heads))
        for i, nm in enumerate(names):
            K, V = self.kv_f64(nm, layer_pos)
            O[i], LSE[i] = decode_attention(bits_to_f64(q_bits[i]), K, V, scale, window)
        return O, LSE

    def expected_extend(self, layer_pos: int, q_rows_bits, n_query, names=None, window: int = 0, scale=None):
        """fp64 (O [rows, Hq, d], LSE [rows, Hq]) of an extend batch: request i's last
        n_query[i] tokens are rows (request-major, token-minor), as spa_extend_plan numbers them."""
        m = self.inputs.recipe.model
        scale = m.softmax_scale if scale is None else scale
        names = self.inputs.batch if names is None else names
        rows = int(sum(n_query))
        O = np.zeros((rows, m.num_q_heads, m.head_dim))
        LSE = np.zeros((rows, m.num_q_heads))
        r0 = 0
        for i, nm in enumerate(names):
            T = int(n_query[i])
            K, V = self.kv_f64(nm, layer_pos)
            O[r0:r0 + T], LSE[r0:r0 + T] = extend_attention(bits_to_f64(q_rows_bits[r0:r0 + T]), K, V, scale, window)
            r0 += T
        return O, LSE
