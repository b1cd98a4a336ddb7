"""Test harness: drive the C ABI on the GPU with seeded inputs and compare with the oracle.

Test infrastructure (imports both the product binding and the oracle; neither imports
the other).  Inputs come only from spa_inputs; expected values only from oracle/.
"""
from __future__ import annotations

import numpy as np
import torch

from oracle.replay import Replay
from paper_2511_20048_b200 import spa
from spa_inputs import families, workloads

O_TOL = 2e-2      # BASELINE.json north_star: max-abs on unit-scale values
LSE_TOL = 1e-3    # BASELINE.json north_star: per-head LSE


def bits_to_torch(bits: np.ndarray, device="cuda") -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).to(device).view(torch.bfloat16)


def torch_to_bits(t: torch.Tensor) -> np.ndarray:
    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def pages_needed(recipe, extra_tokens=0) -> int:
    n = 0
    for g in recipe.groups:
        n += -(-(g.prefix + (g.parent_tail or 0) + extra_tokens) // 16)
        if g.spec_prompt is not None:   # the nested speculative request: CoW page + its prompt
            n += -(-(g.spec_prompt + 16 + extra_tokens) // 16)
        n += sum(-(-(ft + 16 + extra_tokens) // 16) for ft in g.fork_tails)
    return n + 8


class GpuBatch:
    """A recipe's batch built in a GPU pool through the C ABI."""

    def __init__(self, inputs: families.BatchInputs, num_pages=None, device="cuda", shard=(0, 1),
                 pre_shuffle=0, kv_scale=None):
        m = inputs.recipe.model
        self.inputs = inputs
        self.model = m
        r, n = shard
        self.hkv_l = m.num_kv_heads // n
        self.hq_l = m.num_q_heads // n
        self.kv_sl = slice(r * self.hkv_l, (r + 1) * self.hkv_l)
        self.q_sl = slice(r * self.hq_l, (r + 1) * self.hq_l)
        L = len(inputs.layers)
        self.pool = spa.Pool(L, self.hq_l, self.hkv_l, m.head_dim, num_pages or pages_needed(inputs.recipe) + pre_shuffle,
                             device=device, kv_scale=None if kv_scale is None else kv_scale[:, self.kv_sl])
        if pre_shuffle:   # permute physical page ids: occupy, then free every other page
            junk = [self.pool.alloc() for _ in range(pre_shuffle)]
            for j in junk:
                z = torch.zeros((L, 16, self.hkv_l, m.head_dim), dtype=torch.bfloat16, device=device)
                self.pool.append([j], [16], z, z)
            for j in junk[::2]:
                self.pool.free(j)
        self.ids = {}
        for oi, op in enumerate(inputs.ops):
            if op[0] == "alloc":
                self.ids[op[1]] = self.pool.alloc()
            elif op[0] == "append":
                k = bits_to_torch(inputs.append_k[oi][:, :, self.kv_sl], device)
                v = bits_to_torch(inputs.append_v[oi][:, :, self.kv_sl], device)
                self.pool.append([self.ids[op[1]]], [op[4]], k, v)
            elif op[0] == "fork":
                self.ids[op[1]] = self.pool.fork(self.ids[op[2]], op[3])
        self.reqs = [self.ids[nm] for nm in inputs.batch]

    def decode(self, plan: spa.Plan, layer_pos: int, scale=None, q_bits=None):
        m = self.model
        q_bits = self.inputs.q[layer_pos] if q_bits is None else q_bits
        q = bits_to_torch(q_bits[:, self.q_sl]).contiguous()
        o, lse = plan.decode(layer_pos, q, scale=m.softmax_scale if scale is None else scale)
        torch.cuda.synchronize()
        return o, lse


def compare(o: torch.Tensor, lse: torch.Tensor, O_ref: np.ndarray, L_ref: np.ndarray):
    """Returns (max |O - O_ref|, max |LSE - LSE_ref|) with O upcast exactly."""
    og = o.float().cpu().numpy().astype(np.float64)
    lg = lse.cpu().numpy().astype(np.float64)
    return float(np.abs(og - O_ref).max()), float(np.abs(lg - L_ref).max())


def fp8_scales(inputs: families.BatchInputs) -> np.ndarray:
    """Static per-(stored layer, KV head) e4m3 scales (k_scale, v_scale) = amax / 448 over
    the batch's appended K / V (a calibration pass over the synthetic inputs)."""
    m = inputs.recipe.model
    amax = np.zeros((len(inputs.layers), m.num_kv_heads, 2), np.float32)
    for oi, op in enumerate(inputs.ops):
        if op[0] == "append":
            for t, arr in ((0, inputs.append_k[oi]), (1, inputs.append_v[oi])):
                x = np.abs((arr.astype(np.uint32) << 16).view(np.float32))    # [L, n, Hkv, d]
                amax[:, :, t] = np.maximum(amax[:, :, t], x.max(axis=(1, 3)))
    return (np.maximum(amax, 1e-3) / np.float32(448.0)).astype(np.float32)


def run_parity(recipe, family="flat", window=0, sharing=True, max_rows=16, split_pages=0, num_ctas=0,
               layers=None, pre_shuffle=0, merge_mode=0, fp8=False, teams_per_cta=0):
    inp = families.make_inputs(recipe, family, layers=layers)
    scales = fp8_scales(inp) if fp8 else None
    gb = GpuBatch(inp, pre_shuffle=pre_shuffle, kv_scale=scales)
    plan = spa.Plan(gb.pool, sharing=sharing, max_rows=max_rows, split_pages=split_pages, num_ctas=num_ctas,
                    merge_mode=merge_mode, teams_per_cta=teams_per_cta)
    plan.plan(gb.reqs, window)
    rp = Replay(inp, kv_fp8_scale=scales)
    errs = []
    outs = []
    for li in range(len(inp.layers)):
        o, lse = gb.decode(plan, li)
        O_ref, L_ref = rp.expected(li, inp.q[li], window=window)
        errs.append(compare(o, lse, O_ref, L_ref))
        outs.append((o, lse))
    return errs, outs, gb, plan, rp


def derived_tolerance(rp: Replay, layer_pos: int, q_bits: np.ndarray, window: int = 0, names=None, scale=None):
    """Per (row, head) error bounds of the bf16 decode path ("Error budget"),
    from the inputs only:

        tol_O   = V* (2^-8 + 2^-16 (1 + Z1)) + 2^-24
        tol_LSE = 2^-18 (1 + Z1) + 2^-21 |LSE| + n 2^-24 + 2^-20

    V* = max |v| over the attended keys, Z1 = scale max_j sum_c |q_c k_jc|, n = keys.
    2^-9 (P rounded to bf16 for PV) + 2^-9 (O rounded to bf16) give the 2^-8; the fp32
    accumulation of q.k over d = 128 (8 k16 MMA steps, <= 2^-19 sum |q k| worst case) gives
    a logit error <= 2^-18 Z1 and a relative weight error <= 2 of that."""
    m = rp.inputs.recipe.model
    scale = m.softmax_scale if scale is None else scale
    names = rp.inputs.batch if names is None else names
    G = m.num_q_heads // m.num_kv_heads
    tol_o = np.zeros((len(names), m.num_q_heads))
    tol_l = np.zeros((len(names), m.num_q_heads))
    O_ref, L_ref = rp.expected(layer_pos, q_bits, names=names, window=window, scale=scale)
    for i, nm in enumerate(names):
        K, V = rp.kv_f64(nm, layer_pos)
        n = K.shape[0]
        lo = max(0, n - window) if window > 0 else 0
        K, V = K[lo:], V[lo:]
        q = (np.asarray(q_bits[i]).astype(np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)
        for h in range(m.num_q_heads):
            g = h // G
            vstar = np.abs(V[:, g]).max()
            z1 = scale * (np.abs(K[:, g]) @ np.abs(q[h])).max()
            tol_o[i, h] = vstar * (2.0 ** -8 + 2.0 ** -16 * (1 + z1)) + 2.0 ** -24
            tol_l[i, h] = 2.0 ** -18 * (1 + z1) + 2.0 ** -21 * abs(L_ref[i, h]) + K.shape[0] * 2.0 ** -24 + 2.0 ** -20
    return O_ref, L_ref, tol_o, tol_l


def compare_rows(o: torch.Tensor, lse: torch.Tensor, O_ref: np.ndarray, L_ref: np.ndarray):
    """(|O - O_ref| max over channels [N, Hq], |LSE - LSE_ref| [N, Hq])."""
    og = o.float().cpu().numpy().astype(np.float64)
    lg = lse.cpu().numpy().astype(np.float64)
    return np.abs(og - O_ref).max(axis=-1), np.abs(lg - L_ref)
