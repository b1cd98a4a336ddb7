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
               layers=None, pre_shuffle=0, merge_mode=0, fp8=False):
    inp = families.make_inputs(recipe, family, layers=layers)
    scales = fp8_scales(inp) if fp8 else None
    gb = GpuBatch(inp, pre_shuffle=pre_shuffle, kv_scale=scales)
    plan = spa.Plan(gb.pool, sharing=sharing, max_rows=max_rows, split_pages=split_pages, num_ctas=num_ctas,
                    merge_mode=merge_mode)
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
