"""F2: shared-prefix EXTEND attention on the GPU vs the fp64 oracle.

A step where speculative requests prefill their prompt (their last n_query tokens are causal
query rows) while main requests decode (n_query = 1), all rows of a group reading the
shared context c_i once per KV head and sub-group.  Element-wise parity
with oracle.attention.extend_attention on the same seeded inputs; tolerances are the
north_star's (O 2e-2 max-abs, LSE 1e-3).
"""
import numpy as np
import pytest
import torch

from harness import LSE_TOL, O_TOL, GpuBatch, bits_to_torch, compare
from oracle.replay import Replay
from paper_2511_20048_b200 import spa
from spa_inputs import KIND_Q, families, kv_bits_np, workloads

pytestmark = pytest.mark.gpu


def _q_rows(inp, layer_pos, n_query, mode, seed):
    """Query bits per row: the family's query of the row's request (so needles stay aligned)
    or an independent hash per row."""
    m = inp.recipe.model
    rows = int(sum(n_query))
    if mode == "hash":
        return kv_bits_np(seed, KIND_Q, 2_000_000, [layer_pos], np.arange(rows), m.num_q_heads, m.head_dim)[0]
    return np.repeat(inp.q[layer_pos], n_query, axis=0)


def run_extend(recipe, family, n_query, window=0, max_rows=16, split_pages=0, num_ctas=0, qmode="family",
               merge_mode=0, sharing=True):
    inp = families.make_inputs(recipe, family)
    gb = GpuBatch(inp)
    plan = spa.Plan(gb.pool, sharing=sharing, max_rows=max_rows, split_pages=split_pages, num_ctas=num_ctas,
                    merge_mode=merge_mode)
    plan.plan(gb.reqs, window, n_query=n_query)
    rp = Replay(inp)
    errs, outs = [], []
    for li in range(len(inp.layers)):
        qb = _q_rows(inp, li, n_query, qmode, recipe.seed)
        q = bits_to_torch(qb).contiguous()
        o, lse = plan.decode(li, q, scale=recipe.model.softmax_scale)
        torch.cuda.synchronize()
        O_ref, L_ref = rp.expected_extend(li, qb, n_query, window=window)
        errs.append(compare(o, lse, O_ref, L_ref))
        outs.append((o, lse))
    return errs, outs, plan


def _n_query(gb_lengths, rng, cap=40):
    return [int(rng.integers(1, min(n, cap) + 1)) for n in gb_lengths]


def _lengths(recipe):
    inp = families.make_inputs(recipe, "flat", layers=[0])
    rp = Replay(inp)
    return [rp.kv.length(nm) for nm in inp.batch]


def _ok(errs):
    for eo, el in errs:
        assert eo <= O_TOL and el <= LSE_TOL, (eo, el)


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("family", ["flat", "peaky", "needle_shared_pos", "needle_tail_pos"])
def test_extend_random_batches(seed, family):
    rec = workloads.random_small(500 + seed)
    rng = np.random.default_rng(seed)
    nq = _n_query(_lengths(rec), rng)
    errs, _, plan = run_extend(rec, family, nq, window=int(rng.choice([0, 0, 9])),
                               max_rows=int(rng.choice([16, 32, 64])), split_pages=int(rng.choice([0, 2, 5])),
                               qmode="hash" if seed % 2 else "family")
    _ok(errs)
    assert plan.stats()["n_req"] == sum(nq)


@pytest.mark.parametrize("max_rows", [16, 32, 64])
def test_speculative_prompt_prefill_with_parent_decode(max_rows):
    """The paper's mixed step: parents decode one token, forks prefill their prompt tail."""
    G = workloads.Group
    rec = workloads.Recipe("spec", workloads.Model("m", 2, 20, 4, 128),
                           [G(300, 5, [20, 17, 26]), G(250, 0, [16, 19]), G(64, 3, []), G(181, None, [18, 22, 30])],
                           seed=77)
    inp = families.make_inputs(rec, "flat", layers=[0])
    lens = [Replay(inp).kv.length(nm) for nm in inp.batch]
    nq = [1 if nm[1] == "main" else min(16, n) for nm, n in zip(inp.batch, lens)]
    for fam in ("needle_cow_pos", "flat"):
        errs, _, _ = run_extend(rec, fam, nq, max_rows=max_rows)
        _ok(errs)


def test_extend_of_one_token_is_decode_bitwise():
    rec = workloads.random_small(88)
    inp = families.make_inputs(rec, "peaky", layers=[0])
    gb = GpuBatch(inp)
    plan = spa.Plan(gb.pool, split_pages=3)
    plan.plan(gb.reqs, 0)
    o1, l1 = gb.decode(plan, 0)
    plan.plan(gb.reqs, 0, n_query=[1] * len(gb.reqs))
    o2, l2 = gb.decode(plan, 0)
    assert torch.equal(o1, o2) and torch.equal(l1, l2)


def test_full_prefill_of_a_request():
    """n_query = the whole request: plain causal prefill attention (first row sees 1 key)."""
    rec = workloads.random_small(99, max_prefix=120)
    lens = _lengths(rec)
    errs, outs, _ = run_extend(rec, "flat", lens, max_rows=64, qmode="hash")
    _ok(errs)


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_extend_merge_modes_agree_bitwise(mode):
    rec = workloads.random_small(123, max_prefix=300)
    rng = np.random.default_rng(5)
    nq = _n_query(_lengths(rec), rng, cap=20)
    errs, outs, _ = run_extend(rec, "peaky", nq, split_pages=2, max_rows=32, merge_mode=mode)
    _ok(errs)
    _, ref, _ = run_extend(rec, "peaky", nq, split_pages=2, max_rows=32, merge_mode=2)
    assert torch.equal(outs[0][0], ref[0][0]) and torch.equal(outs[0][1], ref[0][1])


def test_extend_sharing_off_agrees():
    rec = workloads.random_small(321, max_prefix=300)
    rng = np.random.default_rng(6)
    nq = _n_query(_lengths(rec), rng, cap=24)
    e1, a, _ = run_extend(rec, "needle_shared_pos", nq, max_rows=64)
    e2, b, _ = run_extend(rec, "needle_shared_pos", nq, max_rows=64, sharing=False)
    _ok(e1)
    _ok(e2)
