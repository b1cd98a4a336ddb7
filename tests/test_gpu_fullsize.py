"""Full-size parity: BASELINE.json configs 1 and 2 at their bench sizes (bf16, and FP8 pages), in the launch
configuration bench.py times (persistent grid, automatic splits, in-kernel tail merge,
PDL-chained layer calls), checked on sampled outputs the fp64 oracle computes one by one.
"""
import numpy as np
import pytest
import torch

import bench
from paper_2511_20048_b200 import spa
from spa_inputs import KIND_K, KIND_Q, KIND_V, kv_bits_np, kv_bits_torch

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _run(config, resident, sample_groups, calls_to_check, fp8=False):
    recipe = bench.recipe_for(config)
    m = recipe.model
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    layers = list(range(resident))
    sched = bench.layer_schedule(recipe, resident)
    pool = spa.Pool(resident, m.num_q_heads, m.num_kv_heads, m.head_dim, bench.pages_for(recipe, 4), device=dev,
                    kv_scale=np.full((resident, m.num_kv_heads, 2), bench.FP8_SCALE, np.float32) if fp8 else None)
    ids, reqs, batch = bench.build_batch(spa, pool, recipe, layers, slice(0, m.num_kv_heads), dev)
    N = len(reqs)
    # one decode step: append the step token, plan every window, run the whole schedule chained
    k = kv_bits_torch(recipe.seed, KIND_K, 500_000, layers, np.arange(N), m.num_kv_heads, m.head_dim, dev).contiguous()
    v = kv_bits_torch(recipe.seed, KIND_V, 500_000, layers, np.arange(N), m.num_kv_heads, m.head_dim, dev).contiguous()
    pool.append(reqs, [1] * N, k, v, stream=stream)
    windows = sorted({w for _, w in sched})
    plans = {w: spa.Plan(pool) for w in windows}
    for w, p in plans.items():
        p.plan(reqs, w, stream=stream)
    q_res = kv_bits_torch(recipe.seed, KIND_Q, 1_000_000, layers, np.arange(N), m.num_q_heads, m.head_dim, dev)
    o = torch.empty((len(sched), N, m.num_q_heads, m.head_dim), dtype=torch.bfloat16, device=dev)
    lse = torch.empty((len(sched), N, m.num_q_heads), dtype=torch.float32, device=dev)
    for ci, (r, w) in enumerate(sched):
        plans[w].decode(r, q_res[r].contiguous(), o[ci], lse[ci], scale=m.softmax_scale, stream=stream)
    torch.cuda.synchronize()
    assert torch.isfinite(o.float()).all() and not torch.isnan(lse).any()
    rows = [i for i, nm in enumerate(batch) if nm[0] in sample_groups]
    worst = (0.0, 0.0)
    for ci in calls_to_check:
        r, w = sched[ci]
        qb = kv_bits_np(recipe.seed, KIND_Q, 1_000_000, [r], np.arange(N), m.num_q_heads, m.head_dim)[0]
        O, L = bench.oracle_sample(recipe, batch, rows, r, qb, steps_appended=1, window=w, fp8=fp8)
        eo = float(np.abs(o[ci, rows].float().cpu().numpy() - O).max())
        el = float(np.abs(lse[ci, rows].cpu().numpy() - L).max())
        worst = (max(worst[0], eo), max(worst[1], el))
    return worst


def test_qwen_config_full_size_sampled():
    eo, el = _run("qwen", 64, {0, 13, 31}, [0, 37, 63])
    assert eo <= 2e-2 and el <= 1e-3, (eo, el)


def test_gemma_config_full_size_sampled():
    eo, el = _run("gemma", 6, {0, 40}, [0, 5, 61])       # local, global, local
    assert eo <= 2e-2 and el <= 1e-3, (eo, el)


def test_qwen_config_full_size_sampled_fp8_pages():
    eo, el = _run("qwen", 64, {0, 31}, [0, 63], fp8=True)
    assert eo <= 2e-2 and el <= 1e-3, (eo, el)


def test_gemma_config_full_size_sampled_fp8_pages():
    eo, el = _run("gemma", 6, {0, 40}, [0, 5], fp8=True)
    assert eo <= 2e-2 and el <= 1e-3, (eo, el)


def test_long32k_config_full_size_sampled():
    """BJ config 4: 128 agents at 30k-32k contexts + one fork each, up to 64 splits per range,
    the 64-call model step over 4 resident layers (bench.py's launch configuration)."""
    eo, el = _run("long", 4, {0, 77, 127}, [0, 33, 63])
    assert eo <= 2e-2 and el <= 1e-3, (eo, el)


def test_extend_mixed_step_full_size_sampled():
    """F2 at BJ config 1's size on the tcgen05 path (bench_extend.py's launch configuration:
    max_rows 128, folded tails, 8 resident layers PDL-chained): every parent decodes one token
    while its fork prefills its 16-token prompt; sampled groups vs the fp64 extend oracle."""
    from oracle.attention import extend_attention
    from oracle.replay import bits_to_f64
    from spa_inputs import workloads

    rec = workloads.qwen()
    m = rec.model
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    Lr = 4
    layers = list(range(Lr))
    pool = spa.Pool(Lr, m.num_q_heads, m.num_kv_heads, m.head_dim, bench.pages_for(rec, 4), device=dev)
    ids, reqs, batch = bench.build_batch(spa, pool, rec, layers, slice(0, m.num_kv_heads), dev)
    lens = [pool.page_table(r)[2] for r in reqs]
    nq = [1 if who == "main" else min(16, n) for (gi, who), n in zip(batch, lens)]
    rows = int(sum(nq))
    q = kv_bits_torch(rec.seed, KIND_Q, 3_000_000, layers, np.arange(rows), m.num_q_heads, m.head_dim, dev)
    o = torch.empty((Lr, rows, m.num_q_heads, m.head_dim), dtype=torch.bfloat16, device=dev)
    lse = torch.empty((Lr, rows, m.num_q_heads), dtype=torch.float32, device=dev)
    plan = spa.Plan(pool, max_rows=128)
    plan.plan(reqs, 0, stream=stream, n_query=nq)
    for i in range(2 * Lr):   # repeated launches of one plan
        plan.decode(i % Lr, q[i % Lr].contiguous(), o[i % Lr], lse[i % Lr], scale=m.softmax_scale, stream=stream)
    torch.cuda.synchronize()
    starts = np.concatenate([[0], np.cumsum(nq)])
    worst = [0.0, 0.0]
    for li in (0, Lr - 1):
        qb = kv_bits_np(rec.seed, KIND_Q, 3_000_000, [li], np.arange(rows), m.num_q_heads, m.head_dim)[0]
        for i, (gi, who) in enumerate(batch):
            if gi not in (0, 17, 31):
                continue
            K = bits_to_f64(bench.logical_kv_np(rec, gi, who, [li], KIND_K)[0])
            V = bits_to_f64(bench.logical_kv_np(rec, gi, who, [li], KIND_V)[0])
            r0, r1 = int(starts[i]), int(starts[i + 1])
            O, L = extend_attention(bits_to_f64(qb[r0:r1]), K, V, m.softmax_scale)
            worst[0] = max(worst[0], float(np.abs(o[li, r0:r1].float().cpu().numpy() - O).max()))
            worst[1] = max(worst[1], float(np.abs(lse[li, r0:r1].cpu().numpy() - L).max()))
    assert worst[0] <= 2e-2 and worst[1] <= 1e-3, worst
