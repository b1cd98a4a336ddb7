"""F2 on the tcgen05 extend kernel (plans with max_rows 128) vs the fp64 oracle."""
import numpy as np
import pytest
import torch

from test_gpu_extend import _lengths, _n_query, _ok, run_extend
from paper_2511_20048_b200 import spa
from spa_inputs import workloads

pytestmark = pytest.mark.gpu


def _model(seed):
    rng = np.random.default_rng(seed)
    kv = int(rng.choice([1, 2, 4]))
    g = int(rng.choice([1, 2, 4, 5, 8]))
    return workloads.Model(f"tc{seed}", 2, kv * g, kv, 128)


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("family", ["flat", "peaky", "needle_shared_pos", "needle_cow_pos"])
def test_tc_extend_random_batches(seed, family):
    rec = workloads.random_small(900 + seed, _model(seed), max_prefix=400)
    rng = np.random.default_rng(seed)
    nq = _n_query(_lengths(rec), rng, cap=24)
    errs, _, plan = run_extend(rec, family, nq, window=int(rng.choice([0, 0, 11])), max_rows=128,
                               split_pages=int(rng.choice([0, 3, 8])), qmode="hash" if seed % 2 else "family")
    _ok(errs)


def test_tc_decode_rows_only():
    """One query row per request through the 128-row kernel (padding rows masked)."""
    rec = workloads.random_small(17, _model(3), max_prefix=300)
    errs, _, _ = run_extend(rec, "needle_tail_pos", [1] * len(_lengths(rec)), max_rows=128)
    _ok(errs)


def test_tc_matches_mma_sync_path():
    rec = workloads.random_small(23, workloads.Model("m", 1, 20, 4, 128), max_prefix=350)
    nq = _n_query(_lengths(rec), np.random.default_rng(1), cap=20)
    e1, a, _ = run_extend(rec, "peaky", nq, max_rows=128)
    e2, b, _ = run_extend(rec, "peaky", nq, max_rows=64)
    _ok(e1)
    _ok(e2)
    d = (a[0][0].float() - b[0][0].float()).abs().max().item()
    assert d <= 1.6e-2, d


@pytest.mark.parametrize("split", [0, 24, 200])
def test_tc_long_items_wrap_the_ring(split):
    """Items of many stages (the ring wraps inside an item; PV lags S by two stages),
    lazy O rescaling across stages (peaky), and both softmax warpgroups' merge."""
    G = workloads.Group
    rec = workloads.Recipe("long_items", workloads.Model("m", 1, 20, 4, 128),
                           [G(2100, 3, [18]), G(1333, None, [16, 21]), G(700, 0, [17])], seed=31)
    lens = _lengths(rec)
    nq = [min(16, n) for n in lens]
    for fam in ("peaky", "needle_shared_pos"):
        errs, _, plan = run_extend(rec, fam, nq, max_rows=128, split_pages=split, num_ctas=8)
        _ok(errs)


@pytest.mark.parametrize("split", [2, 5])
def test_tc_task_merge_over_repeated_launches(split):
    """The tcgen05 path merges split partials with one warp per (row, KV head) task
    (merge_tasks_kernel; exactly-two-record tasks take warp_merge_task_s2): parity over every
    layer of the plan (repeated launches of one plan), and merge modes 0 and 2 agree bitwise."""
    rec = workloads.random_small(77, _model(4), max_prefix=400)
    nq = _n_query(_lengths(rec), np.random.default_rng(3), cap=20)
    errs, outs, plan = run_extend(rec, "peaky", nq, max_rows=128, split_pages=split, merge_mode=0)
    _ok(errs)
    assert plan.stats()["n_records"] > 0
    _, ref, _ = run_extend(rec, "peaky", nq, max_rows=128, split_pages=split, merge_mode=2)
    for (o, l), (ro, rl) in zip(outs, ref):
        assert torch.equal(o, ro) and torch.equal(l, rl)


def test_tc_two_record_merge_matches_merge_splits_abi():
    """warp_merge_task_s2 (the two-record fast path of the task merge) equals the ABI merge
    (spa_merge_splits: warp_merge_head) bit for bit on the same partial records, read back from
    the caller-owned plan workspace (include/spa.h layout: metadata, fp32 O, fp32 LSE)."""
    G = workloads.Group
    rec = workloads.Recipe("s2", workloads.Model("m", 1, 20, 4, 128), [G(700, 0, [17]), G(333, None, [9])], seed=41)
    nq = [min(16, n) for n in _lengths(rec)]
    errs, outs, plan = run_extend(rec, "flat", nq, max_rows=128, split_pages=4096)   # no splits
    _ok(errs)
    rp = plan.debug_array(6)   # SPA_DBG_REC_PTR (include/spa_debug.h)
    n_rec = rp[-1]
    assert n_rec > 0 and all(b - a in (0, 2) for a, b in zip(rp[:-1], rp[1:]))   # the s2 path ran
    Hq, D = 20, 128
    need = plan.workspace_size()
    lse_off = need - n_rec * Hq * 4
    o_off = lse_off - ((n_rec * Hq * D * 4 + 255) // 256) * 256
    ws = plan._ws
    part_o = ws[o_off:o_off + n_rec * Hq * D * 4].view(torch.float32).view(n_rec, Hq, D)
    part_lse = ws[lse_off:lse_off + n_rec * Hq * 4].view(torch.float32).view(n_rec, Hq)
    rec_ptr = torch.tensor(rp, dtype=torch.int32, device="cuda")
    o_k, l_k = outs[-1]
    o2 = torch.zeros_like(o_k)
    l2 = torch.zeros_like(l_k)
    spa.spa_merge_splits(rec_ptr, part_o, part_lse, o2, l2)
    torch.cuda.synchronize()
    rows = [i for i, (a, b) in enumerate(zip(rp[:-1], rp[1:])) if b > a]
    assert torch.equal(o2[rows], o_k[rows]) and torch.equal(l2[rows], l_k[rows])
