"""F2 on the tcgen05 extend kernel (plans with max_rows 128) vs the fp64 oracle."""
import numpy as np
import pytest
import torch

from test_gpu_extend import _lengths, _n_query, _ok, run_extend
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
