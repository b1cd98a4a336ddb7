"""F4 ring-buffer storage (spa_kv_release_window) on the GPU: after releasing every page a
sliding window can no longer reach, windowed decode still matches the fp64 oracle, the
freed pages are reused by later appends, and a plan whose window reaches a released page
is refused."""
import numpy as np
import pytest

from harness import LSE_TOL, O_TOL, GpuBatch, bits_to_torch, compare
from oracle.replay import Replay
from paper_2511_20048_b200 import spa
from spa_inputs import KIND_K, KIND_V, families, kv_bits_np, workloads

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _need_gpu(cuda_device):
    spa.lib()
    yield


@pytest.mark.parametrize("family", ["needle_tail_pos", "flat"])
def test_windowed_decode_after_release(family):
    W = 100
    rec = workloads.random_small(51, workloads.Model("m", 1, 16, 4, 128), max_prefix=400)
    inp = families.make_inputs(rec, family)
    gb = GpuBatch(inp, num_pages=300)
    rp = Replay(inp)
    plan = spa.Plan(gb.pool, split_pages=2)
    N = len(gb.reqs)
    for step in range(4):
        kb = kv_bits_np(61, KIND_K, step, [0], np.arange(N), 4, 128)
        vb = kv_bits_np(61, KIND_V, step, [0], np.arange(N), 4, 128)
        gb.pool.append(gb.reqs, [1] * N, bits_to_torch(kb), bits_to_torch(vb))
        rp.append_step(inp.batch, kb, vb)
        # the documented order: append, release the pages below n - W, plan with W
        gb.pool.release_window(gb.reqs, W)
        plan.plan(gb.reqs, W)
        qb = families.kv_bits_np(5, 3, 70 + step, [0], np.arange(N), 16, 128)[0]
        o, lse = gb.decode(plan, 0, q_bits=qb)
        O, L = rp.expected(0, qb, window=W)
        eo, el = compare(o, lse, O, L)
        assert eo <= O_TOL and el <= LSE_TOL, (step, eo, el)
    released = sum(p < 0 for r in gb.reqs for p in gb.pool.page_table(r)[1])
    assert released > 0
    with pytest.raises(spa.SpaError) as e:                 # a wider window needs released pages
        plan.plan(gb.reqs, 4 * W)
    assert e.value.status == spa.SPA_ERR_INVALID_ARG
    free_before = len(gb.pool.free_pages())
    a = gb.pool.alloc()                                    # released pages are reused
    z = bits_to_torch(np.zeros((1, 16 * free_before, 4, 128), np.uint16))
    gb.pool.append([a], [16 * free_before], z, z)
    assert len(gb.pool.free_pages()) == 0


@pytest.mark.parametrize("family", ["needle_shared_pos", "needle_tail_pos", "flat"])
def test_released_family_shares_and_matches_oracle(family):
    """A parent and 3 forks release different leading pages; the plan still reads their
    common window region once (plus a head range) and decode matches the oracle."""
    W = 200
    model = workloads.Model("m", 1, 16, 4, 128)
    rec = workloads.Recipe("fam", model, [workloads.Group(600, 5, [20, 25, 30]),
                                          workloads.Group(333, 40, [17, 19])], seed=12)
    inp = families.make_inputs(rec, family)
    gb = GpuBatch(inp, num_pages=200)
    gb.pool.release_window(list(gb.ids.values()), W)
    rp = Replay(inp)
    for split in (0, 3):
        plan = spa.Plan(gb.pool, split_pages=split)
        plan.plan(gb.reqs, W)
        st = plan.stats()
        assert st["n_groups"] == 2 and st["unique_tokens"] < st["unshared_tokens"]
        o, lse = gb.decode(plan, 0)
        O, L = rp.expected(0, inp.q[0], window=W)
        eo, el = compare(o, lse, O, L)
        assert eo <= O_TOL and el <= LSE_TOL, (split, eo, el)
