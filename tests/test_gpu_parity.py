"""GPU parity: the CUDA path through the C ABI vs the fp64 oracle (pytest -m gpu).

Tolerances are the north_star's: O within 2e-2 max-abs (unit-scale values), LSE within
1e-3; page tables and gathered KV bytes bit-exact.  Every parity case runs the four
discriminating input families so a dropped or mis-indexed page
moves O by O(1).
"""
import numpy as np
import pytest
import torch

from gpu_compare import assert_bf16_close
from harness import LSE_TOL, O_TOL, GpuBatch, bits_to_torch, compare, run_parity, torch_to_bits
from oracle.attention import merge_partials
from oracle.kvmodel import PagingModel
from oracle.replay import Replay
from paper_2511_20048_b200 import spa
from spa_inputs import families, workloads

pytestmark = pytest.mark.gpu

FAMS = ["flat", "peaky", "needle_shared_pos", "needle_tail_pos", "needle_cow_pos"]


@pytest.fixture(autouse=True)
def _need_gpu(cuda_device):
    spa.lib()
    yield


def _assert_ok(errs):
    for eo, el in errs:
        assert eo <= O_TOL and el <= LSE_TOL, (eo, el)


@pytest.mark.parametrize("prefix", [256, 250])
@pytest.mark.parametrize("family", FAMS)
def test_tiny_config(prefix, family):
    """BJ config 0: 1 layer, 8 Q / 2 KV heads, d=64, reasoning request + 1 fork."""
    errs, outs, gb, plan, _ = run_parity(workloads.tiny(prefix), family)
    _assert_ok(errs)
    # budget: bf16 P rounding <= 2^-9 max|v| + bf16 output rounding
    # <= half an ulp of |O| < 4: 7.7e-3 + 7.8e-3
    assert errs[0][0] < 1.6e-2


@pytest.mark.parametrize("seed", range(10))
@pytest.mark.parametrize("family", FAMS)
def test_random_small(seed, family):
    rng = np.random.default_rng(seed)
    window = int(rng.choice([0, 0, 5, 33, 100]))
    errs, *_ = run_parity(workloads.random_small(seed), family, window=window, split_pages=int(rng.choice([0, 2, 5])),
                          num_ctas=int(rng.choice([0, 3, 17])))
    _assert_ok(errs)


@pytest.mark.parametrize("max_rows", [16, 32])
@pytest.mark.parametrize("sharing", [True, False])
def test_sharing_and_row_tiles(max_rows, sharing):
    rec = workloads.sweep(12, 0.75, seed=7)     # parents with 3 forks: 20 rows per group
    rec.groups = rec.groups[:3]
    for g in rec.groups:
        g.prefix = 300 + g.prefix % 200
    errs, *_ = run_parity(rec, "needle_shared_pos", sharing=sharing, max_rows=max_rows, split_pages=3)
    _assert_ok(errs)


def test_gathered_pool_bytes_bit_exact():
    rec = workloads.random_small(3, workloads.Model("m", 2, 8, 2, 128), max_prefix=200)
    inp = families.make_inputs(rec, "flat")
    gb = GpuBatch(inp)
    rp = Replay(inp, num_pages=gb.pool.num_pages)
    kb = torch_to_bits(gb.pool.k)
    vb = torch_to_bits(gb.pool.v)
    for nm, rid in gb.ids.items():
        st, pages, n = gb.pool.page_table(rid)
        mst, mpages, mn = rp.paging.page_table(rp.rid[nm])
        assert (pages, n) == (mpages, mn)
        idx_p = np.array([pages[t // 16] for t in range(n)], dtype=np.int64)
        idx_s = np.arange(n) % 16
        for li in range(len(inp.layers)):
            gk = kb[li, idx_p, :, idx_s]          # [n, Hkv, d]
            gv = vb[li, idx_p, :, idx_s]
            assert np.array_equal(gk, rp.kv.K[nm][li]), nm
            assert np.array_equal(gv, rp.kv.V[nm][li]), nm


def test_fork_equals_physical_copy():
    """A forked request == the same request whose prefix was appended as fresh tokens."""
    rec = workloads.Recipe("fc", workloads.Model("m", 1, 10, 2, 128), [workloads.Group(250, 11, [9])], seed=4)
    inp = families.make_inputs(rec, "needle_cow_pos")
    gb = GpuBatch(inp)
    plan = spa.Plan(gb.pool, sharing=False, split_pages=1000)
    plan.plan(gb.reqs)
    o1, l1 = gb.decode(plan, 0)
    # the copy: a fresh request per batch member with its full logical KV appended
    rp = Replay(inp)
    pool2 = spa.Pool(1, 10, 2, 128, 64, device="cuda")
    reqs2 = []
    for nm in inp.batch:
        r = pool2.alloc()
        pool2.append([r], [rp.kv.length(nm)], bits_to_torch(rp.kv.K[nm]), bits_to_torch(rp.kv.V[nm]))
        reqs2.append(r)
    plan2 = spa.Plan(pool2, sharing=False, split_pages=1000)
    plan2.plan(reqs2)
    o2, l2 = plan2.decode(0, bits_to_torch(inp.q[0]), scale=rec.model.softmax_scale)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.equal(l1, l2)


def test_split_merge_equals_unsplit():
    rec = workloads.random_small(11, workloads.Model("m", 1, 8, 2, 128), max_prefix=400)
    e1, out1, *_ = run_parity(rec, "peaky", split_pages=1000)
    e2, out2, *_ = run_parity(rec, "peaky", split_pages=1, merge_mode=2)
    e3, out3, *_ = run_parity(rec, "peaky", split_pages=1, merge_mode=1)
    e4, out4, *_ = run_parity(rec, "peaky", split_pages=1, merge_mode=0)
    for e in (e1, e2, e3, e4):
        _assert_ok(e)
    (o1, l1), (o2, l2), (o3, l3), (o4, l4) = out1[0], out2[0], out3[0], out4[0]
    assert_bf16_close(o1, o2)
    assert (l1 - l2).abs().max().item() <= 1e-4
    # the in-kernel merges and the standalone merge kernel run the same warp merge code
    assert torch.equal(o2, o3) and torch.equal(l2, l3)
    assert torch.equal(o2, o4) and torch.equal(l2, l4)


@pytest.mark.parametrize("whole", ["0", "1"])
def test_tail_merge_group_pass_is_bitwise_per_head(monkeypatch, whole):
    """The tail merge's one-warp-per-(request, KV head) pass (G x S <= 32) gives the bits of
    the per-head merges (merge kernel, merge_mode 2)."""
    monkeypatch.setenv("SPA_MERGE_WHOLE", whole)
    rec = workloads.random_small(41, workloads.Model("m", 1, 8, 2, 128), max_prefix=120)
    e0, out0, *_ = run_parity(rec, "peaky", split_pages=3, merge_mode=0)
    e2, out2, *_ = run_parity(rec, "peaky", split_pages=3, merge_mode=2)
    _assert_ok(e0)
    _assert_ok(e2)
    (o0, l0), (o2, l2) = out0[0], out2[0]
    assert torch.equal(o0, o2) and torch.equal(l0, l2)


@pytest.mark.parametrize("mode", [0, 1, 2])
@pytest.mark.parametrize("max_rows", [16, 32])
def test_merge_paths_many_splits(mode, max_rows):
    """Many splits per request, both merge paths, two layers (counters reset between launches)."""
    rec = workloads.random_small(31, workloads.Model("m", 3, 16, 4, 128), max_prefix=500)
    errs, *_ = run_parity(rec, "needle_shared_pos", split_pages=2, max_rows=max_rows, merge_mode=mode,
                          num_ctas=9)
    _assert_ok(errs)


def test_deterministic_and_page_permutation_invariant():
    rec = workloads.random_small(21, workloads.Model("m", 1, 8, 2, 128), max_prefix=300)
    _, a, *_ = run_parity(rec, "flat", split_pages=4, num_ctas=5)
    _, b, *_ = run_parity(rec, "flat", split_pages=4, num_ctas=5)
    _, c, *_ = run_parity(rec, "flat", split_pages=4, num_ctas=5, pre_shuffle=40)
    assert torch.equal(a[0][0], b[0][0]) and torch.equal(a[0][1], b[0][1])
    assert torch.equal(a[0][0], c[0][0]) and torch.equal(a[0][1], c[0][1])


def test_sharing_on_off_agree():
    rec = workloads.qwen(seed=9, n_agents=3)
    for g in rec.groups:
        g.prefix = 500 + g.prefix % 300
    rec.model = workloads.Model("q", 1, 40, 8, 128)
    e1, a, *_ = run_parity(rec, "needle_shared_pos", sharing=True)
    e2, b, *_ = run_parity(rec, "needle_shared_pos", sharing=False)
    _assert_ok(e1)
    _assert_ok(e2)
    assert_bf16_close(a[0][0], b[0][0])


def test_single_key_and_duplicated_heads():
    m = workloads.Model("m", 1, 4, 1, 128)
    rec = workloads.Recipe("one", m, [workloads.Group(1, 0, [])], seed=5)
    inp = families.make_inputs(rec, "flat")
    gb = GpuBatch(inp)
    plan = spa.Plan(gb.pool)
    plan.plan(gb.reqs)
    q = inp.q[0].copy()
    q[:, 1] = q[:, 0]                                   # duplicated q head 0 -> 1
    o, lse = gb.decode(plan, 0, q_bits=q)
    v0 = torch.from_numpy(inp.append_v[1][0, 0, 0].view(np.int16)).view(torch.bfloat16).float()
    for h in range(4):
        assert torch.equal(o[0, h].float().cpu(), v0)   # weight 2^0 = 1 exactly
    assert torch.equal(o[0, 0], o[0, 1]) and lse[0, 0].item() == lse[0, 1].item()
    rp = Replay(inp)
    _, L = rp.expected(0, q)
    assert np.abs(lse[0].cpu().numpy() - L[0]).max() < 1e-5


def test_window_one_returns_last_value():
    rec = workloads.Recipe("w1", workloads.Model("m", 1, 8, 2, 64), [workloads.Group(100, 7, [3])], seed=6)
    errs, outs, gb, plan, rp = run_parity(rec, "flat", window=1)
    _assert_ok(errs)


def test_gemma_shaped_sliding_window():
    rec = workloads.gemma(seed=2, n_agents=3)
    for g in rec.groups:
        g.prefix = 1500 + g.prefix % 1000
    rec.model = workloads.Model("g", 2, 32, 16, 128, scale=168 ** -0.5)
    for fam in ("flat", "needle_tail_pos"):
        errs, *_ = run_parity(rec, fam, window=1024)
        _assert_ok(errs)


def test_merge_splits_abi():
    rng = np.random.default_rng(0)
    N, H, D = 5, 3, 64
    counts = [3, 1, 0, 4, 2]
    rec_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    S = rec_ptr[-1]
    po = rng.standard_normal((S, H, D)).astype(np.float32)
    pl = (rng.standard_normal((S, H)) * 3).astype(np.float32)
    pl[0, 1] = -np.inf
    pl[3:7, 2] = -np.inf               # request 3, head 2: all empty
    o = torch.full((N, H, D), 7.0, dtype=torch.bfloat16, device="cuda")
    lse = torch.full((N, H), 7.0, dtype=torch.float32, device="cuda")
    spa.spa_merge_splits(torch.from_numpy(rec_ptr).cuda(), torch.from_numpy(po).cuda(), torch.from_numpy(pl).cuda(),
                         o, lse)
    torch.cuda.synchronize()
    for r in range(N):
        for h in range(H):
            if counts[r] == 0:
                assert (o[r, h].float() == 7.0).all() and lse[r, h].item() == 7.0   # untouched
                continue
            a, b = rec_ptr[r], rec_ptr[r + 1]
            O, L = merge_partials(po[a:b, h].astype(np.float64), pl[a:b, h].astype(np.float64))
            assert np.abs(o[r, h].float().cpu().numpy() - O).max() <= 1e-2
            if L == -np.inf:
                assert lse[r, h].item() == -np.inf
            else:
                assert abs(lse[r, h].item() - L) <= 1e-5


def test_fake_rank_sharding_bitwise():
    """Rank r's head slice in its own pool, concatenated == the unsharded output (fixed splits)."""
    rec = workloads.qwen(seed=3, n_agents=4)
    for g in rec.groups:
        g.prefix = 300 + g.prefix % 400
    rec.model = workloads.Model("q", 1, 40, 8, 128)
    inp = families.make_inputs(rec, "needle_shared_pos")
    full = GpuBatch(inp)
    plan = spa.Plan(full.pool, split_pages=5, num_ctas=7)
    plan.plan(full.reqs)
    o_ref, l_ref = full.decode(plan, 0)
    for n in (2, 4, 8):
        parts_o, parts_l = [], []
        for r in range(n):
            gb = GpuBatch(inp, shard=(r, n))
            p = spa.Plan(gb.pool, split_pages=5, num_ctas=3)
            p.plan(gb.reqs)
            o, l = gb.decode(p, 0)
            parts_o.append(o)
            parts_l.append(l)
        assert torch.equal(torch.cat(parts_o, dim=1), o_ref)
        assert torch.equal(torch.cat(parts_l, dim=1), l_ref)


def test_append_decode_steps_and_free():
    """Several decode steps (append one token, re-plan, decode), then free + re-fork."""
    rec = workloads.random_small(8, workloads.Model("m", 1, 8, 2, 128), max_prefix=150)
    inp = families.make_inputs(rec, "flat")
    gb = GpuBatch(inp, num_pages=200)
    rp = Replay(inp, num_pages=200)
    plan = spa.Plan(gb.pool, split_pages=2)
    N = len(gb.reqs)
    for step in range(3):
        from spa_inputs import KIND_K, KIND_V, kv_bits_np
        kb = kv_bits_np(99, KIND_K, step, [0], np.arange(N), 2, 128)
        vb = kv_bits_np(99, KIND_V, step, [0], np.arange(N), 2, 128)
        gb.pool.append(gb.reqs, [1] * N, bits_to_torch(kb), bits_to_torch(vb))
        rp.append_step(inp.batch, kb, vb)
        plan.plan(gb.reqs)
        qb = families.kv_bits_np(5, 3, 77 + step, [0], np.arange(N), 8, 128)[0]
        o, lse = gb.decode(plan, 0, q_bits=qb)
        O, L = rp.expected(0, qb)
        eo, el = compare(o, lse, O, L)
        assert eo <= O_TOL and el <= LSE_TOL
        for nm in inp.batch:
            assert gb.pool.page_table(gb.ids[nm])[1:] == rp.paging.page_table(rp.rid[nm])[1:]
    # a speculative request finishes and a new one forks from the same parent
    victim = next(nm for nm in inp.batch if nm[1] != "main")
    gb.pool.free(gb.ids[victim])
    rp.paging.free(rp.rid[victim])
    assert gb.pool.free_pages() == rp.paging.free_pages
    assert gb.pool.refcounts() == rp.paging.refcount
    # ... and a new speculative request forks the same parent at its current length
    parent = (victim[0], "main")
    pst, ppages, plen = gb.pool.page_table(gb.ids[parent])
    child = gb.pool.fork(gb.ids[parent], plen)
    mst, mchild = rp.paging.fork(rp.rid[parent], plen)
    assert (mst, mchild) == (0, child)
    rp.kv.fork(("new", 0), parent, plen)
    kb = kv_bits_np(98, KIND_K, 0, [0], np.arange(5), 2, 128)
    vb = kv_bits_np(98, KIND_V, 0, [0], np.arange(5), 2, 128)
    gb.pool.append([child], [5], bits_to_torch(kb), bits_to_torch(vb))
    rp.kv.append(("new", 0), kb, vb)
    rp.paging.append([mchild], [5])
    names = [nm for nm in inp.batch if nm != victim] + [("new", 0)]
    reqs = [gb.ids[nm] for nm in inp.batch if nm != victim] + [child]
    plan.plan(reqs)
    qb = families.kv_bits_np(5, 3, 90, [0], np.arange(len(reqs)), 8, 128)[0]
    o, lse = plan.decode(0, bits_to_torch(qb), scale=rec.model.softmax_scale)
    torch.cuda.synchronize()
    O, L = rp.expected(0, qb, names=names)
    eo, el = compare(o, lse, O, L)
    assert eo <= O_TOL and el <= LSE_TOL
    assert gb.pool.page_table(child)[1:] == rp.paging.page_table(mchild)[1:]


def test_sharded_single_rank_layout():
    """spa_decode_attention_sharded with a 1-rank comm writes the head-major gather layout
    [Hq][N][d] (+ LSE [Hq][N]) bit-identically to spa_decode_attention."""
    rec = workloads.random_small(13, workloads.Model("m", 1, 10, 2, 128), max_prefix=200)
    errs, outs, gb, plan, rp = run_parity(rec, "flat", split_pages=3)
    _assert_ok(errs)
    o_ref, l_ref = outs[0]
    N, Hq, d = o_ref.shape
    comm = spa.Comm(b"\0" * 128, 0, 1)
    og = torch.empty((Hq, N, d), dtype=torch.bfloat16, device="cuda")
    lg = torch.empty((Hq, N), dtype=torch.float32, device="cuda")
    q = bits_to_torch(gb.inputs.q[0]).contiguous()
    plan.decode_sharded(comm, 0, q, og, lg, scale=rec.model.softmax_scale)
    torch.cuda.synchronize()
    assert torch.equal(og.permute(1, 0, 2), o_ref) and torch.equal(lg.t(), l_ref)
    comm.close()


@pytest.mark.timeout(120, method="thread")
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_back_to_back_launches_same_plan_and_layer(mode):
    """Launches chained by programmatic dependent launch may start while the previous one
    drains; repeating one (plan, layer) back to back must neither deadlock nor mix work
    queues (each launch owns a queue slot by launch id)."""
    rec = workloads.random_small(41, workloads.Model("m", 2, 8, 2, 128), max_prefix=600)
    errs, outs, gb, plan, rp = run_parity(rec, "needle_shared_pos", split_pages=2, merge_mode=mode)
    _assert_ok(errs)
    q = bits_to_torch(gb.inputs.q[1]).contiguous()
    N, Hq, d = q.shape
    o = torch.empty((12, N, Hq, d), dtype=torch.bfloat16, device="cuda")
    lse = torch.empty((12, N, Hq), dtype=torch.float32, device="cuda")
    for i in range(12):                              # no synchronisation in between
        plan.decode(1, q, o[i], lse[i], scale=rec.model.softmax_scale)
    torch.cuda.synchronize()
    for i in range(12):
        assert torch.equal(o[i], outs[1][0]) and torch.equal(lse[i], outs[1][1])
