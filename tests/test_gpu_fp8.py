"""F4: FP8 (e4m3) KV pages through the C ABI vs the oracle.

The pool's codes must equal the oracle quantiser's (oracle/fp8.py) bit for bit -- K in
token-major rows, V transposed per page with the slot permutation include/spa.h states --
and decode over the fp8 pool must match the fp64 oracle run on the dequantised K/V within
the north_star tolerances (2e-2 max-abs O, 1e-3 LSE), across the input families, split
plans, merge modes, sharing on/off and the CoW'd partial pages of forks.
"""
import numpy as np
import pytest
import torch

from harness import LSE_TOL, O_TOL, GpuBatch, bits_to_torch, compare, fp8_scales, run_parity
from oracle.fp8 import quantize_kv
from oracle.replay import Replay
from paper_2511_20048_b200 import spa
from spa_inputs import KIND_K, KIND_V, families, kv_bits_np, workloads

pytestmark = pytest.mark.gpu

FAMS = ["flat", "peaky", "needle_shared_pos", "needle_tail_pos", "needle_cow_pos"]


@pytest.fixture(autouse=True)
def _need_gpu(cuda_device):
    spa.lib()
    yield


def _vcol(s):
    """include/spa.h: page slot s of an fp8 V block sits in column 4((s mod 8) div 2) + (s mod 2) + 2(s div 8)."""
    return 4 * ((s % 8) // 2) + (s % 2) + 2 * (s // 8)


def _model(layers=2):
    return workloads.Model("q", layers, 40, 8, 128)


def test_vcol_is_a_permutation():
    assert sorted(_vcol(s) for s in range(16)) == list(range(16))


@pytest.mark.parametrize("seed", [21, 22])
def test_fp8_pool_codes_bit_exact(seed):
    rec = workloads.random_small(seed, _model(), max_prefix=300)
    inp = families.make_inputs(rec, "flat")
    sc = fp8_scales(inp)
    gb = GpuBatch(inp, kv_scale=sc)
    rp = Replay(inp)
    kp = gb.pool.k.cpu().numpy()       # [L, pages, Hkv, 16, 128]
    vp = gb.pool.v.cpu().numpy()       # [L, pages, Hkv, 128, 16]
    cols = np.array([_vcol(s) for s in range(16)])
    for nm in inp.batch:
        st, pages, n = gb.pool.page_table(gb.ids[nm])
        pos = np.arange(n)
        pg = np.array(pages)[pos // 16]
        sl = pos % 16
        for li in range(len(inp.layers)):
            kf = (rp.kv.K[nm][li].astype(np.uint32) << 16).view(np.float32)      # [n, Hkv, d]
            vf = (rp.kv.V[nm][li].astype(np.uint32) << 16).view(np.float32)
            want_k = quantize_kv(kf, sc[li, :, 0][None, :, None])
            want_v = quantize_kv(vf, sc[li, :, 1][None, :, None])
            got_k = kp[li, pg, :, sl, :]                                          # [n, Hkv, d]
            got_v = vp[li][pg[:, None], np.arange(8)[None, :], :, cols[sl][:, None]]   # [n, Hkv, d]
            assert np.array_equal(got_k, want_k), (nm, li)
            assert np.array_equal(got_v, want_v), (nm, li)


@pytest.mark.parametrize("family", FAMS)
def test_fp8_qwen_shape_parity(family):
    rec = workloads.qwen(seed=3, n_agents=4)
    for g in rec.groups:
        g.prefix = 300 + g.prefix % 500
    rec.model = _model()
    errs, outs, gb, plan, _ = run_parity(rec, family, split_pages=4, fp8=True)
    for eo, el in errs:
        assert eo <= O_TOL and el <= LSE_TOL, (eo, el)


@pytest.mark.parametrize("sharing,merge_mode,split_pages,max_rows",
                         [(True, 0, 0, 16), (False, 0, 2, 16), (True, 1, 3, 32), (True, 2, 5, 64), (True, 0, 1, 16)])
def test_fp8_plan_variants(sharing, merge_mode, split_pages, max_rows):
    rec = workloads.random_small(31, _model(), max_prefix=500)
    errs, *_ = run_parity(rec, "needle_cow_pos", sharing=sharing, merge_mode=merge_mode, split_pages=split_pages,
                          max_rows=max_rows, fp8=True)
    for eo, el in errs:
        assert eo <= O_TOL and el <= LSE_TOL, (eo, el)


@pytest.mark.parametrize("max_rows,teams,merge_mode,geometry", [
    (16, 0, 0, (8, 8)),    # 8 one-warp teams, split merge in merge_kernel (merge_mode 0's choice)
    (16, 0, 1, (8, 8)),    # one-warp teams, last-arriver merge in the kernel
    (16, 4, 0, (4, 8)),    # key-split pairs (explicit teams_per_cta), tail-phase merge
    (16, 2, 1, (2, 4)),
    (16, 1, 0, (1, 2)),
    (32, 0, 0, (4, 8)),    # one warp per 16-row tile, 4 teams
])
def test_fp8_team_geometries(max_rows, teams, merge_mode, geometry):
    """Every fp8 decode instantiation (one-warp teams and key-split pairs) against the oracle,
    with forced splits so the split merge runs (S5 "Team geometry")."""
    rec = workloads.random_small(37, _model(), max_prefix=600)
    errs, _, _, plan, _ = run_parity(rec, "needle_shared_pos", split_pages=3, max_rows=max_rows, merge_mode=merge_mode,
                                     fp8=True, teams_per_cta=teams)
    assert plan.geometry()[1:] == geometry
    assert plan.stats()["n_records"] > 0
    for eo, el in errs:
        assert eo <= O_TOL and el <= LSE_TOL, (eo, el)


@pytest.mark.parametrize("merge_mode", [0, 1])
def test_fp8_windowed_twelve_teams(merge_mode):
    """Windowed fp8 plans run 12 one-warp teams per CTA (2-stage rings); forced splits."""
    rec = workloads.random_small(39, _model(), max_prefix=900)
    errs, _, _, plan, _ = run_parity(rec, "needle_tail_pos", window=200, split_pages=3, merge_mode=merge_mode,
                                     fp8=True)
    assert plan.geometry()[1:] == (12, 12)
    assert plan.stats()["n_records"] > 0
    for eo, el in errs:
        assert eo <= O_TOL and el <= LSE_TOL, (eo, el)


def test_fp8_sliding_window_and_decode_steps():
    rec = workloads.random_small(33, _model(1), max_prefix=700)
    inp = families.make_inputs(rec, "needle_tail_pos")
    sc = fp8_scales(inp)
    gb = GpuBatch(inp, num_pages=400, kv_scale=sc)
    rp = Replay(inp, kv_fp8_scale=sc)
    plan = spa.Plan(gb.pool, split_pages=3)
    N = len(gb.reqs)
    for step in range(2):
        kb = kv_bits_np(77, KIND_K, step, [0], np.arange(N), 8, 128)
        vb = kv_bits_np(77, KIND_V, step, [0], np.arange(N), 8, 128)
        gb.pool.append(gb.reqs, [1] * N, bits_to_torch(kb), bits_to_torch(vb))
        rp.append_step(inp.batch, kb, vb)
        for window in (0, 100):
            plan.plan(gb.reqs, window)
            qb = families.kv_bits_np(5, 3, 50 + step, [0], np.arange(N), 40, 128)[0]
            o, lse = gb.decode(plan, 0, q_bits=qb)
            O, L = rp.expected(0, qb, window=window)
            eo, el = compare(o, lse, O, L)
            assert eo <= O_TOL and el <= LSE_TOL, (step, window, eo, el)


def test_fp8_single_key_returns_its_dequantised_value():
    """n = 1: O = v_0 as stored (v_scale * code), LSE = the scaled logit."""
    rec = workloads.Recipe("one", _model(1), [workloads.Group(prefix=1, parent_tail=0, fork_tails=[])], seed=9)
    errs, outs, gb, plan, rp = run_parity(rec, "flat", fp8=True)
    o, lse = outs[0]
    K, V = rp.kv_f64(rp.inputs.batch[0], 0)
    want = torch.tensor(V[0], dtype=torch.float64).repeat_interleave(5, dim=0)     # G = 5 q-heads per KV head
    assert torch.allclose(o[0].double().cpu(), want, atol=2 ** -8 * want.abs().max().item() + 1e-6)
    assert errs[0][1] <= 1e-5


def test_fp8_rejections():
    with pytest.raises(spa.SpaError) as e:
        spa.Pool(1, 8, 2, 64, 8, device="cuda", kv_scale=np.ones((1, 2, 2), np.float32))
    assert e.value.status == spa.SPA_ERR_UNSUPPORTED
    rec = workloads.random_small(35, _model(1), max_prefix=100)
    inp = families.make_inputs(rec, "flat")
    gb = GpuBatch(inp, kv_scale=fp8_scales(inp))
    plan = spa.Plan(gb.pool, max_rows=128)
    plan.plan(gb.reqs)
    with pytest.raises(spa.SpaError) as e:
        gb.decode(plan, 0)
    assert e.value.status == spa.SPA_ERR_CUDA


@pytest.mark.parametrize("family", ["flat", "needle_shared_pos", "full_n1"])
def test_fp8_error_against_the_bf16_oracle(family):
    """FP8 pages change the inputs: report the error against the oracle on the bf16 K/V
     and bound it by the quantisation error itself plus the parity gate:
    |O_gpu - O_bf16| <= |O_deq - O_bf16| + 2e-2 elementwise, O_deq = the oracle on the
    dequantised K/V (oracle/fp8.py), likewise for the LSE with 1e-3."""
    rec = workloads.qwen(seed=3, n_agents=4)
    for g in rec.groups:
        g.prefix = 300 + g.prefix % 500
    rec.model = _model(1)
    inp = families.make_inputs(rec, family)
    sc = fp8_scales(inp)
    gb = GpuBatch(inp, kv_scale=sc)
    plan = spa.Plan(gb.pool, split_pages=4)
    plan.plan(gb.reqs)
    o, lse = gb.decode(plan, 0)
    O_bf, L_bf = Replay(inp).expected(0, inp.q[0])
    O_dq, L_dq = Replay(inp, kv_fp8_scale=sc).expected(0, inp.q[0])
    og = o.float().cpu().numpy().astype(np.float64)
    lg = lse.cpu().numpy().astype(np.float64)
    e_gpu, e_q = np.abs(og - O_bf), np.abs(O_dq - O_bf)
    assert (e_gpu <= e_q + O_TOL).all()
    assert (np.abs(lg - L_bf) <= np.abs(L_dq - L_bf) + LSE_TOL).all()
    print(f"\nfp8 vs bf16 oracle [{family}]: max|dO| {e_gpu.max():.4f} (quantisation alone {e_q.max():.4f}), "
          f"rms {np.sqrt((e_gpu ** 2).mean()):.5f}, max|dLSE| {np.abs(lg - L_bf).max():.4f}")
