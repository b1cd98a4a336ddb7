"""F1: the fused decode + peer-memory all-gather on one GPU.

The fused call (include/spa.h spa_decode_attention_fused_gather) stores each rank's head
outputs straight into every rank's gathered buffer and meets the peers through signal
flags.  Here `world` VIRTUAL ranks live in one process on one GPU
(spa_peer_connect_local): rank r holds KV heads [r Hkv/n, (r+1) Hkv/n) in its own pool
and runs on its own stream.  With the split plan held fixed, every rank's gathered
buffer must equal the unsharded decode bitwise ("gathered sharded
output == 1-GPU output with the split plan held fixed"), and the oracle within the
north_star tolerances.
"""
import pytest
import torch

from harness import LSE_TOL, O_TOL, GpuBatch, bits_to_torch, compare, fp8_scales
from oracle.replay import Replay
from paper_2511_20048_b200 import spa
from spa_inputs import families, workloads

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _need_gpu(cuda_device):
    spa.lib()
    yield


def _inputs(seed=3, layers=2):
    rec = workloads.qwen(seed=seed, n_agents=4)
    for g in rec.groups:
        g.prefix = 300 + g.prefix % 400
    rec.model = workloads.Model("q", layers, 40, 8, 128)
    return rec, families.make_inputs(rec, "needle_shared_pos")


def _shards(inp, n, merge_mode, kv_scale=None):
    shards = [GpuBatch(inp, shard=(r, n), kv_scale=kv_scale) for r in range(n)]
    plans = []
    for gb in shards:
        p = spa.Plan(gb.pool, split_pages=5, num_ctas=3, merge_mode=merge_mode)
        p.plan(gb.reqs)
        plans.append(p)
    return shards, plans


@pytest.mark.timeout(300, method="thread")
@pytest.mark.parametrize("n,merge_mode", [(1, 0), (2, 0), (4, 0), (8, 0), (2, 1)])
def test_fused_gather_virtual_ranks_bitwise(n, merge_mode):
    rec, inp = _inputs()
    full = GpuBatch(inp)
    plan = spa.Plan(full.pool, split_pages=5, num_ctas=7, merge_mode=merge_mode)
    plan.plan(full.reqs)
    refs = [full.decode(plan, li) for li in range(2)]
    N, Hq, d = refs[0][0].shape
    shards, plans = _shards(inp, n, merge_mode)
    peers = spa.Peer.local_world(n, spa.Peer.buffer_bytes(N, Hq, d), n_bufs=2)
    streams = [torch.cuda.Stream() for _ in range(n)]
    qs = [[bits_to_torch(inp.q[li][:, gb.q_sl]).contiguous() for gb in shards] for li in range(2)]
    torch.cuda.synchronize()
    # six calls queued back to back on every rank's stream (epochs 1..6, buffers alternating),
    # no host synchronisation in between: call k + 1 of a rank may start before its peers
    # have finished call k
    for step in range(6):
        li = step % 2
        for r in range(n):
            peers[r].decode(plans[r], li, qs[li][r], buf_idx=step % 2, scale=rec.model.softmax_scale,
                            stream=streams[r])
    torch.cuda.synchronize()
    for r in range(n):
        assert peers[r].status() == 0
        for b in range(2):   # buffer b holds the last call with step % 2 == b, i.e. layer b
            o, lse = peers[r].views(b, N, Hq, d)
            assert torch.equal(o.permute(1, 0, 2), refs[b][0]), (r, b)
            assert torch.equal(lse.t(), refs[b][1]), (r, b)
    rp = Replay(inp)
    for b in range(2):
        o, lse = peers[n - 1].views(b, N, Hq, d)
        O_ref, L_ref = rp.expected(b, inp.q[b])
        eo, el = compare(o.permute(1, 0, 2), lse.t(), O_ref, L_ref)
        assert eo <= O_TOL and el <= LSE_TOL, (eo, el)
    for p in peers:
        p.close()


@pytest.mark.timeout(120, method="thread")
def test_fused_gather_without_lse_and_rejections():
    rec, inp = _inputs(seed=4, layers=1)
    shards, plans = _shards(inp, 2, 0)
    N, Hq, d = len(shards[0].reqs), 40, 128
    peers = spa.Peer.local_world(2, spa.Peer.buffer_bytes(N, Hq, d, with_lse=False), n_bufs=1)
    # a buffer without room for the LSE refuses with_lse
    with pytest.raises(spa.SpaError) as e:
        peers[0].decode(plans[0], 0, bits_to_torch(inp.q[0][:, shards[0].q_sl]).contiguous(), 0, with_lse=True)
    assert e.value.status == spa.SPA_ERR_INVALID_ARG
    # the standalone merge kernel (merge_mode 2) and 128-row plans are not fused
    p2 = spa.Plan(shards[0].pool, split_pages=5, merge_mode=2)
    p2.plan(shards[0].reqs)
    with pytest.raises(spa.SpaError) as e:
        peers[0].decode(p2, 0, bits_to_torch(inp.q[0][:, shards[0].q_sl]).contiguous(), 0, with_lse=False)
    assert e.value.status == spa.SPA_ERR_UNSUPPORTED
    streams = [torch.cuda.Stream() for _ in range(2)]
    qs = [bits_to_torch(inp.q[0][:, gb.q_sl]).contiguous() for gb in shards]
    torch.cuda.synchronize()
    for r in range(2):
        peers[r].decode(plans[r], 0, qs[r], 0, with_lse=False, scale=rec.model.softmax_scale, stream=streams[r])
    torch.cuda.synchronize()
    ref = [shards[r].decode(plans[r], 0) for r in range(2)]
    for r in range(2):
        o, _ = peers[r].views(0, N, Hq, d)
        assert torch.equal(o.permute(1, 0, 2), torch.cat([ref[0][0], ref[1][0]], dim=1))
        assert peers[r].status() == 0


@pytest.mark.timeout(300, method="thread")
def test_fused_gather_fp8_pages_bitwise():
    """F1 x F4: head-sharded FP8 pools, fused gather == the unsharded FP8 decode, bitwise."""
    rec, inp = _inputs(seed=6)
    sc = fp8_scales(inp)
    full = GpuBatch(inp, kv_scale=sc)
    plan = spa.Plan(full.pool, split_pages=5, num_ctas=7)
    plan.plan(full.reqs)
    refs = [full.decode(plan, li) for li in range(2)]
    N, Hq, d = refs[0][0].shape
    n = 4
    shards, plans = _shards(inp, n, 0, kv_scale=sc)
    peers = spa.Peer.local_world(n, spa.Peer.buffer_bytes(N, Hq, d), n_bufs=2)
    streams = [torch.cuda.Stream() for _ in range(n)]
    qs = [[bits_to_torch(inp.q[li][:, gb.q_sl]).contiguous() for gb in shards] for li in range(2)]
    torch.cuda.synchronize()
    for step in range(2):
        for r in range(n):
            peers[r].decode(plans[r], step, qs[step][r], buf_idx=step, scale=rec.model.softmax_scale,
                            stream=streams[r])
    torch.cuda.synchronize()
    rp = Replay(inp, kv_fp8_scale=sc)
    for r in range(n):
        assert peers[r].status() == 0
        for b in range(2):
            o, lse = peers[r].views(b, N, Hq, d)
            assert torch.equal(o.permute(1, 0, 2), refs[b][0]) and torch.equal(lse.t(), refs[b][1])
    O_ref, L_ref = rp.expected(1, inp.q[1])
    o, lse = peers[0].views(1, N, Hq, d)
    eo, el = compare(o.permute(1, 0, 2), lse.t(), O_ref, L_ref)
    assert eo <= O_TOL and el <= LSE_TOL, (eo, el)
    for p in peers:
        p.close()
