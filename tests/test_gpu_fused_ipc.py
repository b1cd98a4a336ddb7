"""F1 across PROCESSES: the fused decode + peer-memory all-gather wired through CUDA IPC.

Two processes (gloo group for the 64-byte IPC handles, as bench.py does over its process
group) share ONE GPU: each is a rank holding half the KV heads in its own pool, maps the
other's region with cudaIpcOpenMemHandle (spa_peer_connect) and runs the fused call.
The contexts time-slice on the device, so each rank's last CTA waits for the other
process's kernel to be scheduled; the result must still equal the unsharded decode
bitwise (fixed split plan).  This exercises the real multi-GPU wiring (IPC mapping,
system-scope flags between processes) on the single GPU the test box has.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from harness import GpuBatch, bits_to_torch
        from paper_2511_20048_b200 import spa
        from spa_inputs import families, workloads

        torch.cuda.set_device(0)
        rec = workloads.qwen(seed=5, n_agents=3)
        for g in rec.groups:
            g.prefix = 200 + g.prefix % 300
        rec.model = workloads.Model("q", 2, 40, 8, 128)
        inp = families.make_inputs(rec, "needle_shared_pos")
        full = GpuBatch(inp)
        plan = spa.Plan(full.pool, split_pages=4, num_ctas=5)
        plan.plan(full.reqs)
        refs = [full.decode(plan, li) for li in range(2)]
        N, Hq, d = refs[0][0].shape
        gb = GpuBatch(inp, shard=(rank, world))
        p = spa.Plan(gb.pool, split_pages=4, num_ctas=2)
        p.plan(gb.reqs)
        peer = spa.Peer(rank, world, spa.Peer.buffer_bytes(N, Hq, d), n_bufs=2)
        qs = [bits_to_torch(inp.q[li][:, gb.q_sl]).contiguous() for li in range(2)]
        torch.cuda.synchronize()
        dist.barrier()
        for step in range(4):
            peer.decode(p, step % 2, qs[step % 2], buf_idx=step % 2, scale=rec.model.softmax_scale)
        torch.cuda.synchronize()
        ok = peer.status() == 0
        for b in range(2):
            o, lse = peer.views(b, N, Hq, d)
            ok = ok and torch.equal(o.permute(1, 0, 2), refs[b][0]) and torch.equal(lse.t(), refs[b][1])
        dist.barrier()        # the peer's mapping of our region is closed before we free it
        peer.close()
        dist.barrier()
        q.put((rank, bool(ok), ""))
    except Exception as e:  # noqa: BLE001
        q.put((rank, False, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300, method="thread")
def test_fused_gather_two_processes_one_gpu(cuda_device):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=280) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
