"""Host logic of the KV-head-sharded path, world_size 2 over gloo on CPU.

Every rank replays the same allocator calls on its own (metadata-only) pool holding its
head shard; page tables, refcounts and the step plan's structure must come out identical
on every rank without any communication, the head partition must
cover every head exactly once with each query head next to its KV head, and the
ncclUniqueId bytes travel rank 0 -> all through the process group.
"""
import hashlib
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_20048_b200 import spa
from spa_inputs import workloads


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _state_digest(pool, plan, reqs):
    h = hashlib.sha256()
    for r in reqs:
        h.update(repr(pool.page_table(r)).encode())
    h.update(repr(pool.refcounts()).encode())
    h.update(repr(pool.free_pages()).encode())
    for which in (0, 1, 5, 6):        # descriptors, members, pages, record CSR (head-independent)
        h.update(repr(plan.debug_array(which)).encode())
    return h.hexdigest()


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rec = workloads.qwen(seed=1, n_agents=6)
        m = rec.model
        q_sl, kv_sl = spa.shard_heads(m.num_q_heads, m.num_kv_heads, rank, world)
        pool = spa.Pool(m.num_layers, q_sl.stop - q_sl.start, kv_sl.stop - kv_sl.start, m.head_dim, 4000)
        ops, batch = workloads.call_log(rec)
        ids = {}
        for op in ops:
            if op[0] == "alloc":
                ids[op[1]] = pool.alloc()
            elif op[0] == "append":
                pool.append([ids[op[1]]], [op[4]])
            elif op[0] == "fork":
                ids[op[1]] = pool.fork(ids[op[2]], op[3])
        reqs = [ids[n] for n in batch]
        for _ in range(3):                        # decode steps: append one token each
            pool.append(reqs, [1] * len(reqs))
        plan = spa.Plan(pool, split_pages=16, num_ctas=8)
        plan.plan(reqs)
        digests = [None] * world
        dist.all_gather_object(digests, _state_digest(pool, plan, reqs))
        # a windowed (local-layer) step after spa_kv_release_window replicates as well
        pool.append(reqs, [1] * len(reqs))
        pool.release_window(list(ids.values()), 1024)
        plan.plan(reqs, 1024)
        wdig = [None] * world
        dist.all_gather_object(wdig, _state_digest(pool, plan, reqs))
        digests = [a + b for a, b in zip(digests, wdig)]
        uid = [spa.spa_nccl_unique_id() if rank == 0 else None]   # the real NCCL bootstrap id (no GPU needed)
        dist.broadcast_object_list(uid, src=0)
        uids = [None] * world
        dist.all_gather_object(uids, uid[0])
        slices = [None] * world
        dist.all_gather_object(slices, (q_sl.start, q_sl.stop, kv_sl.start, kv_sl.stop))
        q.put((rank, digests, uids, slices))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_replicated_allocator_and_plan(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, digests, uids, slices in res:
        assert len(set(digests)) == 1, "allocator/plan state diverged across ranks"
        assert len(set(uids)) == 1 and len(uids[0]) == 128
    _, _, _, slices = res[0]
    G = 5
    qs = sorted(h for a, b, _, _ in slices for h in range(a, b))
    ks = sorted(h for _, _, a, b in slices for h in range(a, b))
    assert qs == list(range(40)) and ks == list(range(8))
    for a, b, c, d in slices:
        assert all(c <= h // G < d for h in range(a, b))


def test_shard_heads_rejects_bad_worlds():
    with pytest.raises(ValueError):
        spa.shard_heads(40, 8, 0, 3)
    assert spa.shard_heads(32, 16, 7, 8) == (slice(28, 32), slice(14, 16))
