"""Debug driver: build the Gemma-shaped batch and run each layer call with a sync + timing."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2511_20048_b200 import spa  # noqa: E402
from spa_inputs import KIND_Q, kv_bits_torch  # noqa: E402

T0 = time.time()


def log(*a):
    print(f"[{time.time() - T0:7.1f}s]", *a, file=sys.stderr, flush=True)


n_agents = int(sys.argv[1]) if len(sys.argv) > 1 else 64
Lr = int(sys.argv[2]) if len(sys.argv) > 2 else 2
mode = int(sys.argv[3]) if len(sys.argv) > 3 else 0
from spa_inputs import workloads  # noqa: E402

rec = workloads.gemma(2, n_agents=n_agents)
m = rec.model
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
pool = spa.Pool(Lr, m.num_q_heads, m.num_kv_heads, m.head_dim, bench.pages_for(rec, 8), device=dev)
log("pool", pool.num_pages)
ids, reqs, batch = bench.build_batch(spa, pool, rec, list(range(Lr)), slice(0, m.num_kv_heads), dev, fill="reuse")
log("built", len(reqs))
N = len(reqs)
q = kv_bits_torch(rec.seed, KIND_Q, 1, list(range(Lr)), np.arange(N), m.num_q_heads, m.head_dim, dev).contiguous()
for w in (1024, 0):
    plan = spa.Plan(pool, merge_mode=mode)
    plan.plan(reqs, w)
    torch.cuda.synchronize()
    log("plan", w, plan.stats())
    for li in range(Lr):
        t = time.time()
        o, l = plan.decode(li, q[li], scale=m.softmax_scale)
        torch.cuda.synchronize()
        log("decode", w, li, f"{(time.time() - t) * 1e3:.2f} ms", bool(torch.isfinite(o.float()).all()))
log("done")
# chained schedule (as in the bench step): local/global plans alternating, no syncs
plans = {w: spa.Plan(pool, merge_mode=mode) for w in (1024, 0)}
for w, p in plans.items():
    p.plan(reqs, w)
sched = bench.layer_schedule(rec, Lr)
o = torch.empty((len(sched), N, m.num_q_heads, m.head_dim), dtype=torch.bfloat16, device=dev)
for rep in range(3):
    t = time.time()
    for ci, (r, w) in enumerate(sched):
        plans[w].decode(r, q[r], o[ci], None, scale=m.softmax_scale, want_lse=False)
    torch.cuda.synchronize()
    log("chained step", rep, f"{(time.time() - t) * 1e3:.2f} ms")
log("chained done")
