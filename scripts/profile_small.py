"""Small-batch decode launches for ncu (latency floor study): B requests, fraction f."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2511_20048_b200 import spa  # noqa: E402
from spa_inputs import KIND_Q, kv_bits_torch, workloads  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
f = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
max_rows = int(sys.argv[3]) if len(sys.argv) > 3 else 16
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
m = workloads.QWEN25_32B
rec = workloads.sweep(B, f)
Lr = 8
pool = spa.Pool(Lr, m.num_q_heads, m.num_kv_heads, m.head_dim, bench.pages_for(rec, 8), device=dev)
ids, reqs, batch = bench.build_batch(spa, pool, rec, list(range(Lr)), slice(0, m.num_kv_heads), dev, fill="reuse")
N = len(reqs)
q = kv_bits_torch(rec.seed, KIND_Q, 1, list(range(Lr)), np.arange(N), m.num_q_heads, m.head_dim, dev).contiguous()
plan = spa.Plan(pool, max_rows=max_rows)
plan.plan(reqs, 0, stream=stream)
print(plan.stats(), file=sys.stderr)
o = torch.empty((N, m.num_q_heads, m.head_dim), dtype=torch.bfloat16, device=dev)
for i in range(10):
    plan.decode(i % Lr, q[i % Lr], o, None, scale=m.softmax_scale, stream=stream, want_lse=False)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for i in range(6):
    plan.decode(i % Lr, q[i % Lr], o, None, scale=m.softmax_scale, stream=stream, want_lse=False)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
