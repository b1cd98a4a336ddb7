"""Per-team streaming rate vs split size at B=1 (latency-floor study)."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
from paper_2511_20048_b200 import spa
from spa_inputs import KIND_Q, kv_bits_torch, workloads
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream)
m = workloads.QWEN25_32B
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
rec = workloads.sweep(B, 0.0)
Lr = 8
pool = spa.Pool(Lr, m.num_q_heads, m.num_kv_heads, m.head_dim, bench.pages_for(rec, 8), device=dev)
ids, reqs, batch = bench.build_batch(spa, pool, rec, list(range(Lr)), slice(0, m.num_kv_heads), dev, fill="reuse")
N = len(reqs)
q = kv_bits_torch(rec.seed, KIND_Q, 1, list(range(Lr)), np.arange(N), m.num_q_heads, m.head_dim, dev).contiguous()
o = torch.empty((N, m.num_q_heads, m.head_dim), dtype=torch.bfloat16, device=dev)
for sp in (4, 8, 16, 32, 64, 128, 400):
    for mode in (0, 2):
        plan = spa.Plan(pool, split_pages=sp, merge_mode=mode)
        plan.plan(reqs, 0, stream=stream)
        st = plan.stats()
        for i in range(5):
            plan.decode(i % Lr, q[i % Lr], o, None, scale=m.softmax_scale, stream=stream, want_lse=False)
        torch.cuda.synchronize()
        ts = []
        for rep in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for i in range(16):
                plan.decode(i % Lr, q[i % Lr], o, None, scale=m.softmax_scale, stream=stream, want_lse=False)
            e1.record(stream); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 16 * 1e3)
        print(f"B={B} split_pages={sp:4d} merge_mode={mode} items={st['n_items']:5d} records={st['n_records']:4d} "
              f"us/launch={np.median(ts):7.1f}", flush=True)
