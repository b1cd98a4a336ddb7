"""BJ config 3: engine-load sweep (batch 1-256, speculative fraction 0-100 %, Qwen shape, 1 GPU).

The decode-attention share of the paper's T_h(emptyset, N) (Eq. 3): how the
per-step attention time grows with the number of decode requests N and with the fraction of
them that are speculative forks of another request's context -- with prefix sharing (this
library's default) and without it (every request alone, the control).

    python scripts/sweep_load.py [--out profiles/r01_sweep.jsonl] [--batches 1,2,...] [--fracs 0,0.25,...]

KV values are appended from one reused chunk (timing does not depend on the values; parity
is covered by tests/ and the bench gate).  8 resident layers; a step = 64 chained layer
calls (call i reads resident layer i % 8).
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2511_20048_b200 import spa  # noqa: E402
from spa_inputs import KIND_Q, kv_bits_torch, workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "sweep_load.jsonl"))
    ap.add_argument("--batches", default="1,2,4,8,16,32,64,128,256")
    ap.add_argument("--fracs", default="0,0.25,0.5,0.75,1")
    ap.add_argument("--resident", type=int, default=8)
    ap.add_argument("--calls", type=int, default=64)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--plans", default="", help="comma list of plan keys to run (default: all)")
    a = ap.parse_args()
    batches = [int(x) for x in a.batches.split(",")]
    fracs = [float(x) for x in a.fracs.split(",")]
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    m = workloads.QWEN25_32B
    Lr = a.resident
    # one pool for every point: sized for the largest batch
    pages = max(bench.pages_for(workloads.sweep(b, f), 8) for b in batches for f in fracs)
    pool = spa.Pool(Lr, m.num_q_heads, m.num_kv_heads, m.head_dim, pages, device=dev)
    # shared: the library default (max_rows 0: 16- or 32-row items chosen per batch)
    plans = {"shared": spa.Plan(pool), "shared16": spa.Plan(pool, max_rows=16),
             "shared32": spa.Plan(pool, max_rows=32), "unshared": spa.Plan(pool, sharing=False)}
    if a.plans:
        plans = {k: v for k, v in plans.items() if k in a.plans.split(",")}
    rows = []
    out = open(a.out, "w")
    for b in batches:
        for f in fracs:
            rec = workloads.sweep(b, f)
            rec.model = m
            ids, reqs, batch = bench.build_batch(spa, pool, rec, list(range(Lr)), slice(0, m.num_kv_heads), dev,
                                                 fill="reuse")
            N = len(reqs)
            q = kv_bits_torch(rec.seed, KIND_Q, 1, list(range(Lr)), np.arange(N), m.num_q_heads, m.head_dim,
                              dev).contiguous()
            o = torch.empty((Lr, N, m.num_q_heads, m.head_dim), dtype=torch.bfloat16, device=dev)
            lse = torch.empty((Lr, N, m.num_q_heads), dtype=torch.float32, device=dev)
            rec_row = {"B": b, "f": f, "N": N}
            for key, plan in plans.items():
                plan.plan(reqs, 0, stream=stream)
                st = plan.stats()
                for _ in range(2):   # warm-up
                    for i in range(a.calls):
                        plan.decode(i % Lr, q[i % Lr], o[i % Lr], lse[i % Lr], scale=m.softmax_scale, stream=stream)
                torch.cuda.synchronize()
                ts = []
                for _ in range(a.reps):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    for i in range(a.calls):
                        plan.decode(i % Lr, q[i % Lr], o[i % Lr], lse[i % Lr], scale=m.softmax_scale, stream=stream)
                    e1.record(stream)
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1) / a.calls)
                layer_ms = float(np.median(ts))
                ab = bench.alg_bytes(st, N, m.num_kv_heads, m.num_q_heads, m.head_dim)   # method bytes (B_alg)
                rec_row[key] = {"layer_us": layer_ms * 1e3, "attn_ms_per_step": layer_ms * m.num_layers,
                                "tokens_per_s": N / (layer_ms * 1e-3 * m.num_layers),
                                "alg_gbs": ab / (layer_ms * 1e-3) / 1e9, "alg_tokens_per_head": st["alg_tokens"],
                                "read_tokens_per_head": st["unique_tokens"],
                                "overhead_bytes": bench.overhead_bytes(st, m.num_kv_heads, m.num_q_heads, m.head_dim),
                                "records": st["n_records"], "rows_max": st["rows_max"]}
            rows.append(rec_row)
            out.write(json.dumps(rec_row) + "\n")
            out.flush()
            print(f"B={b:4d} f={f:4.2f} N={N:4d} " + " | ".join(
                f"{k} {v['layer_us']:7.1f} us {v['tokens_per_s']:7.0f} tok/s {v['alg_gbs']:5.0f} GB/s"
                for k, v in rec_row.items() if isinstance(v, dict)), flush=True)
            for nm in ids.values():   # release the batch (and the parents of forks)
                pool.free(nm)
    out.close()


if __name__ == "__main__":
    main()
