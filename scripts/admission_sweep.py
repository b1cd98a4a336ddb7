"""Speculation-first vs FCFS decode-batch composition under a batch cap, on the real kernels.

    python scripts/admission_sweep.py [--agents 64] [--k 3] [--caps 32,64,128] [--out file.jsonl]

S8(f) F4 "SJF speculation-first batch composition in the bench's batch builder".
Queue: every agent's main request is already decoding (arrived first, "main agent
reasoning may decode hundreds" of tokens), then each agent's k speculative requests arrive
(forks of its context c_i).  With a cap of B requests per step, FCFS admits
the mains first; speculation-first (paper_2511_20048_b200/admission.py) admits the forks
first.  For each (cap, policy) the script plans and runs one decode step over 8 resident
layers (Qwen2.5-32B shape, contexts 2k-8k) and reports who was admitted, the unique KV
bytes per layer (forks of one agent share its prefix pages; a fork admitted without its
parent still reads the prefix once per group) and the measured per-layer time.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2511_20048_b200 import spa  # noqa: E402
from paper_2511_20048_b200.admission import Waiting, compose_batch  # noqa: E402
from spa_inputs import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--agents", type=int, default=64)
    ap.add_argument("--k", type=int, default=3)
    ap.add_argument("--caps", default="32,64,128")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    rng = np.random.default_rng(77)
    m = workloads.QWEN25_32B
    groups = [workloads.Group(int(rng.integers(2048, 8193)), int(rng.integers(0, 257)),
                              [16 + int(rng.integers(1, 11)) for _ in range(a.k)]) for _ in range(a.agents)]
    rec = workloads.Recipe("admission", m, groups, seed=77)
    Lr = 8
    pool = spa.Pool(Lr, m.num_q_heads, m.num_kv_heads, m.head_dim, bench.pages_for(rec, 8), device=dev)
    ids, reqs, batch = bench.build_batch(spa, pool, rec, list(range(Lr)), slice(0, m.num_kv_heads), dev, fill="reuse")
    # arrival: all mains, then the forks agent by agent
    mains = [nm for nm in batch if nm[1] == "main"]
    forks = [nm for nm in batch if nm[1] != "main"]
    waiting = [Waiting(nm, False, i) for i, nm in enumerate(mains)] + \
              [Waiting(nm, True, len(mains) + i) for i, nm in enumerate(forks)]
    q = torch.randn((len(batch), m.num_q_heads, m.head_dim), device=dev).to(torch.bfloat16)
    o = torch.empty_like(q)
    lse = torch.empty((len(batch), m.num_q_heads), dtype=torch.float32, device=dev)
    out = open(a.out, "a") if a.out else None
    for cap in [int(c) for c in a.caps.split(",")]:
        for policy in ("fcfs", "sjf"):
            names = compose_batch(waiting, cap, policy)
            sub = [ids[nm] for nm in names]
            plan = spa.Plan(pool)
            plan.plan(sub, stream=stream)
            N = len(sub)
            for _ in range(3):
                for li in range(Lr):
                    plan.decode(li, q[:N], o[:N], lse[:N], scale=m.softmax_scale, stream=stream)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 10
            e0.record(stream)
            for _ in range(reps):
                for li in range(Lr):
                    plan.decode(li, q[:N], o[:N], lse[:N], scale=m.softmax_scale, stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            layer_us = e0.elapsed_time(e1) * 1e3 / (reps * Lr)
            st = plan.stats()
            kv = st["alg_tokens"] * m.num_kv_heads * m.head_dim * 4
            row = {"cap": cap, "policy": policy, "admitted": N,
                   "speculative": sum(1 for nm in names if nm[1] != "main"),
                   "main": sum(1 for nm in names if nm[1] == "main"),
                   "groups": st["n_groups"], "kv_mb_per_layer": kv / 1e6, "layer_us": layer_us,
                   "tokens_per_s_64_layers": N / (64 * layer_us * 1e-6),
                   "gbs": bench.alg_bytes(st, N, m.num_kv_heads, m.num_q_heads, m.head_dim) / (layer_us * 1e-6) / 1e9}
            print(json.dumps(row), flush=True)
            if out:
                out.write(json.dumps(row) + "\n")
            plan.close()


if __name__ == "__main__":
    main()
