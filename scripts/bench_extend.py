"""F2 measurement: shared-prefix extend attention (a mixed step where every agent's main
request decodes one token while its speculative fork prefills its 16-token prompt over the
shared context c_i, "prefill overhead is added once per speculative request").

    python scripts/bench_extend.py [--max-rows 64] [--n-query 16] [--reps 20] [--profile]

Workload: BJ config 1's batch (Qwen2.5-32B attention shape, 32 agents, contexts 2k-8k, one
fork each); the fork's last n_query tokens are query rows, the parent has one.  8 resident
layers (each far larger than L2), a measured "step" = 64 chained layer calls.  Prints one
JSON line: per-layer time, query rows/s, algorithmic HBM GB/s (shared prefix once per KV
head and group: the decode plan's unique keys) and FLOP/s against the measured peaks,
parity of sampled rows against the fp64 oracle, and the oracle's own CPU rate.
"""
from __future__ import annotations

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
from spa_inputs import KIND_K, KIND_Q, KIND_V, kv_bits_np, kv_bits_torch, workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-rows", type=int, default=64)
    ap.add_argument("--n-query", type=int, default=16)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--calls", type=int, default=64)
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--profile", action="store_true", help="profiler start/stop around 4 launches only")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    rec = workloads.qwen()
    m = rec.model
    Lr = a.layers
    layers = list(range(Lr))
    pool = spa.Pool(Lr, m.num_q_heads, m.num_kv_heads, m.head_dim, bench.pages_for(rec, 8), device=dev)
    ids, reqs, batch = bench.build_batch(spa, pool, rec, layers, slice(0, m.num_kv_heads), dev,
                                         fill="reuse" if a.profile else "hash")
    lens = [pool.page_table(r)[2] for r in reqs]
    nq = [1 if who == "main" else min(a.n_query, n) for (gi, who), n in zip(batch, lens)]
    rows = int(sum(nq))
    q = kv_bits_torch(rec.seed, KIND_Q, 3_000_000, layers, np.arange(rows), m.num_q_heads, m.head_dim, dev).contiguous()
    o = torch.empty((Lr, rows, m.num_q_heads, m.head_dim), dtype=torch.bfloat16, device=dev)
    lse = torch.empty((Lr, rows, m.num_q_heads), dtype=torch.float32, device=dev)
    plan = spa.Plan(pool, max_rows=a.max_rows)
    plan.plan(reqs, 0, stream=stream, n_query=nq)
    st = plan.stats()
    kv_alg_tokens = st["alg_tokens"]            # distinct attended keys: the sharing lower bound
    d = m.head_dim
    alg = kv_alg_tokens * m.num_kv_heads * d * 2 * 2 + rows * m.num_q_heads * (d * 2 * 2 + 4)
    plan_bytes = bench.alg_bytes(st, rows, m.num_kv_heads, m.num_q_heads, d, method=False)
    # flops: QK^T and PV over every row's live keys
    keys = 0
    for n, t in zip(lens, nq):
        keys += sum(n - t + j + 1 for j in range(t))
    flops = keys * m.num_q_heads * 4 * d

    def run(n):
        for i in range(n):
            plan.decode(i % Lr, q[i % Lr], o[i % Lr], lse[i % Lr], scale=m.softmax_scale, stream=stream)

    run(16)
    torch.cuda.synchronize()
    if a.profile:
        torch.cuda.profiler.start()
        run(4)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        return
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run(a.calls)
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / a.calls)
    layer_ms = float(np.median(ts))
    peaks, kind = bench.peaks()
    res = {"metric": "extend-attn query rows/s (mixed decode + speculative-prompt prefill step)",
           "value": rows / (layer_ms * 1e-3 * m.num_layers), "unit": "query rows/s",
           "config": {"workload": "BJ config 1 batch, forks prefill their last n_query tokens", "rows": rows,
                      "requests": len(reqs), "n_query_fork": a.n_query, "max_rows": a.max_rows,
                      "resident_layers": Lr, "calls_per_step": m.num_layers},
           "layer_us": layer_ms * 1e3, "stats": st,
           "alg_bytes": alg, "plan_bytes": plan_bytes, "flops": flops,
           "hbm_gbs_algorithmic": alg / (layer_ms * 1e-3) / 1e9,
           "hbm_gbs_plan": plan_bytes / (layer_ms * 1e-3) / 1e9,
           "tflops": flops / (layer_ms * 1e-3) / 1e12}
    res["roofline"] = {"bound": "hbm", "achieved": res["hbm_gbs_algorithmic"], "peak": peaks["hbm_gbs"],
                       "unit": "GB/s", "frac": res["hbm_gbs_algorithmic"] / peaks["hbm_gbs"], "peak_kind": kind,
                       "tensor_frac_of_bf16_peak": res["tflops"] / peaks["bf16_tflops"],
                       "intensity_flop_per_byte": flops / alg}
    # parity: group 0 (parent decode row + the fork's prompt rows) and group 13, layer 0
    if not a.no_parity:
        from oracle.attention import extend_attention
        from oracle.replay import bits_to_f64

        qb = kv_bits_np(rec.seed, KIND_Q, 3_000_000, [0], np.arange(rows), m.num_q_heads, d)[0]
        starts = np.concatenate([[0], np.cumsum(nq)])
        worst = [0.0, 0.0]
        t0 = time.perf_counter()
        checked = 0
        for i, (gi, who) in enumerate(batch):
            if gi not in (0, 13):
                continue
            K = bits_to_f64(bench.logical_kv_np(rec, gi, who, [0], KIND_K)[0])
            V = bits_to_f64(bench.logical_kv_np(rec, gi, who, [0], KIND_V)[0])
            r0, r1 = int(starts[i]), int(starts[i + 1])
            O, L = extend_attention(bits_to_f64(qb[r0:r1]), K, V, m.softmax_scale)
            og = o[0, r0:r1].float().cpu().numpy()
            lg = lse[0, r0:r1].cpu().numpy()
            worst[0] = max(worst[0], float(np.abs(og - O).max()))
            worst[1] = max(worst[1], float(np.abs(lg - L).max()))
            checked += r1 - r0
        res["parity"] = {"rows": checked, "max_abs_o": worst[0], "max_abs_lse": worst[1],
                         "pass": worst[0] <= 2e-2 and worst[1] <= 1e-3}
        # the oracle as it stands, on a bounded sample: whole requests at one layer
        t_or, done_rows = 0.0, 0
        t0 = time.perf_counter()
        for i, (gi, who) in enumerate(batch):
            K = bits_to_f64(bench.logical_kv_np(rec, gi, who, [0], KIND_K)[0])
            V = bits_to_f64(bench.logical_kv_np(rec, gi, who, [0], KIND_V)[0])
            r0, r1 = int(starts[i]), int(starts[i + 1])
            ts0 = time.perf_counter()
            extend_attention(bits_to_f64(qb[r0:r1]), K, V, m.softmax_scale)
            t_or += time.perf_counter() - ts0
            done_rows += r1 - r0
            if time.perf_counter() - t0 > a.cpu_seconds:
                break
        res["cpu_baseline"] = {"value": done_rows / (t_or * m.num_layers), "unit": "query rows/s",
                               "cores": os.cpu_count(), "kind": "oracle",
                               "sample": f"{done_rows} of {rows} rows x 1 layer, scaled to {m.num_layers} layers"}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
