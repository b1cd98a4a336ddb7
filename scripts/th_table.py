"""Measured attention share of the paper's hybrid-batch time T_h(P, N) on one B200 (S8(f) F3).

    python scripts/th_table.py [--out profiles/r01_th_table.csv]

T_h(P, N) (Table I, Eq. 3, Eq. 4) is the time of an engine step
that decodes N requests while prefilling a set P of prompts.  Under SPAgent, a selected
speculative request forks its agent's context c_i and prefills its L_s-token prompt over
it ("prefill overhead is added once per speculative request, since all samples of
one request share the same prefix").  This script measures the attention part of that
step on this library: N agents decode one token each (contexts 2k-8k, Qwen2.5-32B shape)
while |S| of them have a fork prefilling L_s tokens over the agent's shared pages.  One
layer = the agents with a prefilling fork as 128-row groups on the tcgen05 extend kernel
(parent decode row + fork prompt rows read c_i once) + the other agents on the decode
kernel; 64 PDL-chained layer calls (8 resident layers rotated, each far larger than L2).
Rows are written with the header SPEC.md's cost model reads
(`prefill_len,prefill_count,decode_count,seconds`), seconds = attention time of one
64-layer step.
"""
import argparse
import csv
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2511_20048_b200 import spa  # noqa: E402
from spa_inputs import KIND_Q, kv_bits_torch, workloads  # noqa: E402


def recipe(n_dec, n_spec, l_s, seed):
    rng = np.random.default_rng(seed)
    groups = []
    for a in range(n_dec):
        p = int(rng.integers(2048, 8193))
        groups.append(workloads.Group(p, int(rng.integers(0, 257)), [l_s] if a < n_spec else []))
    return workloads.Recipe(f"th_{n_dec}_{n_spec}_{l_s}", workloads.QWEN25_32B, groups, seed=seed)


def recipe_forks(n_dec, k, seed):
    """n_dec agents decoding, each with k speculative samples forked from its context c_i
    (PAPER.md:189 / :198) decoding too: their short tails (16-26 tokens) are all they read
    beyond the shared c_i."""
    rng = np.random.default_rng(seed)
    groups = []
    for _ in range(n_dec):
        p = int(rng.integers(2048, 8193))
        groups.append(workloads.Group(p, int(rng.integers(0, 257)), [16 + int(rng.integers(0, 11)) for _ in range(k)]))
    return workloads.Recipe(f"thf_{n_dec}_{k}", workloads.QWEN25_32B, groups, seed=seed)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_th_table.csv"))
    ap.add_argument("--decode", default="1,4,16,64,256")
    ap.add_argument("--spec", default="0,1,4,16")
    ap.add_argument("--ls", default="16,128,512")
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--calls", type=int, default=64)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--forks", default="1,3", help="samples per agent in the decode-with-forks rows (fork_count)")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    m = workloads.QWEN25_32B
    Lr = a.layers
    rows_out = []
    decs = [int(x) for x in a.decode.split(",")]
    specs = [int(x) for x in a.spec.split(",")]
    lss = [int(x) for x in a.ls.split(",")]
    forks = [int(x) for x in a.forks.split(",") if x]
    biggest = recipe(max(decs), min(max(specs), max(decs)), max(lss), 7)
    need = max(bench.pages_for(biggest, 40), bench.pages_for(recipe_forks(max(decs), max(forks + [0]), 7), 40))
    pool = spa.Pool(Lr, m.num_q_heads, m.num_kv_heads, m.head_dim, need, device=dev)
    for nd in decs:
        for ns in specs:
            if ns > nd:
                continue
            for ls in (lss if ns else [0]):
                rec = recipe(nd, ns, max(ls, 1), 1000 + nd * 31 + ns * 7 + ls)
                ids, reqs, batch = bench.build_batch(spa, pool, rec, list(range(Lr)), slice(0, m.num_kv_heads), dev,
                                                     fill="reuse")
                nq = [1 if who == "main" else ls for (gi, who) in batch]
                # the engine's composition: agents with a prefilling fork run as 128-row groups on
                # the tcgen05 extend kernel (parent + fork read c_i once); the other agents' decode
                # rows run on the decode kernel (a second launch per layer on the same stream)
                spec_groups = {gi for (gi, who) in batch if who != "main"}
                sel_x = [i for i, (gi, who) in enumerate(batch) if gi in spec_groups]
                sel_d = [i for i, (gi, who) in enumerate(batch) if gi not in spec_groups]
                launches = []
                for sel, ext in ((sel_x, True), (sel_d, False)):
                    if not sel:
                        continue
                    r_nq = [nq[i] for i in sel]
                    nrows = int(sum(r_nq))
                    qq = kv_bits_torch(rec.seed, KIND_Q, 1 + ext, list(range(Lr)), np.arange(nrows), m.num_q_heads,
                                       m.head_dim, dev).contiguous()
                    oo = torch.empty((Lr, nrows, m.num_q_heads, m.head_dim), dtype=torch.bfloat16, device=dev)
                    pl = spa.Plan(pool, max_rows=128 if ext else 16)
                    pl.plan([reqs[i] for i in sel], 0, stream=stream, n_query=r_nq if ext else None)
                    launches.append((pl, qq, oo))
                rows = int(sum(nq))

                def run(n):
                    for i in range(n):
                        for pl, qq, oo in launches:
                            pl.decode(i % Lr, qq[i % Lr], oo[i % Lr], None, scale=m.softmax_scale, stream=stream,
                                      want_lse=False)

                run(8)
                torch.cuda.synchronize()
                ts = []
                for _ in range(a.reps):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    run(a.calls)
                    e1.record(stream)
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1) / a.calls)
                layer_ms = float(np.median(ts))
                step_s = layer_ms * 1e-3 * m.num_layers
                rows_out.append((ls, ns, nd, step_s, 0))
                print(f"decode {nd:4d}  spec {ns:3d} x {ls:4d} tokens  rows {rows:5d}  layer {layer_ms * 1e3:8.1f} us  "
                      f"step {step_s * 1e3:7.2f} ms", flush=True)
                for nm in ids.values():
                    pool.free(nm)
    # decode batches with forked samples (fork_count column; reading F3-a): N agents + k N forks
    for nd in decs:
        for k in forks:
            rec = recipe_forks(nd, k, 5000 + nd * 13 + k)
            ids, reqs, batch = bench.build_batch(spa, pool, rec, list(range(Lr)), slice(0, m.num_kv_heads), dev,
                                                 fill="reuse")
            n = len(reqs)
            qq = kv_bits_torch(rec.seed, KIND_Q, 3, list(range(Lr)), np.arange(n), m.num_q_heads, m.head_dim,
                               dev).contiguous()
            oo = torch.empty((Lr, n, m.num_q_heads, m.head_dim), dtype=torch.bfloat16, device=dev)
            pl = spa.Plan(pool)
            pl.plan(reqs, 0, stream=stream)

            def runf(c):
                for i in range(c):
                    pl.decode(i % Lr, qq[i % Lr], oo[i % Lr], None, scale=m.softmax_scale, stream=stream,
                              want_lse=False)

            runf(8)
            torch.cuda.synchronize()
            ts = []
            for _ in range(a.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                runf(a.calls)
                e1.record(stream)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) / a.calls)
            layer_ms = float(np.median(ts))
            step_s = layer_ms * 1e-3 * m.num_layers
            rows_out.append((0, 0, nd, step_s, nd * k))
            print(f"decode {nd:4d} + {nd * k:4d} forks  layer {layer_ms * 1e3:8.1f} us  step {step_s * 1e3:7.2f} ms",
                  flush=True)
            for nm in ids.values():
                pool.free(nm)
    with open(a.out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["prefill_len", "prefill_count", "decode_count", "seconds", "fork_count"])
        for r in rows_out:
            w.writerow([r[0], r[1], r[2], f"{r[3]:.6e}", r[4]])


if __name__ == "__main__":
    main()
