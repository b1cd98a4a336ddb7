"""Timeline of one decode launch (spa_debug_set_trace): where a launch's time goes.

    python scripts/trace_timeline.py [qwen | sweep:B:f | long | gemma] [--window W] [--teams N] [--split P] [--out file.json]

Runs the workload PDL-chained over 8 resident layers (as the bench chains layer calls),
traces the last launch and prints: entry spread, ramp (first item start per team), busy
fraction, the drain (teams finishing their last item), the tail-merge window, and the
CUDA-graph per-launch time (no host submission in it) next to the eager chained time and
the host-side cost of one decode call.
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


def team_rates(tr, item_pages, warps_per_cta):
    """Per team (first warp of each pair): pages streamed / busy time; summary by CTA and team slot."""
    tr = tr.cpu().numpy().astype(np.uint64)
    gt = tr[:, :, 0].astype(np.int64)
    w1 = tr[:, :, 1]
    tag = (w1 >> np.uint64(56)).astype(np.int64)
    ids = ((w1 >> np.uint64(32)) & np.uint64(0xFFFFFF)).astype(np.int64)
    rates, slots, ctas, busy = [], [], [], []
    for w in range(0, tr.shape[0], 2):
        st, en = gt[w][tag[w] == 2], gt[w][tag[w] == 3]
        its = ids[w][tag[w] == 2]
        if len(st) == 0 or len(en) != len(st):
            continue
        pages = sum(item_pages[i] for i in its)
        b = float((en - st).sum()) / 1e3
        rates.append(pages / b if b > 0 else 0)
        busy.append(b)
        slots.append((w % warps_per_cta) // 2)
        ctas.append(w // warps_per_cta)
    gaps = []
    for w in range(0, tr.shape[0], 2):
        st, en = gt[w][tag[w] == 2], gt[w][tag[w] == 3]
        if len(st) > 1 and len(en) == len(st):
            gaps.extend(((st[1:] - en[:-1]) / 1e3).tolist())
    rates, slots, ctas = np.array(rates), np.array(slots), np.array(ctas)
    out = {"pages_per_us": [float(np.percentile(rates, p)) for p in (0, 10, 50, 90, 100)],
           "by_slot": [float(rates[slots == k].mean()) for k in range(int(slots.max()) + 1)],
           "gap_us": [float(np.percentile(gaps, p)) for p in (0, 50, 90, 100)] if gaps else None,
           "gaps_per_team": len(gaps) / max(1, len(rates))}
    per_cta = np.array([rates[ctas == c].mean() for c in np.unique(ctas)])
    out["cta_mean_pages_per_us"] = [float(np.percentile(per_cta, p)) for p in (0, 10, 50, 90, 100)]
    out["cta_rate_by_parity"] = [float(per_cta[0::2].mean()), float(per_cta[1::2].mean())]
    return out


def analyse(tr, n_items_cost=None):
    tr = tr.cpu().numpy().astype(np.uint64)
    gt = tr[:, :, 0].astype(np.int64)
    w1 = tr[:, :, 1]
    tag = (w1 >> np.uint64(56)).astype(np.int64)
    ids = ((w1 >> np.uint64(32)) & np.uint64(0xFFFFFF)).astype(np.int64)
    valid = tag > 0
    t0 = gt[valid].min()
    rel = (gt - t0) / 1e3   # us
    out = {}
    ent = rel[tag == 1]
    ext = rel[tag == 6]
    out["entry_us"] = [float(ent.min()), float(np.median(ent)), float(ent.max())]
    out["exit_us"] = [float(ext.min()), float(np.median(ext)), float(ext.max())]
    first_start, last_end, busy = [], [], []
    for t in range(tr.shape[0]):
        s = rel[t][tag[t] == 2]
        e = rel[t][tag[t] == 3]
        if len(s):
            first_start.append(s.min())
            last_end.append(e.max())
            busy.append(float((e - s[: len(e)]).sum()))
    fs, le = np.array(first_start), np.array(last_end)
    span = float(ext.max() - ent.min())
    out["span_us"] = span
    out["teams_with_items"] = int(len(fs))
    out["first_item_start_us"] = [float(np.percentile(fs, p)) for p in (0, 50, 90, 100)] if len(fs) else None
    out["last_item_end_us"] = [float(np.percentile(le, p)) for p in (0, 10, 50, 90, 100)] if len(le) else None
    out["busy_frac"] = float(np.sum(busy) / (tr.shape[0] * span)) if span > 0 else None
    ms = rel[tag == 4]
    me = rel[tag == 5]
    out["merge_tasks"] = int(len(ms))
    out["merge_us"] = [float(ms.min()), float(me.max())] if len(ms) else None
    if len(ms):
        # per merge subtask of the traced warps: pop time and duration (pop -> merged)
        pops, durs, waits = [], [], []
        for t in range(tr.shape[0]):
            tg = tag[t]
            for k in np.nonzero(tg == 4)[0]:
                if k + 2 < len(tg) and tg[k + 1] == 7 and tg[k + 2] == 5:
                    pops.append(rel[t][k])
                    waits.append(rel[t][k + 1] - rel[t][k])
                    durs.append(rel[t][k + 2] - rel[t][k + 1])
        pops, durs = np.array(pops), np.array(durs)
        out["merge_pop_us"] = [float(np.percentile(pops, p)) for p in (0, 50, 90, 100)]
        out["merge_dur_us"] = [float(np.percentile(durs, p)) for p in (0, 50, 90, 100)]
        out["merge_wait_us"] = [float(np.percentile(waits, p)) for p in (0, 50, 90, 100)]
        ends = pops + np.array(waits) + durs
        out["merge_end_us"] = [float(np.percentile(ends, p)) for p in (0, 50, 90, 99, 100)]
    cnt = rel[tag == 8]
    if len(cnt):
        # item end (tag 3) -> its records counted in (tag 8)
        d38 = []
        for t in range(tr.shape[0]):
            tg = tag[t]
            for k in np.nonzero(tg == 8)[0]:
                if k > 0 and tg[k - 1] == 3:
                    d38.append(rel[t][k] - rel[t][k - 1])
        out["count_lag_us"] = [float(np.percentile(d38, p)) for p in (0, 50, 90, 100)] if d38 else None
    nsub = np.array([(tag[t] == 4).sum() for t in range(tr.shape[0])])
    out["subtasks_per_warp_even_odd"] = [float(nsub[0::2].mean()), float(nsub[1::2].mean())]
    tin = np.array([rel[t][tag[t] == 4].min() if (tag[t] == 4).any() else np.nan for t in range(tr.shape[0])])
    out["tail_entry_even_odd_us"] = [float(np.nanmedian(tin[0::2])), float(np.nanmedian(tin[1::2]))]
    out["items_per_team"] = [int(x) for x in np.percentile([(tag[t] == 2).sum() for t in range(tr.shape[0])],
                                                            [0, 50, 100])]
    # per-item phases of every traced warp: start (2) -> row setup landed (9) -> pages done (10)
    # -> epilogue done (3); record-count fence (11 -> 8)
    ph = {"setup": [], "pages": [], "epilogue": [], "count_fence": []}
    for t in range(tr.shape[0]):
        tg, tt = tag[t], rel[t]
        for k in range(len(tg)):
            if tg[k] == 2 and k + 3 < len(tg):
                seq = {}
                for j in range(k + 1, min(len(tg), k + 8)):
                    if tg[j] in (9, 10, 3) and tg[j] not in seq:
                        seq[tg[j]] = tt[j]
                    if tg[j] == 3:
                        break
                if 9 in seq and 10 in seq and 3 in seq:
                    ph["setup"].append(seq[9] - tt[k])
                    ph["pages"].append(seq[10] - seq[9])
                    ph["epilogue"].append(seq[3] - seq[10])
            if tg[k] == 11 and k + 1 < len(tg) and tg[k + 1] == 8:
                ph["count_fence"].append(tt[k + 1] - tt[k])
            if tg[k] == 10 and k + 1 < len(tg) and tg[k + 1] == 13:
                ph["epi_publish"] = ph.get("epi_publish", []) + [tt[k + 1] - tt[k]]
            if tg[k] == 13 and k + 1 < len(tg) and tg[k + 1] == 14:
                ph["epi_pair_wait"] = ph.get("epi_pair_wait", []) + [tt[k + 1] - tt[k]]
            if tg[k] == 14 and k + 1 < len(tg) and tg[k + 1] == 15:
                ph["epi_gather"] = ph.get("epi_gather", []) + [tt[k + 1] - tt[k]]
            if tg[k] == 15 and k + 1 < len(tg) and tg[k + 1] == 3:
                ph["epi_store"] = ph.get("epi_store", []) + [tt[k + 1] - tt[k]]
    out["item_phases_us"] = {k: ([float(np.percentile(v, q)) for q in (10, 50, 90)] + [float(np.sum(v) / tr.shape[0])])
                             for k, v in ph.items() if v}   # p10, p50, p90, total per warp
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload", nargs="?", default="qwen")
    ap.add_argument("--teams", type=int, default=0)
    ap.add_argument("--split", type=int, default=0)
    ap.add_argument("--merge", type=int, default=0)
    ap.add_argument("--out", default=None)
    ap.add_argument("--kv", default="bf16", choices=["bf16", "fp8"])
    ap.add_argument("--rows", type=int, default=16, help="plan max_rows (0 auto, 16, 32, 64)")
    ap.add_argument("--window", type=int, default=0, help="sliding window (gemma local layers: 1024)")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    if a.workload == "qwen":
        rec = workloads.qwen()
    elif a.workload == "long":
        rec = workloads.long32k()
    elif a.workload == "gemma":
        rec = workloads.gemma()
    else:
        _, b, f = a.workload.split(":")
        rec = workloads.sweep(int(b), float(f))
    m = rec.model
    Lr = 8 if a.workload != "long" else 2
    fp8 = a.kv == "fp8"
    pool = spa.Pool(Lr, m.num_q_heads, m.num_kv_heads, m.head_dim, bench.pages_for(rec, 8), device=dev,
                    kv_scale=np.full((Lr, m.num_kv_heads, 2), bench.FP8_SCALE, np.float32) if fp8 else None)
    ids, reqs, batch = bench.build_batch(spa, pool, rec, list(range(Lr)), slice(0, m.num_kv_heads), dev, fill="reuse")
    N = len(reqs)
    q = kv_bits_torch(rec.seed, KIND_Q, 1, list(range(Lr)), np.arange(N), m.num_q_heads, m.head_dim, dev).contiguous()
    o = torch.empty((Lr, N, m.num_q_heads, m.head_dim), dtype=torch.bfloat16, device=dev)
    lse = torch.empty((Lr, N, m.num_q_heads), dtype=torch.float32, device=dev)
    plan = spa.Plan(pool, split_pages=a.split, merge_mode=a.merge, teams_per_cta=a.teams, max_rows=a.rows)
    plan.plan(reqs, a.window, stream=stream)
    st = plan.stats()

    def run(n):
        for i in range(n):
            plan.decode(i % Lr, q[i % Lr], o[i % Lr], lse[i % Lr], scale=m.softmax_scale, stream=stream)

    run(16)
    torch.cuda.synchronize()
    # eager chained per-launch time and host cost per call
    calls = 64
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    h0 = time.perf_counter()
    run(calls)
    h1 = time.perf_counter()
    e1.record(stream)
    torch.cuda.synchronize()
    eager_us = e0.elapsed_time(e1) / calls * 1e3
    host_us = (h1 - h0) / calls * 1e6
    # CUDA graph of `calls` chained launches (the plan's launch counter advances in capture)
    g = torch.cuda.CUDAGraph()
    plan.plan(reqs, a.window, stream=stream)
    with torch.cuda.graph(g, stream=stream):
        run(calls)
    graph_us = []
    for _ in range(5):
        plan.plan(reqs, a.window, stream=stream)   # resets the launch ids the graph was captured with
        torch.cuda.synchronize()
        e0.record(stream)
        g.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        graph_us.append(e0.elapsed_time(e1) / calls * 1e3)
    # trace the last of 8 chained launches
    plan.plan(reqs, a.window, stream=stream)
    run(7)
    buf = plan.set_trace(256)   # zeroed on the stream; the traced launch follows 7 chained ones
    plan.decode(7 % Lr, q[7 % Lr], o[7 % Lr], lse[7 % Lr], scale=m.softmax_scale, stream=stream)
    torch.cuda.synchronize()
    res = {"workload": a.workload, "rows": a.rows, "N": N, "stats": st, "eager_chained_us": eager_us,
           "graph_chained_us": float(np.median(graph_us)), "host_us_per_call": host_us,
           "alg_bytes": bench.alg_bytes(st, N, m.num_kv_heads, m.num_q_heads, m.head_dim, 1 if fp8 else 2), "kv": a.kv}
    res["trace"] = analyse(buf)
    descs = plan.debug_array(0)
    items = plan.debug_array(2)
    item_pages = [descs[d][1] for d, _ in items]
    res["rates"] = team_rates(buf, item_pages, buf.shape[0] // plan.num_ctas_hint())
    res["graph_gbs"] = res["alg_bytes"] / (res["graph_chained_us"] * 1e-6) / 1e9
    res["overhead_bytes"] = bench.overhead_bytes(st, m.num_kv_heads, m.num_q_heads, m.head_dim, 1 if fp8 else 2)
    plan.set_trace(0)
    print(json.dumps(res), flush=True)
    if a.out:
        with open(a.out, "a") as f:
            f.write(json.dumps(res) + "\n")


if __name__ == "__main__":
    main()
