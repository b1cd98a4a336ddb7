"""Timeline of the tcgen05 extend kernel (CTA 0) on the mixed BJ-config-1 step: where a
CTA's time goes (per-stage waits, item transitions, epilogue), from the kernel's trace
points (spa_debug_set_trace; tags in csrc/ext.cu)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2511_20048_b200 import spa  # noqa: E402
from spa_inputs import KIND_Q, kv_bits_torch, workloads  # noqa: E402

NAMES = {10: "P issue", 11: "P rows", 12: "P K-issued", 13: "P V-free", 20: "M kfull", 21: "M S-issued", 22: "M item", 23: "M qready", 24: "M P-ready", 25: "M V-ready", 26: "M PV-issued", 30: "W sfull",
         31: "W pfull-arr", 32: "W item", 33: "W q-written", 34: "W epi-wait", 35: "W ofull", 36: "W item-done", 37: "W S-loaded", 38: "W max-done", 39: "W exp-done", 40: "W O-rescaled", 41: "W max-only", 50: "V merge-ready", 51: "W tail-merge", 52: "merge-done"}


def main():
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    rec = workloads.qwen()
    m = rec.model
    Lr = 2
    pool = spa.Pool(Lr, m.num_q_heads, m.num_kv_heads, m.head_dim, bench.pages_for(rec, 8), device=dev)
    ids, reqs, batch = bench.build_batch(spa, pool, rec, list(range(Lr)), slice(0, m.num_kv_heads), dev, fill="reuse")
    nq = [1 if who == "main" else 16 for (gi, who) in batch]
    rows = sum(nq)
    q = kv_bits_torch(rec.seed, KIND_Q, 3_000_000, list(range(Lr)), np.arange(rows), m.num_q_heads, m.head_dim,
                      dev).contiguous()
    o = torch.empty((rows, m.num_q_heads, m.head_dim), dtype=torch.bfloat16, device=dev)
    plan = spa.Plan(pool, max_rows=128)
    plan.plan(reqs, 0, stream=stream, n_query=nq)
    for i in range(4):
        plan.decode(i % Lr, q[i % Lr], o, None, scale=m.softmax_scale, stream=stream, want_lse=False)
    torch.cuda.synchronize()
    cap = 2048
    buf = torch.zeros((8, cap, 2), dtype=torch.int64, device=dev)
    spa.lib().spa_debug_set_trace(plan.h, spa._ptr(buf), cap)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    plan.decode(0, q[0], o, None, scale=m.softmax_scale, stream=stream, want_lse=False)
    e1.record(stream)
    torch.cuda.synchronize()
    spa.lib().spa_debug_set_trace(plan.h, None, 0)
    tr = buf.cpu().numpy().astype(np.uint64)
    ev = []
    for w in range(5):
        for k in range(cap):
            w1 = tr[w, k, 1]
            tag = int(w1 >> np.uint64(56))
            if tag == 0:
                break
            ev.append((int(tr[w, k, 0]), w, tag, int((w1 >> np.uint64(32)) & np.uint64(0xffffff))))
    ev.sort()
    t0 = ev[0][0]
    se = tr[7, :, :].astype(np.int64)
    print("row 7 nonzero:", int((se != 0).sum()), se[:2].tolist())
    se = se[(se[:, 0] > 0) & (se[:, 1] > 0)]
    if len(se):
        s0 = se[:, 0].min()
        st_, en_ = (se[:, 0] - s0) / 1e3, (se[:, 1] - s0) / 1e3
        print(f"CTAs {len(se)}: start spread {st_.max():.1f} us; end min {en_.min():.1f} median {np.median(en_):.1f} "
              f"p90 {np.percentile(en_, 90):.1f} max {en_.max():.1f} us; busy fraction {(en_ - st_).sum() / (len(se) * en_.max()):.3f}")
    span = (ev[-1][0] - t0) / 1e3
    print(f"launch (events) {e0.elapsed_time(e1) * 1e3:.1f} us; CTA 0 trace span {span:.1f} us, {len(ev)} events")
    by = {}
    for t, w, tag, i in ev:
        by.setdefault(tag, []).append((t, i))
    n_items = len(by.get(22, []))
    n_st = len(by.get(21, []))
    print(f"CTA 0: {n_items} items, {n_st} stages, {span / max(n_st, 1) * 1e3:.0f} ns per stage overall")

    def pair_sum(a, b):   # sum of (b_k - a_k) over matched k-th occurrences
        A, B = by.get(a, []), by.get(b, [])
        k = min(len(A), len(B))
        return sum(B[j][0] - A[j][0] for j in range(k)) / 1e3, k

    for a, b, what in ((22, 23, "MMA waits for the next item's Q tile (QREADY)"),
                       (32, 33, "WG item setup (member rows, Q tile load + write)"),
                       (34, 35, "WG waits for the item's last PV (OFULL)"),
                       (35, 36, "WG epilogue (merge halves, write O / partials)")):
        s, k = pair_sum(a, b)
        print(f"  {what}: total {s:.1f} us over {k}")
    # MMA: time blocked on K data (from the previous MMA event to 'M kfull')
    mma = [(t, tag, i) for t, w, tag, i in ev if w == 1]
    wait_k = 0.0
    for j in range(1, len(mma)):
        if mma[j][1] == 20:
            wait_k += (mma[j][0] - mma[j - 1][0]) / 1e3
    print(f"  S issuer: time between its previous event and each K-full wake: {wait_k:.1f} us")
    iss = [t for t, tag, i in mma if tag == 10]
    P = [t for t, w, tag, i in ev if w == 0 and tag == 10]
    K = [t for t, w, tag, i in ev if w == 1 and tag == 20]
    k = min(len(P), len(K))
    lat = np.array([K[j] - P[j] for j in range(k)]) / 1e3
    if k:
        print(f"  producer issue -> MMA sees K: median {np.median(lat):.2f} us, p90 {np.percentile(lat, 90):.2f} us")
    pe = [(t, tag) for t, w, tag, i in ev if w == 0]
    seg = {}
    for j in range(1, len(pe)):
        key = (pe[j - 1][1], pe[j][1])
        seg.setdefault(key, []).append(pe[j][0] - pe[j - 1][0])
    for key, v in sorted(seg.items()):
        print(f"  producer {NAMES.get(key[0])} -> {NAMES.get(key[1])}: n {len(v)} median {np.median(v):.0f} ns")
    for wi, who in ((1, "S issuer"), (3, "PV issuer")):
        me = [(t, tag) for t, w, tag, i in ev if w == wi]
        seg = {}
        for j in range(1, len(me)):
            key = (me[j - 1][1], me[j][1])
            seg.setdefault(key, []).append(me[j][0] - me[j - 1][0])
        for key, v in sorted(seg.items()):
            print(f"  {who} {NAMES.get(key[0])} -> {NAMES.get(key[1])}: n {len(v)} median {np.median(v):.0f} ns, "
                  f"total {sum(v) / 1e3:.1f} us")
    we = [(t, tag) for t, w, tag, i in ev if w == 2]
    seg = {}
    for j in range(1, len(we)):
        key = (we[j - 1][1], we[j][1])
        seg.setdefault(key, []).append(we[j][0] - we[j - 1][0])
    for key, v in sorted(seg.items()):
        print(f"  WG0 {NAMES.get(key[0])} -> {NAMES.get(key[1])}: n {len(v)} median {np.median(v):.0f} ns, "
              f"total {sum(v) / 1e3:.1f} us")
    for tag, who in ((50, "V producer merges (ready tasks)"), (51, "WG0 warp tail merges")):
        ts = [t for t, w, tg, i in ev if tg == tag]
        if ts:
            print(f"  {who}: {len(ts)} from {(ts[0] - t0) / 1e3:.1f} to {(ts[-1] - t0) / 1e3:.1f} us")
    print("first 60 events:")
    for t, w, tag, i in ev[:60]:
        print(f"{(t - t0):8d} ns  w{w} {NAMES.get(tag, tag):12s} {i}")
    print("last 30 events:")
    for t, w, tag, i in ev[-30:]:
        print(f"{(t - t0):8d} ns  w{w} {NAMES.get(tag, tag):12s} {i}")


if __name__ == "__main__":
    main()
