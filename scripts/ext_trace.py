"""Stage timeline of the tcgen05 extend kernel (CTA 0, first item): clock64 deltas per role."""
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
rec = workloads.qwen(); m = rec.model; Lr = 2
pool = spa.Pool(Lr, m.num_q_heads, m.num_kv_heads, m.head_dim, bench.pages_for(rec, 8), device=dev)
ids, reqs, batch = bench.build_batch(spa, pool, rec, list(range(Lr)), slice(0, m.num_kv_heads), dev, fill="reuse")
lens = [pool.page_table(r)[2] for r in reqs]
nq = [1 if who == "main" else 16 for (gi, who), n in zip(batch, lens)]
rows = sum(nq)
q = kv_bits_torch(rec.seed, KIND_Q, 3_000_000, list(range(Lr)), np.arange(rows), m.num_q_heads, m.head_dim, dev).contiguous()
o = torch.empty((rows, m.num_q_heads, m.head_dim), dtype=torch.bfloat16, device=dev)
plan = spa.Plan(pool, max_rows=128)
plan.plan(reqs, 0, stream=stream, n_query=nq)
for i in range(4):
    plan.decode(i % Lr, q[i % Lr], o, None, scale=m.softmax_scale, stream=stream, want_lse=False)
torch.cuda.synchronize()
cap = 512
buf = torch.zeros((8, cap, 2), dtype=torch.int64, device=dev)
spa.lib().spa_debug_set_trace(plan.h, spa._ptr(buf), cap)
plan.decode(0, q[0], o, None, scale=m.softmax_scale, stream=stream, want_lse=False)
torch.cuda.synchronize()
spa.lib().spa_debug_set_trace(plan.h, None, 0)
tr = buf.cpu().numpy().astype(np.uint64)
ev = []
for w in range(3):
    for k in range(cap):
        w1 = tr[w, k, 1]
        tag = int(w1 >> np.uint64(56))
        if tag == 0:
            break
        ev.append((int(w1 & np.uint64(0xffffffff)), w, tag, int((w1 >> np.uint64(32)) & np.uint64(0xffffff))))
ev.sort()
t0 = ev[0][0]
names = {10: "P issue", 20: "M full", 21: "M S-issued", 22: "M pfull", 30: "W sfull", 31: "W pfull-arr"}
for c, w, tag, st in ev[:160]:
    print(f"{(c - t0) % (1 << 32):9d}  w{w} {names.get(tag, tag):12s} st={st}")
# per-stage period of the WG
wg = [c for c, w, tag, st in ev if tag == 30]
d = np.diff(np.array(wg, dtype=np.int64) % (1 << 32))
print("WG s_full period cycles: median", np.median(d[5:]) if len(d) > 6 else d, "n", len(wg))
sw = {st: c for c, w, tag, st in ev if tag == 30}
pa = {st: c for c, w, tag, st in ev if tag == 31}
print("WG compute (sfull->pfull arrive) median", np.median([(pa[k] - sw[k]) % (1 << 32) for k in sw if k in pa]))
mf = {st: c for c, w, tag, st in ev if tag == 22}
print("p_full arrive -> MMA wake median", np.median([(mf[k + 1] - pa[k]) % (1 << 32) for k in pa if k + 1 in mf]))
si = {st: c for c, w, tag, st in ev if tag == 21}
print("S issued -> WG s_full wake median", np.median([(sw[k] - si[k]) % (1 << 32) for k in si if k in sw]))
fu = {st: c for c, w, tag, st in ev if tag == 20}
print("MMA full-wait done -> S issued median", np.median([(si[k] - fu[k]) % (1 << 32) for k in fu if k in si]))
