"""Benchmark of the SPAgent decode-attention step (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config qwen|gemma|long|tiny]
                    [--impl spa|reference] [--no-parity] [--no-e2e] [--graph]

A step = one pass of the whole hot path over one batch:
  a2 spa_kv_append of one new token per request (all layers),
  a4 spa_decode_plan (host planning + one upload; one plan per distinct window),
  a5+a6 spa_decode_attention for every layer of the model (decode kernel; split merge
        in-kernel by default),
  a7 (N > 1) the NCCL all-gather of head-sharded outputs.
Fork/alloc/free (a1, a3, a8) build the batch before timing (host calls; the copy-on-write
kernels run there).

Default workload: BJ config 1 (Qwen2.5-32B attention: 40 Q / 8 KV heads, d=128, 64 layers,
32 agents + 32 speculative forks, contexts 2k-8k), synthetic seeded data, all 64 layers
resident.  value = decode tokens/s = N_requests / step time (each request decodes one
token per step through all layers), max over ranks.  Prints ONE JSON line on rank 0.

--config gemma (BJ config 2): 62 attention calls per step, 52 with a 1024-token sliding
window (5:1 local/global), over 6 resident layers (call i reads resident layer i % 6; each
layer's KV is far larger than L2, so reuse gives no cache benefit).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from spa_inputs import KIND_K, KIND_Q, KIND_V, kv_bits_np, kv_bits_torch, workloads  # noqa: E402
from spa_inputs.families import origin_id  # noqa: E402

_T0 = time.time()


def _log(*a):
    """Progress on stderr (the JSON line on stdout stays the only stdout output)."""
    print(f"[bench {time.time() - _T0:7.1f}s]", *a, file=sys.stderr, flush=True)


METRIC = "decode-attn tokens/s and achieved HBM GB/s (% of peak) at 1/2/4/8 B200"
BJ_INDEX = {"tiny": 0, "qwen": 1, "gemma": 2, "long": 4}


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="qwen", choices=["qwen", "tiny", "gemma", "long"])
    ap.add_argument("--impl", default="spa", choices=["spa", "reference"])
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--graph", action="store_true", help="replay the per-step layer loop as a CUDA graph")
    ap.add_argument("--profile", action="store_true",
                    help="cudaProfilerStart/Stop around the timed steps only (ncu --profile-from-start off); "
                         "skips parity, e2e and the cpu baseline")
    ap.add_argument("--sharing", type=int, default=1)
    ap.add_argument("--kv", default="bf16", choices=["bf16", "fp8"],
                    help="KV page format: bf16, or e4m3 with static per-(layer, head) scales (S8(f) F4 variant)")
    ap.add_argument("--gather", default="fused", choices=["fused", "nccl"],
                    help="N > 1: fused decode + peer-memory all-gather (S8(f) F1) or decode + ncclAllGather")
    ap.add_argument("--merge-mode", type=int, default=0,
                    help="split merge: 0 in-kernel tail phase, 1 in-kernel last arriver, 2 PDL-chained merge kernel")
    ap.add_argument("--split-pages", type=int, default=0, help="max pages per split (0 = auto)")
    ap.add_argument("--layers", type=int, default=0, help="resident layers (0 = config default)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="budget of the oracle cpu_baseline sample")
    return ap.parse_args(argv)


def recipe_for(name):
    return {"qwen": workloads.qwen, "tiny": workloads.tiny, "gemma": workloads.gemma,
            "long": workloads.long32k}[name]()


def default_resident_layers(name, model):
    return {"gemma": 6, "long": 4}.get(name, model.num_layers)


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except (OSError, ValueError):
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def layer_schedule(recipe, resident):
    """[(resident layer, window)] of the attention calls of one model step: one call per model
    layer (S8(d): a step is the whole model's attention), cycling through the resident layers
    when the pool holds fewer (Gemma-3: 62 calls over 6; long-32k: 64 calls over 4 -- each
    call reads more than the L2 holds, so a re-used resident layer is not served from cache)."""
    m = recipe.model
    if recipe.local_layers:
        local = set(recipe.local_layers)
        return [(i % resident, recipe.window if i in local else 0) for i in range(m.num_layers)]
    return [(i % resident, 0) for i in range(m.num_layers)]


# ----------------------------------------------------------------------------- oracle (cpu)
def logical_kv_np(recipe, gi, who, layers, kind):
    """Host bits [L, n, Hkv, d] of a batch member's logical KV (parent stream + own tail)."""
    g = recipe.groups[gi]
    m = recipe.model
    main = origin_id((gi, "main"))
    if who == "main":
        n = g.prefix + (g.parent_tail or 0)
        return kv_bits_np(recipe.seed, kind, main, layers, np.arange(n), m.num_kv_heads, m.head_dim)
    j = int(who[1:])
    a = kv_bits_np(recipe.seed, kind, main, layers, np.arange(g.prefix), m.num_kv_heads, m.head_dim)
    own = origin_id((gi, who))
    b = kv_bits_np(recipe.seed, kind, own, layers, np.arange(g.prefix, g.prefix + g.fork_tails[j]),
                   m.num_kv_heads, m.head_dim)
    return np.concatenate([a, b], axis=1)


# F4: the counter-hash generator's values lie in [-126/32, 126/32] (spa_inputs._h2v_np), so a
# static scale of (126/32)/448 maps every K/V value into e4m3's range without saturation
FP8_SCALE = np.float32((126.0 / 32.0) / 448.0)


def oracle_sample(recipe, batch, rows, layer, q_bits, steps_appended, window=0, fp8=False):
    """fp64 oracle outputs for batch rows `rows` at one (resident) layer."""
    from oracle.attention import decode_attention
    from oracle.fp8 import dequantize_e4m3, quantize_kv
    from oracle.replay import bits_to_f64

    m = recipe.model
    out_o, out_l = [], []
    for r in rows:
        gi, who = batch[r]
        K = logical_kv_np(recipe, gi, who, [layer], KIND_K)[0]
        V = logical_kv_np(recipe, gi, who, [layer], KIND_V)[0]
        for s in range(steps_appended):
            kb = kv_bits_np(recipe.seed, KIND_K, 500_000 + s, [layer], np.arange(len(batch)), m.num_kv_heads, m.head_dim)
            vb = kv_bits_np(recipe.seed, KIND_V, 500_000 + s, [layer], np.arange(len(batch)), m.num_kv_heads, m.head_dim)
            K = np.concatenate([K, kb[0, r:r + 1]])
            V = np.concatenate([V, vb[0, r:r + 1]])
        Kf, Vf = bits_to_f64(K), bits_to_f64(V)
        if fp8:   # the pool holds scale * e4m3(fp32(x) / scale) (oracle/fp8.py)
            Kf = dequantize_e4m3(quantize_kv(Kf.astype(np.float32), FP8_SCALE), FP8_SCALE)
            Vf = dequantize_e4m3(quantize_kv(Vf.astype(np.float32), FP8_SCALE), FP8_SCALE)
        O, L = decode_attention(bits_to_f64(q_bits[r]), Kf, Vf, m.softmax_scale, window)
        out_o.append(O)
        out_l.append(L)
    return np.stack(out_o), np.stack(out_l)


def cpu_baseline(recipe, batch, budget_s):
    """The oracle as it stands, timed on this host's cores on a bounded sample of the
    workload: whole requests at one layer until ~budget_s of CPU work, scaled to tokens/s
    of the full model step (one token = one request through all of the step's layer calls,
    each at its own window)."""
    from oracle.attention import decode_attention
    from oracle.replay import bits_to_f64

    m = recipe.model
    sched = layer_schedule(recipe, default_resident_layers("gemma" if recipe.local_layers else "x", m))
    windows = sorted({w for _, w in sched})
    calls_per_window = {w: sum(1 for _, ww in sched if ww == w) for w in windows}
    rng = np.random.default_rng(0)
    order = rng.permutation(len(batch))
    q = kv_bits_np(recipe.seed, KIND_Q, 1_000_000, [0], np.arange(len(batch)), m.num_q_heads, m.head_dim)[0]
    done = 0
    t_work = {w: 0.0 for w in windows}
    t0 = time.perf_counter()
    for r in order:
        gi, who = batch[r]
        K = bits_to_f64(logical_kv_np(recipe, gi, who, [0], KIND_K)[0])
        V = bits_to_f64(logical_kv_np(recipe, gi, who, [0], KIND_V)[0])
        qf = bits_to_f64(q[r])
        for w in windows:
            ts = time.perf_counter()
            decode_attention(qf, K, V, m.softmax_scale, w)
            t_work[w] += time.perf_counter() - ts
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    elapsed = time.perf_counter() - t0
    per_req_step = sum(t_work[w] / done * calls_per_window[w] for w in windows)
    tok_s = 1.0 / per_req_step
    cores = os.cpu_count()
    try:
        import threadpoolctl

        info = threadpoolctl.threadpool_info()
        cores = max([i.get("num_threads", 1) for i in info] + [1])
    except Exception:  # noqa: BLE001
        pass
    return {"value": tok_s, "unit": "tokens/s", "cores": cores, "kind": "oracle", "elapsed_s": elapsed,
            "sample": f"{done} of {len(batch)} requests x 1 layer per window {windows} (fp64 NumPy, BLAS dgemm "
                      f"per KV head), {per_req_step * 1e3:.1f} ms per request-step over {len(sched)} layer calls"}


# ----------------------------------------------------------------------------- clocks
class Clocks:
    def __init__(self, path):
        self.path = path
        self.proc = None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()
            self.f.close()

    def summary(self, device_index):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            p = [x.strip() for x in line.split(",")]
            if len(p) < 9 or p[0] != str(device_index):
                continue
            try:
                sm.append(float(p[1]))
                mx.append(float(p[2]))
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- batch build
def build_batch(spa, pool, recipe, layers, kv_sl, dev, fill="hash", chunk=256):
    """Replay the recipe's call log through the C ABI (a1 alloc, a2 append, a3 fork).

    fill="hash": every appended token carries its own counter-hash K/V (parity-checkable);
    fill="reuse": one chunk of counter-hash values is appended repeatedly (throughput
    sweeps: timing does not depend on the values).
    """
    import torch

    m = recipe.model
    ops, batch = workloads.call_log(recipe)
    ids = {}
    reuse = None
    if fill == "reuse":
        pos = np.arange(chunk)
        reuse = (kv_bits_torch(recipe.seed, KIND_K, 0, layers, pos, m.num_kv_heads, m.head_dim, dev)[:, :, kv_sl]
                 .contiguous(),
                 kv_bits_torch(recipe.seed, KIND_V, 0, layers, pos, m.num_kv_heads, m.head_dim, dev)[:, :, kv_sl]
                 .contiguous())
    for op in ops:
        if op[0] == "alloc":
            ids[op[1]] = pool.alloc()
        elif op[0] == "append":
            _, name, origin, start, n = op
            for s0 in range(start, start + n, chunk):
                s1 = min(start + n, s0 + chunk)
                if reuse is not None:
                    k, v = reuse[0][:, :s1 - s0].contiguous(), reuse[1][:, :s1 - s0].contiguous()
                else:
                    pos = np.arange(s0, s1)
                    k = kv_bits_torch(recipe.seed, KIND_K, origin_id(origin), layers, pos, m.num_kv_heads,
                                      m.head_dim, dev)[:, :, kv_sl].contiguous()
                    v = kv_bits_torch(recipe.seed, KIND_V, origin_id(origin), layers, pos, m.num_kv_heads,
                                      m.head_dim, dev)[:, :, kv_sl].contiguous()
                pool.append([ids[name]], [s1 - s0], k, v)
        elif op[0] == "fork":
            ids[op[1]] = pool.fork(ids[op[2]], op[3])
    torch.cuda.synchronize()
    return ids, [ids[nm] for nm in batch], batch


def pages_for(recipe, extra_tokens):
    pages = 8
    for g in recipe.groups:
        pages += -(-(g.prefix + (g.parent_tail or 0) + extra_tokens) // 16)
        if g.spec_prompt is not None:
            pages += -(-(g.spec_prompt + 16 + extra_tokens) // 16)
        pages += sum(-(-(ft + 16 + extra_tokens) // 16) for ft in g.fork_tails)
    return pages


def alg_bytes(st, N, hkv_l, hq_l, d, kv_elem=2, method=True):
    """Algorithmic bytes of one decode_attention launch (per GPU), SURVEY.md Sec. 8(d) B_alg:
    every distinct attended KV key read once (alg_tokens per KV head: distinct (page, slot)
    positions) x Hkv_l x d x 2 (K, V) x kv_elem B (2 bf16, 1 fp8) + Q + O (bf16) + LSE
    (fp32).  method=False adds the implementation's overheads (overhead_bytes)."""
    kv = st["alg_tokens"] * hkv_l * d * 2 * kv_elem
    qo = N * hq_l * d * 2 * 2 + N * hq_l * 4
    if method:
        return kv + qo
    o = overhead_bytes(st, hkv_l, hq_l, d, kv_elem)
    return kv + qo + o["reread_kv"] + o["partials"]


def overhead_bytes(st, hkv_l, hq_l, d, kv_elem=2):
    """Bytes the plan moves beyond B_alg: KV keys read again by a class cut into max_rows
    chunks (unique_tokens - alg_tokens; served by L2 when the chunks run close in time) and
    the fp32 split partials (written, then read by the merge)."""
    return {"reread_kv": (st["unique_tokens"] - st["alg_tokens"]) * hkv_l * d * 2 * kv_elem,
            "partials": st["n_records"] * hq_l * (d + 1) * 4 * 2}


# ----------------------------------------------------------------------------- main arm
def run_spa(args):
    import torch
    import torch.distributed as dist

    from paper_2511_20048_b200 import spa

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    # SPA_BENCH_SHARE_DEVICE=1: every rank on cuda:0 over a gloo group -- a functional check
    # of the multi-process (fused, CUDA IPC) path on a one-GPU box; its timings time-slice
    # the contexts and mean nothing
    share = os.environ.get("SPA_BENCH_SHARE_DEVICE") == "1"
    if share:
        local = 0
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE {world}"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    spa.lib()

    recipe = recipe_for(args.config)
    m = recipe.model
    Lr = args.layers or default_resident_layers(args.config, m)
    layers = list(range(Lr))
    sched = layer_schedule(recipe, Lr)
    C = len(sched)
    windows = sorted({w for _, w in sched})
    q_sl, kv_sl = spa.shard_heads(m.num_q_heads, m.num_kv_heads, rank, world)
    hkv_l, hq_l = kv_sl.stop - kv_sl.start, q_sl.stop - q_sl.start
    d = m.head_dim
    total_steps = args.warmup + args.steps + 32
    # one non-default stream carries every launch and copy (CUDA-graph capture needs a
    # non-legacy stream); torch ops use it as their current stream
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    fp8 = args.kv == "fp8"
    pool = spa.Pool(Lr, hq_l, hkv_l, d, pages_for(recipe, total_steps), device=dev,
                    kv_scale=np.full((Lr, hkv_l, 2), FP8_SCALE, np.float32) if fp8 else None)

    t_build = time.perf_counter()
    ids, reqs, batch = build_batch(spa, pool, recipe, layers, kv_sl, dev)
    t_build = time.perf_counter() - t_build
    _log('built batch', t_build)
    N = len(batch)

    # ---- per-step inputs (resident in HBM for the device-timed value)
    q_res = kv_bits_torch(recipe.seed, KIND_Q, 1_000_000, layers, np.arange(N), m.num_q_heads, d, dev)[:, :, q_sl]
    q_all = torch.stack([q_res[r] for r, _ in sched]).contiguous()          # [C, N, Hq_l, d]
    step_k = [kv_bits_torch(recipe.seed, KIND_K, 500_000 + s, layers, np.arange(N), m.num_kv_heads, d, dev)[:, :, kv_sl]
              .contiguous() for s in range(2)]
    step_v = [kv_bits_torch(recipe.seed, KIND_V, 500_000 + s, layers, np.arange(N), m.num_kv_heads, d, dev)[:, :, kv_sl]
              .contiguous() for s in range(2)]
    comm = peer = None
    gather = "none (1 GPU)"
    if world > 1 and args.gather == "fused":
        # F1: the library's peer region holds 3C gathered buffers (the e2e leg rotates three
        # output sets); handles are all-gathered over the process group
        # every stage is agreed collectively, so a failure on one rank sends ALL ranks to NCCL
        def agree(flag):
            t = torch.tensor([1 if flag else 0], device="cpu" if share else dev)
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            return bool(t.item())

        why = ""
        handle = None
        try:
            peer = spa.Peer(rank, world, spa.Peer.buffer_bytes(N, m.num_q_heads, d), n_bufs=3 * C, connect=False)
            handle = peer.ipc_handle()
        except Exception as e:  # noqa: BLE001 -- fall back to NCCL, reported in the JSON line
            why = repr(e)
        if agree(handle is not None):
            handles = [None] * world
            dist.all_gather_object(handles, handle)
            try:
                peer.connect(handles)
                o_views, l_views = peer.views_all(N, m.num_q_heads, d, device=dev)
            except Exception as e:  # noqa: BLE001
                why = repr(e)
        if not agree(not why):
            if peer is not None:
                dist.barrier()
                peer.close()
            peer = None
            gather = f"nccl (fused setup failed: {why[:120] or 'on another rank'})"
        else:
            o_all, lse_all = o_views[:C], l_views[:C]
            gather = "fused decode + peer-memory all-gather (CUDA IPC over NVLink)"
    if world > 1 and peer is None:
        comm_id = [spa.spa_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(comm_id, src=0)
        comm = spa.Comm(comm_id[0], rank, world)
        o_all = torch.empty((C, m.num_q_heads, N, d), dtype=torch.bfloat16, device=dev)   # gathered, head-major
        lse_all = torch.empty((C, m.num_q_heads, N), dtype=torch.float32, device=dev)
        if not gather.startswith("nccl"):
            gather = "decode + in-place ncclAllGather"
    elif world == 1:
        o_all = torch.empty((C, N, hq_l, d), dtype=torch.bfloat16, device=dev)
        lse_all = torch.empty((C, N, hq_l), dtype=torch.float32, device=dev)
    plans = {w: spa.Plan(pool, sharing=bool(args.sharing), split_pages=args.split_pages, merge_mode=args.merge_mode)
             for w in windows}
    state = {"step": 0, "graph": None}

    def launch(ci, qq, oo, ll):
        r, w = sched[ci]
        if peer is not None:   # oo / ll are views of the peer buffers: recover the buffer index
            b = (oo.data_ptr() - o_views.data_ptr()) // (o_views.stride(0) * 2)
            peer.decode(plans[w], r, qq[ci], buf_idx=int(b) + ci, scale=m.softmax_scale, stream=stream)
        elif comm is None:
            plans[w].decode(r, qq[ci], oo[ci], ll[ci], scale=m.softmax_scale, stream=stream)
        else:
            plans[w].decode_sharded(comm, r, qq[ci], oo[ci], ll[ci], scale=m.softmax_scale, stream=stream)

    def layer_loop(qq, oo, ll):
        for ci in range(C):
            launch(ci, qq, oo, ll)

    def one_step(kk, vv, qq=None, oo=None, ll=None):
        qq = q_all if qq is None else qq
        oo = o_all if oo is None else oo
        ll = lse_all if ll is None else ll
        s = state["step"]
        pool.append(reqs, [1] * N, kk[s % 2] if isinstance(kk, list) else kk,
                    vv[s % 2] if isinstance(vv, list) else vv, stream=stream)
        for w, p in plans.items():
            p.plan(reqs, w, stream=stream)
        if state["graph"] is not None and qq is q_all and oo is o_all:
            state["graph"].replay()
        else:
            layer_loop(qq, oo, ll)
        state["step"] = s + 1

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- fused gather: one probe call first (a peer that never arrives costs the kernel's
    #      20-s timeout once, not once per call); every rank must agree, else all use NCCL
    if peer is not None:
        pool.append(reqs, [1] * N, step_k[0], step_v[0], stream=stream)
        for w, p in plans.items():
            p.plan(reqs, w, stream=stream)
        launch(0, q_all, o_all, lse_all)
        torch.cuda.synchronize()
        state["step"] = 1
        ok = torch.tensor([1 if peer.status() == 0 else 0], device="cpu" if share else dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()) == 0:
            barrier()
            peer.close()
            peer = None
            gather = "nccl (the fused gather's probe call timed out)"
            comm_id = [spa.spa_nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(comm_id, src=0)
            comm = spa.Comm(comm_id[0], rank, world)
            o_all = torch.empty((C, m.num_q_heads, N, d), dtype=torch.bfloat16, device=dev)
            lse_all = torch.empty((C, m.num_q_heads, N), dtype=torch.float32, device=dev)

    # ---- parity gate: the first step's sampled outputs vs the fp64 oracle
    parity = None
    one_step(step_k, step_v)
    torch.cuda.synchronize()
    if peer is not None and peer.status() != 0:
        print(json.dumps({"error": "fused gather: a peer did not arrive (spa_peer_status)"}))
        sys.exit(1)
    if args.profile:
        args.no_parity = args.no_e2e = True
    if not args.no_parity and rank == 0:
        gsel = sorted({0, len(recipe.groups) // 2})
        rows = [i for i, nm in enumerate(batch) if nm[0] in gsel]
        calls = sorted({0, C - 1} | {next((i for i, (_, w) in enumerate(sched) if w == 0), 0)})
        worst_o = worst_l = 0.0
        for ci in calls:
            r, w = sched[ci]
            qb = kv_bits_np(recipe.seed, KIND_Q, 1_000_000, [r], np.arange(N), m.num_q_heads, d)[0]
            O, Lo = oracle_sample(recipe, batch, rows, r, qb, steps_appended=state["step"], window=w, fp8=fp8)
            if world == 1:
                og = o_all[ci, rows].float().cpu().numpy()
                lg = lse_all[ci, rows].cpu().numpy()
                O, Lo = O[:, q_sl], Lo[:, q_sl]
            else:
                og = o_all[ci][:, rows].permute(1, 0, 2).float().cpu().numpy()
                lg = lse_all[ci][:, rows].permute(1, 0).cpu().numpy()
            worst_o = max(worst_o, float(np.abs(og - O).max()))
            worst_l = max(worst_l, float(np.abs(lg - Lo).max()))
        parity = {"max_abs_o": worst_o, "max_abs_lse": worst_l, "rows": len(rows),
                  "calls": [{"call": ci, "layer": sched[ci][0], "window": sched[ci][1]} for ci in calls],
                  "pass": worst_o <= 2e-2 and worst_l <= 1e-3}
        if not parity["pass"]:
            print(json.dumps({"error": "parity gate failed", "parity": parity}))
            sys.exit(1)

    _log('parity', parity)
    # the peers' next step may write the buffers rank 0 just read on the host (fused gather)
    barrier()
    # ---- optional CUDA graph of the layer loop (plan device buffers are stable across steps)
    if args.graph and peer is not None:
        # a captured fused launch would replay its epoch: the peer flags would not order calls
        raise SystemExit("--graph is not supported with --gather fused (use --gather nccl)")
    if args.graph:
        gens = {w: p.stats()["generation"] for w, p in plans.items()}
        g = torch.cuda.CUDAGraph()
        barrier()
        with torch.cuda.graph(g, stream=stream):
            layer_loop(q_all, o_all, lse_all)
        state["graph"] = g
        barrier()

    # ---- warm-up, then K timed steps (device events on the launching stream)
    for _ in range(args.warmup):
        one_step(step_k, step_v)
    barrier()
    if args.graph:
        assert all(p.stats()["generation"] == gens[w] for w, p in plans.items()), "plan buffers moved"
    clocks = Clocks(os.path.join(ROOT, "gpurun_out", f"clocks_rank{rank}.csv")
                    if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else f"/tmp/spa_clocks_{rank}.csv")
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with clocks:
        time.sleep(0.3)
        barrier()
        if args.profile:
            torch.cuda.profiler.start()
        ev0.record(stream)
        for _ in range(args.steps):
            one_step(step_k, step_v)
        ev1.record(stream)
        barrier()
        if args.profile:
            torch.cuda.profiler.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    _log('timed steps', ms)
    if world > 1:
        t = torch.tensor([ms], device="cpu" if share else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # ---- per-launch timing per window class: events around the chained loop of every call
    #      of that class (PDL chaining as in the step), and around each call in isolation
    barrier()
    pool.append(reqs, [1] * N, step_k[0], step_v[0], stream=stream)
    for w, p in plans.items():
        p.plan(reqs, w, stream=stream)
    per_window = {}
    for w in windows:
        cis = [ci for ci, (_, ww) in enumerate(sched) if ww == w]
        chained = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for ci in cis:
                launch(ci, q_all, o_all, lse_all)
            e1.record(stream)
            barrier()
            chained.append(e0.elapsed_time(e1) / len(cis))
        iso = []
        for ci in cis[: min(len(cis), 16)]:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            launch(ci, q_all, o_all, lse_all)
            e1.record(stream)
            barrier()
            iso.append(e0.elapsed_time(e1))
        st = plans[w].stats()
        per_window[w] = {"calls": len(cis), "layer_ms": float(np.median(chained)),
                         "layer_ms_isolated": float(np.median(iso)), "stats": st,
                         "alg_bytes": alg_bytes(st, N, hkv_l, hq_l, d, 1 if fp8 else 2)}
    _log('per-window timing done')
    # the dominant launch class: most total time per step
    wdom = max(windows, key=lambda w: per_window[w]["layer_ms"] * per_window[w]["calls"])
    dom = per_window[wdom]
    st = dom["stats"]
    pk, pk_kind = peaks()
    achieved = dom["alg_bytes"] / (dom["layer_ms"] * 1e-3) / 1e9
    ceilings = spa.read_ceilings(pool) if not args.profile else None
    _log('ceilings', ceilings)
    traffic = None
    try:
        nc = json.load(open(os.path.join(ROOT, "profiles", "latest_ncu.json")))
        if nc.get("config") == args.config and world == 1 and args.sharing and not fp8:
            traffic = nc["traffic_bytes_per_launch"]
    except (OSError, ValueError, KeyError):
        pass

    # ---- end-to-end through the public API with host buffers (pinned), copies inside the
    #      timed region: every step copies its q / new K,V host->device and its O / LSE
    #      device->host.  The copies run on a second stream, double-buffered, so step s+1's
    #      inputs and step s-1's outputs move while step s computes (a serving loop's
    #      pipelining; the dependencies are events, nothing is skipped).
    e2e = None
    if not args.no_e2e:
        hq = q_all.cpu().pin_memory()
        hk = step_k[0].cpu().pin_memory()
        hv = step_v[0].cpu().pin_memory()
        # output sets: with the fused gather a peer's step i+1 may write step i-2's set as soon as
        # this rank finished step i, so its copy-out must be done by then (3 sets, wait on i-2)
        nb = 3 if peer is not None else 2
        ho = [torch.empty(o_all.shape, dtype=o_all.dtype).pin_memory() for _ in range(nb)]
        hl = [torch.empty(lse_all.shape, dtype=lse_all.dtype).pin_memory() for _ in range(nb)]
        dq = [torch.empty_like(q_all) for _ in range(2)]
        dk = [torch.empty_like(step_k[0]) for _ in range(2)]
        dv = [torch.empty_like(step_v[0]) for _ in range(2)]
        if peer is not None:
            do = [o_views[j * C:(j + 1) * C] for j in range(nb)]
            dl = [l_views[j * C:(j + 1) * C] for j in range(nb)]
        else:
            do = [o_all, torch.empty_like(o_all)]
            dl = [lse_all, torch.empty_like(lse_all)]
        cs = torch.cuda.Stream(device=dev)
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_done = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(nb)]
        e2e_steps = max(4, min(args.steps, 10))
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        cs.wait_event(e0)

        def stage_in(i):
            b = i % 2
            with torch.cuda.stream(cs):
                if i >= 2:
                    cs.wait_event(ev_done[b])      # step i-2 finished reading buffer b
                dq[b].copy_(hq, non_blocking=True)
                dk[b].copy_(hk, non_blocking=True)
                dv[b].copy_(hv, non_blocking=True)
                ev_in[b].record(cs)

        stage_in(0)
        for i in range(e2e_steps):
            b, bo = i % 2, i % nb
            if i + 1 < e2e_steps:
                stage_in(i + 1)
            stream.wait_event(ev_in[b])
            if i >= 2:
                stream.wait_event(ev_out[(i - 2) % nb])   # step i-2's outputs have been copied out
            one_step(dk[b], dv[b], dq[b], do[bo], dl[bo])
            ev_done[b].record(stream)
            with torch.cuda.stream(cs):
                cs.wait_event(ev_done[b])
                ho[bo].copy_(do[bo], non_blocking=True)
                hl[bo].copy_(dl[bo], non_blocking=True)
                ev_out[bo].record(cs)
        e1.record(cs)
        barrier()
        e2e_ms = e0.elapsed_time(e1) / e2e_steps
        if world > 1:
            t = torch.tensor([e2e_ms], device="cpu" if share else dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        h2d = hq.numel() * 2 + hk.numel() * 2 * 2
        d2h = ho[0].numel() * 2 + hl[0].numel() * 4
        e2e = {"value": N / (e2e_ms * 1e-3), "unit": "tokens/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "pipelining": "H2D/D2H on a copy stream, double-buffered"}

    ws_step = sum(pw["alg_bytes"] * pw["calls"] for pw in per_window.values())   # distinct layers per call
    result = None
    if rank == 0:
        cpu = cpu_baseline(recipe, batch, args.cpu_seconds) if world == 1 and not args.profile else None
        ck = clocks.summary(local)
        # merge_mode 0 on fp8 pools decoded by one-warp teams (teams == warps per CTA) without
        # the fused gather also launches merge_kernel (include/spa.h merge_mode)
        _, g_teams, g_warps = next(iter(plans.values())).geometry()
        sep = args.merge_mode == 2 or (args.merge_mode == 0 and fp8 and g_teams == g_warps and peer is None)
        launches_per_step = (-(-N // 896)) + sum(
            1 + (1 if sep and per_window[w]["stats"]["n_records"] > 0 else 0) for _, w in sched)
        kname = {0: "decode_kernel + merge_kernel (fp8 one-warp teams)" if sep else
                 "decode_kernel (split merge in-kernel, tail phase)",
                 1: "decode_kernel (split merge in-kernel, last arriver)",
                 2: "decode_kernel + merge_kernel (one spa_decode_attention call)"}[args.merge_mode]
        result = {
            "metric": METRIC,
            "value": N / (ms * 1e-3),
            "unit": "tokens/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "bf16 (KV pages e4m3, f16 MMA)" if fp8 else "bf16",
            "data": "synthetic (seeded counter-hash bf16 K/V/Q, agent-shaped batch recipe)",
            "config": {"workload": f"{recipe.name} (BJ config {BJ_INDEX[args.config]})",
                       "n_requests": N, "agents": len(recipe.groups), "layer_calls_per_step": C,
                       "resident_layers": Lr, "windows": windows,
                       "q_heads": m.num_q_heads, "kv_heads": m.num_kv_heads, "head_dim": d,
                       "parallelism": f"kv-head sharded x{world}" if world > 1 else "1 GPU",
                       "gather": gather,
                       "kv_pages": f"e4m3, static scale {float(FP8_SCALE):.6g} per (layer, KV head)" if fp8 else "bf16",
                       "sharing": bool(args.sharing), "cuda_graph": bool(args.graph),
                       "l2": "inputs larger than L2 (the KV a step's calls read > 4 x 126 MB, layers rotate), no flush"
                       if ws_step > 4 * 126e6 else "KV of a step fits L2: latency, not bandwidth"},
            "gpu_launches": int(launches_per_step * args.steps),
            "layer_ms": dom["layer_ms"],
            "layer_ms_isolated": dom["layer_ms_isolated"],
            "per_window": {str(w): {k: v for k, v in pw.items() if k != "stats"} | {
                "n_records": pw["stats"]["n_records"], "unique_tokens": pw["stats"]["unique_tokens"],
                "gbs": pw["alg_bytes"] / (pw["layer_ms"] * 1e-3) / 1e9} for w, pw in per_window.items()},
            "hbm_gbs_algorithmic": achieved,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / pk["hbm_gbs"], "traffic": traffic,
                         "traffic_source": "profiles/latest_ncu.json (ncu dram__bytes_read+write per launch)",
                         "kernel": kname, "window": wdom,
                         "peak_kind": pk_kind, "alg_bytes_per_launch": int(dom["alg_bytes"]),
                         "frac_of_8tbs": achieved / 8000.0,
                         "same_run_read_ceilings_gbs": ceilings,
                         "frac_of_tma_ceiling": (achieved / ceilings["tma_pool_read_gbs"])
                         if ceilings and "tma_pool_read_gbs" in ceilings else None},
            "sharing": {"unique_tokens_per_kv_head": st["unique_tokens"],
                        "unshared_tokens_per_kv_head": st["unshared_tokens"],
                        "bytes_vs_unshared": st["unique_tokens"] / st["unshared_tokens"]},
            "plan": {k: st[k] for k in ("n_groups", "n_desc", "n_items", "n_records", "n_teams", "rows_max")},
            "parity": parity,
            "clocks": ck,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "build_s": t_build,
        }
        print(json.dumps(result), flush=True)
    if world > 1:
        torch.cuda.synchronize()
        dist.barrier()
        if comm is not None:
            comm.close()
        if peer is not None:
            fail = peer.status()
            dist.barrier()   # every rank is done with the others' buffers before any is freed
            peer.close()
            if fail and rank == 0:
                print(json.dumps({"error": "fused gather: a peer did not arrive (spa_peer_status)"}), flush=True)
        dist.destroy_process_group()
    return result


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    """The oracle as it stands on the host cores, same metric/config/unit (tokens/s)."""
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return None
    recipe = recipe_for(args.config)
    ops, batch = workloads.call_log(recipe)
    budget = max(2.0, min(20.0, 120.0 / max(1, args.steps + args.warmup)))
    vals, secs = [], []
    info = None
    for i in range(args.warmup + args.steps):
        info = cpu_baseline(recipe, batch, budget)
        if i >= args.warmup:
            vals.append(info["value"])
            secs.append(info["elapsed_s"])
    v = float(np.mean(vals))
    # ms_per_step: the wall time each timed step actually ran (a bounded sample of the batch);
    # value: the oracle's measured rate on that sample, in tokens/s of the full model step
    per_step_ms = 1e3 * float(np.mean(secs))
    res = {"impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step_ms, "higher_is_better": True,
           "step_is_sample": True, "full_step_ms_estimate": 1e3 * len(batch) / v,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"{recipe.name} (BJ config {BJ_INDEX[args.config]})", "n_requests": len(batch)},
           "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": info["cores"], "kind": "oracle",
                            "sample": info["sample"]},
           "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(res), flush=True)
    return res


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_spa(a)
