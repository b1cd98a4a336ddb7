"""Summarise ncu captures for profiles/: key counters of a full capture, launch-list shares.

    python scripts/ncu_summary.py full  gpurun_out/prof_decode_TAG.ncu-rep  [--top 25]
    python scripts/ncu_summary.py launches gpurun_out/launches_TAG.csv
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__bytes.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_active.avg", "sm__cycles_elapsed.max", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
    "sm__pipe_tma_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
]


def ncu_csv(args):
    out = subprocess.run(["ncu", "-i", *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def full(rep, top=25):
    rows = ncu_csv([rep, "--page", "raw"])
    h, units, vals = rows[0], rows[1], rows[2:]
    name = vals[0][h.index("Kernel Name")] if "Kernel Name" in h else "?"
    print(f"kernel: {name[:100]}  (launches captured: {len(vals)})")
    for k in KEYS:
        if k in h:
            i = h.index(k)
            print(f"  {k:80s} {units[i]:>10s} " + " ".join(v[i] for v in vals))
    # per-instruction stall samples, grouped by SASS opcode class
    rows = ncu_csv([rep, "--page", "source", "--print-source", "sass"])
    blocks, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = []
            blocks.append(cur)
        elif cur is not None:
            cur.append(r)
    if not blocks:
        return
    b = blocks[0]
    hh, data = b[0], b[1:]
    si = hh.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(r[si]) for r in data if r[si].isdigit())
    cls = collections.Counter()
    for r in data:
        if not r[si].isdigit():
            continue
        op = r[1].split()[0] if not r[1].strip().startswith("@") else r[1].split()[1]
        op = op.split(".")[0]
        cls[op] += int(r[si])
    print(f"  warp-stall samples: {tot}; by opcode (share):")
    for op, n in cls.most_common(16):
        print(f"    {op:12s} {n / tot:6.3f}")
    print(f"  top {top} instructions:")
    for r in sorted(data, key=lambda r: -int(r[si]) if r[si].isdigit() else 0)[:top]:
        print(f"    {r[si]:>6s} {r[1][:100]}")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, data = rows[hi], rows[hi + 1:]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    mi = h.index("Metric Name")
    ui = h.index("Metric Unit") if "Metric Unit" in h else None
    to_ns = {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}
    agg = collections.defaultdict(list)
    for r in data:
        # only the duration rows: a launch list taken with other metrics has bytes/cycles rows too
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            scale = to_ns.get(r[ui], 1.0) if ui is not None else 1.0
            agg[r[ki].split("(")[0][:60]].append(float(r[vi].replace(",", "")) * scale)
    tot = sum(sum(v) for v in agg.values())
    print(f"launch list {path}: {sum(len(v) for v in agg.values())} launches, {tot / 1e3:.1f} us total (ncu: serialised, cold)")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"  {k:60s} n={len(v):5d} mean={sum(v) / len(v) / 1e3:9.2f} us  share={sum(v) / tot:.3f}")


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], int(sys.argv[4]) if len(sys.argv) > 4 else 25)
    else:
        launches(sys.argv[2])
