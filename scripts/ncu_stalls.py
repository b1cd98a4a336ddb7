"""Stall-reason breakdown of an ncu source-page CSV (--page source --csv --print-source sass):
totals per reason, and the top instructions with their dominant reasons, in program order.
    python scripts/ncu_stalls.py file.csv[.gz] [--top 40]"""
import collections
import csv
import gzip
import io
import sys


def load(path):
    """The first kernel's source table (a capture of several launches repeats the table,
    each behind its own "Kernel Name" line)."""
    f = io.TextIOWrapper(gzip.open(path)) if path.endswith(".gz") else open(path)
    rows = list(csv.reader(f))
    ends = [i for i, r in enumerate(rows) if i > 0 and r and r[0] == "Kernel Name"]
    rows = rows[:ends[0]] if ends else rows
    return rows[1], [r for r in rows[2:] if len(r) == len(rows[1])]


def main():
    path = sys.argv[1]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    h, data = load(path)
    reasons = [c for c in h if c.startswith("stall_") and "(Not Issued)" not in c]
    ri = {r: h.index(r) for r in reasons}
    si = h.index("Warp Stall Sampling (All Samples)")
    tot = collections.Counter()
    for r in data:
        for k, i in ri.items():
            if r[i].isdigit():
                tot[k] += int(r[i])
    all_s = sum(tot.values())
    print(f"samples {all_s}: " + ", ".join(f"{k[6:]} {v / all_s:.3f}" for k, v in tot.most_common(10)))
    idx = sorted(range(len(data)), key=lambda j: -int(data[j][si]) if data[j][si].isdigit() else 0)[:top]
    for j in sorted(idx):
        r = data[j]
        rs = sorted(((int(r[i]), k[6:]) for k, i in ri.items() if r[i].isdigit() and int(r[i]) > 0), reverse=True)[:3]
        print(f"{j:6d} {r[si]:>6s} {r[1].strip()[:60]:60s} " + " ".join(f"{k}:{v}" for v, k in rs))


if __name__ == "__main__":
    main()
