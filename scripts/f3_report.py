"""F3: SPAgent's speculation selection driven by measured B200 costs.

    python scripts/f3_report.py [--table profiles/r02_th_table.csv] [--out profiles/r02_f3_admission.json]

1. Calibrates SPEC's affine-plus-knee T_h (paper Table I, Eqs. 3-4,
   /root/reference/PAPER.md:311-340) by least squares on the attention-time table
   scripts/th_table.py measured with this library's kernels (decode-only rows, hybrid rows
   with |S| prefilling forks of L_s tokens, and decode rows with k forked samples per agent).
2. Runs Algorithm 1 at engine loads N = 1..256 with
   every agent a fresh candidate (k = 3, the paper's default), once with the
   measured per-fork decode slope gamma_f (prefix sharing: a fork reads only its tail) and
   once with gamma_f = gamma (no sharing, SPEC's model), and reports the admitted |S|.

The measured T_h is the ATTENTION share of an engine step (the hot path this repo builds);
the paper's T_h also holds the model's GEMMs, so absolute admission counts here are those
of an attention-only engine (reading F3-b).  Host logic only: no GPU needed.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_20048_b200 import scheduler  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--table", default=os.path.join(ROOT, "profiles", "r02_th_table.csv"))
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_f3_admission.json"))
    ap.add_argument("--loads", default="1,2,4,8,16,32,64,96,128,192,256")
    ap.add_argument("--k", type=int, default=3)
    ap.add_argument("--max-rel-err", type=float, default=10.0, help="refuse a worse fit (default: report it)")
    a = ap.parse_args()
    table = scheduler.load_table(a.table)
    params, rep = scheduler.calibrate(table, max_rel_err=a.max_rel_err, relative=True)
    plain = scheduler.CostModelParams(params.base_step_time, params.decode_cost_per_request, params.decode_knee,
                                      params.decode_slowdown, params.prefill_fixed_cost,
                                      params.prefill_cost_per_token, None)
    loads = [int(x) for x in a.loads.split(",")]
    shared = scheduler.admitted_vs_load(params, loads, k=a.k)
    unshared = scheduler.admitted_vs_load(plain, loads, k=a.k)
    res = {"table": os.path.relpath(a.table, ROOT), "calibration": rep,
           "params": {k: getattr(params, k) for k in ("base_step_time", "decode_cost_per_request", "decode_knee",
                                                       "decode_slowdown", "prefill_fixed_cost",
                                                       "prefill_cost_per_token", "decode_cost_per_fork")},
           "k": a.k,
           "admitted": [{"N": n, "S_shared": s1, "T_r_shared": b1, "S_unshared": s2, "T_r_unshared": b2}
                        for (n, s1, b1), (_, s2, b2) in zip(shared, unshared)]}
    print(f"calibrated on {rep['rows']} rows: max rel err {rep['max_rel_err']:.1%}, mean {rep['mean_rel_err']:.1%}")
    print("params:", json.dumps(res["params"]))
    print(f"{'N':>5} {'|S| shared':>11} {'|S| unshared':>13}")
    for r in res["admitted"]:
        print(f"{r['N']:5d} {r['S_shared']:11d} {r['S_unshared']:13d}")
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
