"""Planner statistics on CPU (metadata-only pool): items, records, split size, planning time."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from test_planner import build  # noqa: E402
from spa_inputs import workloads  # noqa: E402
from paper_2511_20048_b200 import spa  # noqa: E402

cases = [("qwen", workloads.qwen()), ("long", workloads.long32k()), ("gemma", workloads.gemma())]
cases += [(f"sweep{b}:{f}", workloads.sweep(b, f)) for b in (1, 8, 32, 64, 256) for f in (0, 0.5)]
for name, rec in cases:
    pool, reqs = build(rec)
    for w in sorted({0, 1024 if name == "gemma" else 0}):
        plan = spa.Plan(pool)
        t = time.perf_counter()
        plan.plan(reqs, w)
        dt = time.perf_counter() - t
        st = plan.stats()
        d = plan.debug_array(0)
        print(f"{name:>12} w={w:5d} items={st['n_items']:6d} rec={st['n_records']:5d} max_desc_pages={max(x[1] for x in d):5d} "
              f"plan_ms={dt * 1e3:6.2f}")
