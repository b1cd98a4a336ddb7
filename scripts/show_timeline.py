"""Print a compact table of scripts/trace_timeline.py output (jsonl)."""
import json
import sys

for path in sys.argv[1:]:
    for line in open(path):
        d = json.loads(line)
        t, s = d["trace"], d["stats"]
        r = lambda xs: [round(x, 1) for x in xs] if xs else xs  # noqa: E731
        print(f"{d['workload']:>12} N={d['N']:4d} items={s['n_items']:5d} rec={s['n_records']:4d} "
              f"eager={d['eager_chained_us']:7.1f} graph={d['graph_chained_us']:7.1f} host={d['host_us_per_call']:5.1f} "
              f"GB/s={d['graph_gbs']:6.0f} {d.get('env', '')}")
        print(f"{'':14}first={r(t['first_item_start_us'])} last_end={r(t['last_item_end_us'])} "
              f"merge={t['merge_tasks']}:{r(t['merge_us'])} exit={r(t['exit_us'])} busy={t['busy_frac']:.2f}")
        if t.get("merge_pop_us"):
            print(f"{'':14}merge pop={r(t['merge_pop_us'])} wait={r(t.get('merge_wait_us'))} merge={r(t['merge_dur_us'])} "
                  f"end={r(t['merge_end_us'])} count_lag={r(t.get('count_lag_us'))}")
        if "rates" in d:
            print(f"{'':14}rates pages/us team={r(d['rates']['pages_per_us'])} by_slot={r(d['rates']['by_slot'])} "
                  f"cta={r(d['rates']['cta_mean_pages_per_us'])} gaps={r(d['rates'].get('gap_us'))} x{d['rates'].get('gaps_per_team', 0):.1f}")
        if "subtasks_per_warp_even_odd" in t:
            print(f"{'':14}subtasks/warp even,odd={r(t['subtasks_per_warp_even_odd'])} first pop even,odd={r(t['tail_entry_even_odd_us'])}")
