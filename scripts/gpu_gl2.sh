#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out/gl2; mkdir -p $O
run() { timeout 300 python scripts/trace_timeline.py gemma --window 1024 $2 > $O/tl_$1.txt 2>&1
  python - $O/tl_$1.txt $1 <<'PY'
import json,sys
for line in open(sys.argv[1]):
    if line.startswith('{'):
        d=json.loads(line); t=d['trace']; print(sys.argv[2], 'graph_us', round(d['graph_chained_us'],1), 'items', d['stats']['n_items'], 'rec', d['stats']['n_records'], 'busy', round(t['busy_frac'],3), 'first', t['first_item_start_us'][1], 'last_end', t['last_item_end_us'], 'merge_end', t['merge_end_us'][-1] if t.get('merge_end_us') else None)
PY
}
for dv in 1.5 2 3 4; do SPA_KW=1 SPA_SPLIT_DIV=$dv run kw1_div$dv ""; done
for dv in 1.5 2; do SPA_SPLIT_DIV=$dv run kw2_div$dv "--teams 4"; done
