#!/bin/bash
# Gemma local-layer (W = 1024) geometry options on the trace tool (8 resident layers, chained)
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out/gl; mkdir -p $O
run() { timeout 300 python scripts/trace_timeline.py gemma --window 1024 $2 > $O/tl_$1.txt 2>&1
  python - $O/tl_$1.txt $1 <<'PY'
import json,sys
for line in open(sys.argv[1]):
    if line.startswith('{'):
        d=json.loads(line); t=d['trace']; print(sys.argv[2], 'graph_us', round(d['graph_chained_us'],1), 'items', d['stats']['n_items'], 'rec', d['stats']['n_records'], 'busy', round(t['busy_frac'],3), 'first', t['first_item_start_us'][1], 'last_end', t['last_item_end_us'])
PY
}
run t4 "--teams 4"
run t2 "--teams 2"
run t1 "--teams 1"
SPA_KW=1 run kw1 ""
run t4b "--teams 4"
for dv in 0.75 0.5; do SPA_SPLIT_DIV=$dv run div$dv "--teams 4"; done
SPA_POLL_MIN=16 SPA_POLL_MAX=64 run poll "--teams 4"
