#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out/f8s2; mkdir -p $O
run() { timeout 300 python scripts/trace_timeline.py $2 > $O/tl_$1.txt 2>&1
  python - $O/tl_$1.txt $1 <<'PY'
import json,sys
for line in open(sys.argv[1]):
    if line.startswith('{'):
        d=json.loads(line); t=d['trace']; print(sys.argv[2], 'graph_us', round(d['graph_chained_us'],1), 'items', d['stats']['n_items'], 'rec', d['stats']['n_records'], 'busy', round(t['busy_frac'],3), 'last_end', t['last_item_end_us'])
PY
}
run base "qwen --kv fp8"
for dv in 1.25 1.5 2 3; do SPA_SPLIT_DIV=$dv run div$dv "qwen --kv fp8"; done
run gbase "gemma --kv fp8 --window 1024"
SPA_SPLIT_DIV=2 run gdiv2 "gemma --kv fp8 --window 1024"
