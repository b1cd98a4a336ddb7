#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out/q12; mkdir -p $O
run() { timeout 300 python scripts/trace_timeline.py $2 > $O/tl_$1.txt 2>&1
  python - $O/tl_$1.txt $1 <<'PY'
import json,sys
for line in open(sys.argv[1]):
    if line.startswith('{'):
        d=json.loads(line); t=d['trace']; print(sys.argv[2], 'graph_us', round(d['graph_chained_us'],1), 'items', d['stats']['n_items'], 'rec', d['stats']['n_records'], 'busy', round(t['busy_frac'],3))
    elif 'rror' in line: print(sys.argv[2], line.strip()[:200])
PY
}
run q8 "qwen --kv fp8"
SPA_TEAMS=12 run q12 "qwen --kv fp8"
run l8 "long --kv fp8"
SPA_TEAMS=12 run l12 "long --kv fp8"
run s8 "sweep:128:1 --kv fp8"
SPA_TEAMS=12 run s12 "sweep:128:1 --kv fp8"
