#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out/mm; mkdir -p $O
run() { timeout 300 python scripts/trace_timeline.py $2 > $O/tl_$1.txt 2>&1
  python - $O/tl_$1.txt $1 <<'PY'
import json,sys
for line in open(sys.argv[1]):
    if line.startswith('{'):
        d=json.loads(line); t=d['trace']; print(sys.argv[2], 'graph_us', round(d['graph_chained_us'],1), 'items', d['stats']['n_items'], 'rec', d['stats']['n_records'], 'busy', round(t['busy_frac'],3), 'last_end', t['last_item_end_us'], 'merge_end', t['merge_end_us'][-1] if t.get('merge_end_us') else None)
PY
}
for m in 0 1 2; do
  run q_m$m "qwen --merge $m"
  run f_m$m "qwen --kv fp8 --merge $m"
  run g_m$m "gemma --window 1024 --teams 4 --merge $m"
done
