#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out/m32; mkdir -p $O
run() { timeout 300 python scripts/trace_timeline.py $2 > $O/tl_$1.txt 2>&1
  python - $O/tl_$1.txt $1 <<'PY'
import json,sys
for line in open(sys.argv[1]):
    if line.startswith('{'):
        d=json.loads(line); t=d['trace']; print(sys.argv[2], 'graph_us', round(d['graph_chained_us'],1), 'items', d['stats']['n_items'], 'rec', d['stats']['n_records'], 'rows', d['stats']['rows_max'], 'busy', round(t['busy_frac'],3))
PY
}
for m in 0 2; do
  run bf_m$m "sweep:256:0.75 --rows 0 --merge $m"
  run f8_m$m "sweep:256:0.75 --rows 0 --kv fp8 --merge $m"
  run bf64_m$m "sweep:64:0.75 --rows 0 --merge $m"
  run long_m$m "long --merge $m"
done
