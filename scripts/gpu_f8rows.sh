#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out/f8rows; mkdir -p $O
for w in sweep:256:0.75 sweep:64:0.75 sweep:256:0.5; do
 for r in 0 16; do
  timeout 300 python scripts/trace_timeline.py $w --kv fp8 --rows $r > $O/tl_${w}_r$r.txt 2>&1
  python - $O/tl_${w}_r$r.txt $w $r <<'PY'
import json,sys
for line in open(sys.argv[1]):
    if line.startswith('{'):
        d=json.loads(line); print(sys.argv[2], 'rows', sys.argv[3], 'graph_us', round(d['graph_chained_us'],1), 'alg GB/s', round(d.get('graph_gbs',0)), d['stats']['n_items'], d['stats']['rows_max'])
PY
 done
done
