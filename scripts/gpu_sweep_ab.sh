#!/bin/bash
# A/B of one sweep point (B=256, f=0.75) and config 1 between the main library and a variant
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out/sab; mkdir -p $O
for rep in 1 2 3; do
for v in main $1; do
  if [ "$v" = "main" ]; then L=libspa.so; else L=libspa_$v.so; fi
  for r in 0 32; do
    SPA_LIB=$L timeout 300 python scripts/trace_timeline.py sweep:256:0.75 --rows $r > $O/tl_${v}_$r.txt 2>&1
    python - $O/tl_${v}_$r.txt $v $r <<'PY'
import json,sys
for line in open(sys.argv[1]):
    if line.startswith('{'):
        d=json.loads(line); print(sys.argv[2], 'rows', sys.argv[3], 'graph_us', round(d['graph_chained_us'],1), 'eager', round(d['eager_chained_us'],1), d['stats']['n_items'], d['stats']['rows_max'])
PY
  done
done
done
