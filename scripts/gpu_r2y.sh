#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
for D in "" 1.25 1.5 2 3; do
  if [ -z "$D" ]; then unset SPA_SPLIT_DIV; else export SPA_SPLIT_DIV=$D; fi
  timeout 300 python scripts/bench_extend.py --max-rows 128 --no-parity --cpu-seconds 0 > gpurun_out/r2y_ext_$D.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/r2y_ext_$D.json')); print('div=$D', round(d['layer_us'],1), 'us', round(d['roofline']['frac'],3), d['stats']['n_items'], d['stats']['n_records'])"
done
