#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out/extsplit2; mkdir -p $O
for dv in 1 1.1 1.2 1.3; do
  SPA_SPLIT_DIV=$dv timeout 600 python scripts/bench_extend.py --max-rows 128 --no-parity > $O/ext_div$dv.json 2>>$O/err.txt; python -c "import json; d=json.load(open('$O/ext_div$dv.json')); print('div $dv', round(d['layer_us'],1), d['stats']['n_items'], d['stats']['n_records'])"
done
