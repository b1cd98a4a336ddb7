#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out/f8split; mkdir -p $O
pw() { python -c "import json,sys; d=json.loads(open('$1').read().strip().splitlines()[-1]); print('$1', round(d['value'],1), {k:(round(v['layer_ms']*1000,1), v['n_records']) for k,v in d['per_window'].items()}, d['roofline']['frac'])" 2>&1 | tail -1; }
timeout 600 python bench.py --kv fp8 --steps 10 --warmup 3 --no-e2e > $O/f8_default.json 2>$O/err.txt; pw $O/f8_default.json
for dv in 1.5 2 3; do
  SPA_SPLIT_DIV=$dv timeout 600 python bench.py --kv fp8 --steps 10 --warmup 3 --no-e2e > $O/f8_div$dv.json 2>>$O/err.txt; pw $O/f8_div$dv.json
done
for dv in 1.5 2; do
  SPA_SPLIT_DIV=$dv timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e > $O/bf_div$dv.json 2>>$O/err.txt; pw $O/bf_div$dv.json
done
SPA_SPLIT_DIV=2 timeout 300 python scripts/trace_timeline.py qwen --kv fp8 > $O/tl_fp8_div2.txt 2>&1
