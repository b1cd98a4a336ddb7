#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out/k7; mkdir -p $O
pw() { python -c "import json,sys; d=json.loads(open('$1').read().strip().splitlines()[-1]); print('$1', round(d['value'],1), {k:round(v['layer_ms']*1000,1) for k,v in d['per_window'].items()}, d['roofline']['frac'])" 2>&1 | tail -1; }
SPA_LIB=libspa_k7.so SPA_KW=1 SPA_TEAMS=7 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $O/pytest_k7.log 2>&1; echo "parity k7 rc=$?"; tail -n 1 $O/pytest_k7.log
for cfg in qwen gemma long; do
  a=""; [ $cfg != qwen ] && a="--config $cfg"
  timeout 600 python bench.py $a --steps 5 --warmup 3 --no-e2e > $O/${cfg}_main.json 2> $O/err; pw $O/${cfg}_main.json
  SPA_LIB=libspa_k7.so SPA_KW=1 SPA_TEAMS=7 timeout 600 python bench.py $a --steps 5 --warmup 3 --no-e2e > $O/${cfg}_k7.json 2>> $O/err; pw $O/${cfg}_k7.json
done
