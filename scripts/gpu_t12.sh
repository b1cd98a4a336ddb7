#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out/t12; mkdir -p $O
pw() { python -c "import json,sys; d=json.loads(open('$1').read().strip().splitlines()[-1]); print('$1', round(d['value'],1), {k:round(v['layer_ms']*1000,1) for k,v in d['per_window'].items()}, round(d['roofline']['frac'],3))" 2>&1 | tail -1; }
SPA_LIB=libspa_t12.so SPA_TEAMS=12 timeout 600 python -m pytest tests/test_gpu_fp8.py -x -q -k "qwen_shape or single_key or sliding" > $O/pytest.log 2>&1; echo "t12 parity rc=$?"; tail -n 1 $O/pytest.log
for rep in 1 2; do
  timeout 600 python bench.py --kv fp8 --steps 10 --warmup 3 --no-e2e > $O/f_main.json 2> $O/err; pw $O/f_main.json
  SPA_LIB=libspa_t12.so SPA_TEAMS=12 timeout 600 python bench.py --kv fp8 --steps 10 --warmup 3 --no-e2e > $O/f_t12.json 2>> $O/err; pw $O/f_t12.json
  SPA_LIB=libspa_t12.so SPA_TEAMS=12 timeout 600 python bench.py --kv fp8 --config gemma --steps 5 --warmup 3 --no-e2e > $O/fg_t12.json 2>> $O/err; pw $O/fg_t12.json
done
SPA_LIB=libspa_t12.so SPA_TEAMS=12 timeout 300 python scripts/trace_timeline.py qwen --kv fp8 > $O/tl_t12.txt 2>&1
