#!/bin/bash
# A/B: main library vs one variant; parity subset on main first.  Usage: gpu_ab2.sh VARIANT
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out/ab2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp8.py tests/test_gpu_window_release.py -x -q > $O/pytest.log 2>&1; echo "parity rc=$?"; tail -n 1 $O/pytest.log
pw() { python -c "import json,sys; d=json.loads(open('$1').read().strip().splitlines()[-1]); print('$1', round(d['value'],1), {k:round(v['layer_ms']*1000,1) for k,v in d['per_window'].items()}, round(d['roofline']['frac'],3))" 2>&1 | tail -1; }
for rep in 1 2; do
for v in main $1; do
  if [ "$v" = "main" ]; then L=libspa.so; else L=libspa_$v.so; fi
  SPA_LIB=$L timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e > $O/q_$v.json 2> $O/err; pw $O/q_$v.json
  SPA_LIB=$L timeout 600 python bench.py --config gemma --steps 5 --warmup 3 --no-e2e > $O/g_$v.json 2>> $O/err; pw $O/g_$v.json
  SPA_LIB=$L timeout 600 python bench.py --kv fp8 --steps 10 --warmup 3 --no-e2e > $O/f_$v.json 2>> $O/err; pw $O/f_$v.json
done
done
timeout 300 python scripts/trace_timeline.py qwen > $O/tl_q_main.txt 2>&1
timeout 300 python scripts/trace_timeline.py gemma --window 1024 > $O/tl_g_main.txt 2>&1
