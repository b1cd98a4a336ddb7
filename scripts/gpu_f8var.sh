#!/bin/bash
# fp8 consumer variants: parity (fp8 tests) + config 1 / Gemma fp8 benches per variant
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out/f8var; mkdir -p $O
pw() { python -c "import json,sys; d=json.loads(open('$1').read().strip().splitlines()[-1]); print('$1', round(d['value'],1), {k:round(v['layer_ms']*1000,1) for k,v in d['per_window'].items()}, round(d['roofline']['frac'],3))" 2>&1 | tail -1; }
for v in $1; do
  SPA_LIB=libspa_$v.so timeout 600 python -m pytest tests/test_gpu_fp8.py -x -q > $O/pytest_$v.log 2>&1; echo "$v fp8 parity rc=$?"; tail -n 1 $O/pytest_$v.log
done
for rep in 1 2; do
for v in main $1; do
  if [ "$v" = "main" ]; then L=libspa.so; else L=libspa_$v.so; fi
  SPA_LIB=$L timeout 600 python bench.py --kv fp8 --steps 10 --warmup 3 --no-e2e > $O/f_$v.json 2> $O/err; pw $O/f_$v.json
  SPA_LIB=$L timeout 600 python bench.py --kv fp8 --config gemma --steps 5 --warmup 3 --no-e2e > $O/fg_$v.json 2>> $O/err; pw $O/fg_$v.json
done
done
SPA_LIB=libspa_qk2.so timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e > $O/q_qk2.json 2>> $O/err; pw $O/q_qk2.json
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e > $O/q_main.json 2>> $O/err; pw $O/q_main.json
