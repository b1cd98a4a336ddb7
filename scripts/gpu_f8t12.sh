#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out/f8t12; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fp8.py tests/test_gpu_window_release.py tests/test_gpu_parity.py -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -n 3 $O/pytest.log
pw() { python -c "import json,sys; d=json.loads(open('$1').read().strip().splitlines()[-1]); print('$1', round(d['value'],1), {k:round(v['layer_ms']*1000,1) for k,v in d['per_window'].items()}, round(d['roofline']['frac'],3), d['gpu_launches'], d.get('e2e',{}) and round(d['e2e']['value']))" 2>&1 | tail -1; }
for rep in 1 2; do
timeout 600 python bench.py --kv fp8 --config gemma --steps 10 --warmup 3 > $O/fp8_gemma_$rep.json 2> $O/err; pw $O/fp8_gemma_$rep.json
done
timeout 600 python bench.py --kv fp8 --steps 10 --warmup 3 --no-e2e > $O/fp8_qwen.json 2>> $O/err; pw $O/fp8_qwen.json
timeout 600 python bench.py --config gemma --steps 5 --warmup 3 --no-e2e > $O/bf16_gemma.json 2>> $O/err; pw $O/bf16_gemma.json
