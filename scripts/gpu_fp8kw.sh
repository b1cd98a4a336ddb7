#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out/fp8kw; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -n 2 $O/pytest_gpu.log
pw() { python -c "import json,sys; d=json.loads(open('$1').read().strip().splitlines()[-1]); print('$1', round(d['value'],1), {k:round(v['layer_ms']*1000,1) for k,v in d['per_window'].items()}, d['roofline']['frac'])" 2>&1 | tail -1; }
timeout 600 python bench.py --kv fp8 --steps 20 --warmup 5 > $O/fp8_qwen.json 2> $O/fp8_qwen.err; pw $O/fp8_qwen.json
timeout 600 python bench.py --kv fp8 --config gemma --steps 10 --warmup 3 --no-e2e > $O/fp8_gemma.json 2> $O/fp8_gemma.err; pw $O/fp8_gemma.json
timeout 600 python bench.py --kv fp8 --config long --steps 5 --warmup 3 --no-e2e > $O/fp8_long.json 2> $O/fp8_long.err; pw $O/fp8_long.json
timeout 300 python scripts/trace_timeline.py qwen --kv fp8 > $O/tl_fp8.txt 2>&1
timeout 300 python scripts/trace_timeline.py sweep:256:0.75 --kv fp8 --rows 0 > $O/tl_fp8_sweep.txt 2>&1
SPA_KW=2 timeout 300 python scripts/trace_timeline.py sweep:256:0.75 --kv fp8 --rows 0 > $O/tl_fp8_sweep_kw2.txt 2>&1
