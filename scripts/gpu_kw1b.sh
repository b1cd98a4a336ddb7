#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out/kw1b; mkdir -p $O
SPA_KW=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_window_release.py -x -q > $O/pytest_kw1.log 2>&1; echo "parity kw1 rc=$?"; tail -n 2 $O/pytest_kw1.log
pw() { python -c "import json,sys; d=json.loads(open('$1').read().strip().splitlines()[-1]); print('$1', round(d['value'],1), {k:round(v['layer_ms']*1000,1) for k,v in d['per_window'].items()}, d['roofline']['frac'])" 2>&1 | tail -1; }
for kw in 2 1; do
  SPA_KW=$kw timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e > $O/bf16_kw$kw.json 2> $O/bf16_kw$kw.err; pw $O/bf16_kw$kw.json
  SPA_KW=$kw timeout 600 python bench.py --config gemma --steps 5 --warmup 3 --no-e2e > $O/gemma_kw$kw.json 2> $O/gemma_kw$kw.err; pw $O/gemma_kw$kw.json
  SPA_KW=$kw timeout 600 python bench.py --config long --steps 3 --warmup 3 --no-e2e > $O/long_kw$kw.json 2> $O/long_kw$kw.err; pw $O/long_kw$kw.json
done
SPA_KW=1 timeout 300 python scripts/trace_timeline.py qwen > $O/tl_bf16_kw1.txt 2>&1
SPA_KW=1 timeout 300 python scripts/trace_timeline.py gemma --window 1024 > $O/tl_gemma_kw1.txt 2>&1
timeout 300 python scripts/trace_timeline.py gemma --window 1024 > $O/tl_gemma_kw2.txt 2>&1
