#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out/kw1; mkdir -p $O
SPA_KW=1 timeout 600 python -m pytest tests/test_gpu_fp8.py -x -q > $O/pytest_fp8_kw1.log 2>&1; echo "fp8 tests kw1 rc=$?"; tail -n 2 $O/pytest_fp8_kw1.log
for kw in 2 1; do
  for rep in 1 2; do
    SPA_KW=$kw timeout 600 python bench.py --kv fp8 --steps 10 --warmup 3 --no-e2e > $O/fp8_kw${kw}_$rep.json 2> $O/fp8_kw$kw.err
    python -c "import json,sys; d=json.loads(open('$O/fp8_kw${kw}_$rep.json').read().strip().splitlines()[-1]); print('kw$kw', d['value'], d['per_window']['0']['layer_ms'] if 'per_window' in d else d.get('extra',{}).get('per_window'))" 2>&1 | tail -1
    SPA_KW=$kw timeout 600 python bench.py --kv fp8 --config gemma --steps 5 --warmup 3 --no-e2e > $O/fp8g_kw${kw}_$rep.json 2> $O/fp8g_kw$kw.err
    python -c "import json,sys; d=json.loads(open('$O/fp8g_kw${kw}_$rep.json').read().strip().splitlines()[-1]); print('gemma kw$kw', d['value'], {k:v['layer_ms'] for k,v in d['per_window'].items()})" 2>&1 | tail -1
  done
done
SPA_KW=1 timeout 300 python scripts/trace_timeline.py qwen --kv fp8 > $O/tl_fp8_kw1.txt 2>&1
