#!/bin/bash
# round 2: folded member tails (reading #19): full GPU suite, bench (qwen, gemma), extend bench, sweep point
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2q_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 3 gpurun_out/r2q_pytest.log
for F in 1 0; do
SPA_FOLD=$F timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e > gpurun_out/r2q_bench_qwen_$F.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/r2q_bench_qwen_$F.json')); print('qwen fold=$F', round(d['value']), round(d['layer_ms']*1e3,1), 'us', round(d['roofline']['frac'],3), d['plan'])"
SPA_FOLD=$F timeout 900 python bench.py --config gemma --steps 10 --warmup 3 --no-e2e > gpurun_out/r2q_bench_gemma_$F.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/r2q_bench_gemma_$F.json')); print('gemma fold=$F', round(d['value']), {k:(round(v['layer_ms']*1e3,1), round(v['gbs'])) for k,v in d['per_window'].items()})"
SPA_FOLD=$F timeout 300 python scripts/bench_extend.py --max-rows 128 --no-parity --cpu-seconds 0 > gpurun_out/r2q_ext_$F.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/r2q_ext_$F.json')); print('ext fold=$F', round(d['layer_us'],1), 'us', round(d['roofline']['frac'],3), d['stats']['n_items'], d['stats']['n_records'])"
done
