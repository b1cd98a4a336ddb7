#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2r_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/r2r_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e > gpurun_out/r2r_bench_qwen.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/r2r_bench_qwen.json')); print('qwen', round(d['value']), round(d['layer_ms']*1e3,1), 'us', round(d['roofline']['frac'],3), d['plan'])"
timeout 900 python bench.py --config gemma --steps 10 --warmup 3 --no-e2e > gpurun_out/r2r_bench_gemma.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/r2r_bench_gemma.json')); print('gemma', round(d['value']), {k:(round(v['layer_ms']*1e3,1), round(v['gbs'])) for k,v in d['per_window'].items()})"
timeout 300 python scripts/bench_extend.py --max-rows 128 > gpurun_out/r2r_ext.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/r2r_ext.json')); print('ext', round(d['layer_us'],1), 'us', round(d['roofline']['frac'],3), d['stats']['n_items'], d['stats']['n_records'], d['parity'])"
timeout 300 python scripts/trace_timeline.py gemma --window 1024 --out gpurun_out/r2r_timeline.jsonl > /dev/null 2>> gpurun_out/r2r_timeline.err
python - <<'PY'
import json
for l in open('gpurun_out/r2r_timeline.jsonl'):
    d=json.loads(l); t=d['trace']
    print(d['workload'], 'graph', round(d['graph_chained_us'],1), 'GB/s', round(d['graph_gbs']), 'first', [round(x,1) for x in t['first_item_start_us']], 'last', [round(x,1) for x in t['last_item_end_us']], 'busy', round(t['busy_frac'],3), 'items/team', t['items_per_team'], 'merge', t.get('merge_us'), 'rates', [round(x,2) for x in d['rates']['pages_per_us']])
PY
