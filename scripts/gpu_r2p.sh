#!/bin/bash
# round 2: fresh Gemma (local/global) and FP8 bench lines + local-layer and fp8 timelines
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 900 python bench.py --config gemma --steps 10 --warmup 3 --no-e2e > gpurun_out/r2p_bench_gemma.json 2> gpurun_out/r2p_bench_gemma.err; echo "gemma rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r2p_bench_gemma.json')); print('gemma', round(d['value']), d['unit'], {k:(round(v['layer_ms']*1e3,1), round(v['gbs'])) for k,v in d['per_window'].items()})"
timeout 900 python bench.py --kv fp8 --steps 10 --warmup 3 --no-e2e > gpurun_out/r2p_bench_fp8.json 2> gpurun_out/r2p_bench_fp8.err; echo "fp8 rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r2p_bench_fp8.json')); print('fp8', round(d['value']), d['unit'], {k:(round(v['layer_ms']*1e3,1), round(v['gbs'])) for k,v in d['per_window'].items()})"
for R in 16 0; do
timeout 300 python scripts/trace_timeline.py gemma --window 1024 --rows $R --out gpurun_out/r2p_timeline.jsonl > /dev/null 2>> gpurun_out/r2p_timeline.err; echo "timeline gemma rows=$R rc=$?"
done
timeout 300 python scripts/trace_timeline.py qwen --kv fp8 --out gpurun_out/r2p_timeline.jsonl > /dev/null 2>> gpurun_out/r2p_timeline.err; echo "timeline fp8 rc=$?"
python - <<'PY'
import json
for l in open('gpurun_out/r2p_timeline.jsonl'):
    d=json.loads(l); t=d['trace']
    print(d['workload'], d['kv'], 'rows', d['rows'], 'eager', round(d['eager_chained_us'],1), 'graph', round(d['graph_chained_us'],1), 'GB/s', round(d['graph_gbs']),
          'first', [round(x,1) for x in t['first_item_start_us']], 'last', [round(x,1) for x in t['last_item_end_us']], 'busy', round(t['busy_frac'],3),
          'items/team', t['items_per_team'], 'rates', [round(x,2) for x in d['rates']['pages_per_us']], 'gap', d['rates']['gap_us'])
PY
