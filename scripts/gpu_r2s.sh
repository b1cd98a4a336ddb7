#!/bin/bash
# round 2: split-size sensitivity of the decode step (bf16 / fp8 Qwen, Gemma local) + long-32k 64-layer bench
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
rm -f gpurun_out/r2s_timeline.jsonl
for S in 0 16 24 32 48; do
  timeout 300 python scripts/trace_timeline.py qwen --split $S --out gpurun_out/r2s_timeline.jsonl > /dev/null 2>> gpurun_out/r2s.err
  timeout 300 python scripts/trace_timeline.py qwen --kv fp8 --split $S --out gpurun_out/r2s_timeline.jsonl > /dev/null 2>> gpurun_out/r2s.err
done
for S in 0 16 32; do
  timeout 300 python scripts/trace_timeline.py gemma --window 1024 --split $S --out gpurun_out/r2s_timeline.jsonl > /dev/null 2>> gpurun_out/r2s.err
done
python - <<'PY'
import json
for l in open('gpurun_out/r2s_timeline.jsonl'):
    d=json.loads(l); t=d['trace']
    print(d['workload'], d['kv'], 'graph', round(d['graph_chained_us'],1), 'GB/s', round(d['graph_gbs']), 'items', d['stats']['n_items'], 'recs', d['stats']['n_records'], 'last', [round(x,1) for x in t['last_item_end_us']], 'merge', t.get('merge_us'), 'busy', round(t['busy_frac'],3))
PY
timeout 900 python bench.py --config long --steps 5 --warmup 3 > gpurun_out/r2s_bench_long.json 2> gpurun_out/r2s_bench_long.err; echo "long rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r2s_bench_long.json')); print('long', round(d['value']), d['unit'], round(d['ms_per_step'],1), 'ms', d['config']['layer_calls_per_step'], 'e2e', d.get('e2e',{}).get('value'), round(d['roofline']['frac'],3))"
