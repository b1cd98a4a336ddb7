#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
rm -f gpurun_out/r2u_timeline.jsonl
timeout 300 python scripts/trace_timeline.py qwen --out gpurun_out/r2u_timeline.jsonl > /dev/null 2>> gpurun_out/r2u.err
timeout 300 python scripts/trace_timeline.py qwen --split 48 --out gpurun_out/r2u_timeline.jsonl > /dev/null 2>> gpurun_out/r2u.err
timeout 300 python scripts/trace_timeline.py qwen --kv fp8 --out gpurun_out/r2u_timeline.jsonl > /dev/null 2>> gpurun_out/r2u.err
timeout 300 python scripts/trace_timeline.py gemma --window 1024 --out gpurun_out/r2u_timeline.jsonl > /dev/null 2>> gpurun_out/r2u.err
python - <<'PY'
import json
for l in open('gpurun_out/r2u_timeline.jsonl'):
    d=json.loads(l); t=d['trace']
    print(d['workload'], d['kv'], 'graph', round(d['graph_chained_us'],1), 'items', d['stats']['n_items'], {k:[round(x,2) for x in v] for k,v in t['item_phases_us'].items()})
PY
