#!/bin/bash
# round 2: tail-fraction cuts (small final items for the dynamic queue's drain)
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
rm -f gpurun_out/r2t_timeline.jsonl
for TF in 0 0.1 0.2 0.35; do for TD in 4 8; do
  [ "$TF" = "0" ] && [ "$TD" = "8" ] && continue
  SPA_TAIL_FRAC=$TF SPA_TAIL_DIV=$TD timeout 300 python scripts/trace_timeline.py qwen --out gpurun_out/r2t_timeline.jsonl > /dev/null 2>> gpurun_out/r2t.err
  SPA_TAIL_FRAC=$TF SPA_TAIL_DIV=$TD timeout 300 python scripts/trace_timeline.py qwen --kv fp8 --out gpurun_out/r2t_timeline.jsonl > /dev/null 2>> gpurun_out/r2t.err
  echo "$TF $TD" >> gpurun_out/r2t_keys.txt
done; done
python - <<'PY'
import json
for l in open('gpurun_out/r2t_timeline.jsonl'):
    d=json.loads(l); t=d['trace']
    print(d['workload'], d['kv'], 'graph', round(d['graph_chained_us'],1), 'GB/s', round(d['graph_gbs']), 'items', d['stats']['n_items'], 'recs', d['stats']['n_records'], 'last', [round(x,1) for x in t['last_item_end_us']], 'merge', t.get('merge_us'), 'busy', round(t['busy_frac'],3))
PY
cat gpurun_out/r2t_keys.txt
