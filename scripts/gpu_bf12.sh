#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out/bf12; mkdir -p $O
run() { timeout 300 python scripts/trace_timeline.py $2 > $O/tl_$1.txt 2>&1
  python - $O/tl_$1.txt $1 <<'PY'
import json,sys
for line in open(sys.argv[1]):
    if line.startswith('{'):
        d=json.loads(line); t=d['trace']; print(sys.argv[2], 'graph_us', round(d['graph_chained_us'],1), 'items', d['stats']['n_items'], 'rec', d['stats']['n_records'], 'busy', round(t['busy_frac'],3), 'last_end', t['last_item_end_us'])
    elif 'rror' in line: print(sys.argv[2], line.strip()[:200])
PY
}
run g_base "gemma --window 1024 --teams 4"
SPA_KW=1 SPA_TEAMS=12 run g_kw1t12 "gemma --window 1024"
SPA_KW=1 SPA_TEAMS=12 run g_kw1t12m2 "gemma --window 1024 --merge 2"
SPA_KW=1 SPA_TEAMS=12 run q_kw1t12 "qwen"
SPA_KW=1 SPA_TEAMS=12 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "window or tiny" > $O/pytest.log 2>&1; echo "parity rc=$?"; tail -n 1 $O/pytest.log
