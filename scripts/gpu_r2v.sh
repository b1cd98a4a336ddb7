#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_full.py tests/test_gpu_extend_tc.py tests/test_gpu_fp8.py -m gpu -q -x > gpurun_out/r2v_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/r2v_pytest.log
bash scripts/gpu_r2u.sh
python - <<'PY'
import json
for l in open('gpurun_out/r2u_timeline.jsonl'):
    d=json.loads(l); t=d['trace']
    print(d['workload'], d['kv'], d['stats']['n_items'], 'graph', round(d['graph_chained_us'],1), {k:[round(x,2) for x in v] for k,v in t['item_phases_us'].items() if k.startswith('epi') or k=='setup'})
PY
