#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out/rec; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -n 1 $O/pytest.log
pw() { python -c "import json,sys; d=json.loads(open('$1').read().strip().splitlines()[-1]); print('$1', round(d['value'],1), {k:(round(v['layer_ms']*1000,1), v['n_records']) for k,v in d['per_window'].items()}, round(d['roofline']['frac'],3), d['roofline']['kernel'], d['gpu_launches'], d.get('e2e') and round(d['e2e']['value']))" 2>&1 | tail -1; }
timeout 900 python bench.py --config long --steps 5 --warmup 3 > $O/long.json 2> $O/err; pw $O/long.json
timeout 900 python bench.py --steps 20 --warmup 5 > $O/qwen.json 2>> $O/err; pw $O/qwen.json
timeout 900 python bench.py --config gemma --steps 10 --warmup 3 > $O/gemma.json 2>> $O/err; pw $O/gemma.json
