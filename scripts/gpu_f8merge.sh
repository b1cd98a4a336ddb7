#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out/f8m; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fp8.py tests/test_gpu_parity.py tests/test_gpu_fused_gather.py tests/test_gpu_workspace.py -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -n 1 $O/pytest.log
pw() { python -c "import json,sys; d=json.loads(open('$1').read().strip().splitlines()[-1]); print('$1', round(d['value'],1), {k:round(v['layer_ms']*1000,1) for k,v in d['per_window'].items()}, round(d['roofline']['frac'],3), d['roofline']['kernel'], d['gpu_launches'], d.get('e2e',{}) and round(d['e2e']['value']))" 2>&1 | tail -1; }
for rep in 1 2; do
timeout 600 python bench.py --kv fp8 --steps 20 --warmup 5 > $O/fp8_qwen_$rep.json 2> $O/err; pw $O/fp8_qwen_$rep.json
done
timeout 600 python bench.py --kv fp8 --config gemma --steps 10 --warmup 3 > $O/fp8_gemma.json 2>> $O/err; pw $O/fp8_gemma.json
timeout 600 python bench.py --kv fp8 --config long --steps 5 --warmup 3 > $O/fp8_long.json 2>> $O/err; pw $O/fp8_long.json
timeout 600 python bench.py --kv fp8 --merge-mode 0 --steps 10 --warmup 3 --no-e2e > /dev/null 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file $O/fp8_launches.csv python bench.py --kv fp8 --steps 2 --warmup 2 --profile --no-e2e > /dev/null 2>&1
python scripts/ncu_summary.py launches $O/fp8_launches.csv > $O/fp8_launches.txt 2>&1; cat $O/fp8_launches.txt | head -5
