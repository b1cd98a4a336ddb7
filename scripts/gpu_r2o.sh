#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_extend_tc.py tests/test_gpu_extend.py tests/test_gpu_workspace.py -m gpu -q -x > gpurun_out/r2o_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 3 gpurun_out/r2o_pytest.log
timeout 300 python scripts/bench_extend.py --max-rows 128 > gpurun_out/r2o_ext.json 2>/dev/null
python -c "import json,sys; d=json.load(open('gpurun_out/r2o_ext.json')); print(round(d['layer_us'],1), 'us', round(d['hbm_gbs_algorithmic']), 'GB/s', round(d['roofline']['frac'],3), d['parity'])"
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2o_launches.csv python scripts/bench_extend.py --max-rows 128 --profile > /dev/null 2>&1
grep gpu__time gpurun_out/r2o_launches.csv | awk -F'","' '{print $5, $NF}' | head -4
