#!/bin/bash
# round 2: ext kernel with K / V producer warps (multi-lane TMA issue): parity, bench, trace
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_extend_tc.py tests/test_gpu_extend.py tests/test_gpu_umma.py -m gpu -q -x > gpurun_out/r2i_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/r2i_pytest.log
timeout 300 python scripts/bench_extend.py --max-rows 128 > gpurun_out/r2i_ext.json 2> gpurun_out/r2i_ext.err; echo "ext rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r2i_ext.json')); print(round(d['layer_us'],1), 'us', round(d['hbm_gbs_algorithmic']), 'GB/s', round(d['roofline']['frac'],3), round(d['tflops']), 'TF/s', d.get('parity'))"
timeout 300 python scripts/ext_trace.py > gpurun_out/r2i_ext_trace.txt 2>&1; echo "trace rc=$?"; head -n 16 gpurun_out/r2i_ext_trace.txt
