#!/bin/bash
# round 2: ext kernel with 1 or 2 K producer warps: parity + bench + trace
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_extend_tc.py tests/test_gpu_extend.py -m gpu -q -x > gpurun_out/r2l_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 1 gpurun_out/r2l_pytest.log
for V in "" kw1; do
  L=libspa.so; [ -n "$V" ] && L=libspa_$V.so
  SPA_LIB=$L timeout 300 python scripts/bench_extend.py --max-rows 128 --no-parity --cpu-seconds 0 > gpurun_out/r2l_ext_$V.json 2> gpurun_out/r2l_ext_$V.err; echo "ext $V rc=$?"
  python -c "import json,sys; d=json.load(open('gpurun_out/r2l_ext_$V.json')); print('$V', round(d['layer_us'],1), 'us', round(d['hbm_gbs_algorithmic']), 'GB/s', round(d['roofline']['frac'],3), round(d['tflops']), 'TF/s')"
  SPA_LIB=$L timeout 300 python scripts/ext_trace.py > gpurun_out/r2l_trace_$V.txt 2>&1; sed -n 2,3p gpurun_out/r2l_trace_$V.txt; grep "issue -> MMA sees\|PV-issued -> M kfull\|WG0 W pfull-arr -> W sfull\|K-issued" gpurun_out/r2l_trace_$V.txt
done
