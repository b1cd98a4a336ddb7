#!/bin/bash
# round 2: split K/V rings in the tcgen05 extend kernel: parity (extend + workspace tests), bench per NK variant, trace
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_extend_tc.py tests/test_gpu_extend.py tests/test_gpu_workspace.py tests/test_gpu_umma.py -m gpu -q -x > gpurun_out/r2g_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2g_pytest.log
for V in "" nk3 nk6; do
  L=libspa.so; [ -n "$V" ] && L=libspa_$V.so
  SPA_LIB=$L timeout 300 python scripts/bench_extend.py --max-rows 128 --no-parity --cpu-seconds 0 > gpurun_out/r2g_ext_$V.json 2> gpurun_out/r2g_ext_$V.err; echo "ext $V rc=$?"
  python -c "import json,sys; d=json.load(open('gpurun_out/r2g_ext_$V.json')); print('$V', round(d['layer_us'],1), 'us', round(d['hbm_gbs_algorithmic']), 'GB/s', round(d['roofline']['frac'],3), round(d['tflops']), 'TF/s')"
done
timeout 300 python scripts/bench_extend.py --max-rows 128 > gpurun_out/r2g_ext_parity.json 2> gpurun_out/r2g_ext_parity.err; echo "ext parity rc=$?"; python -c "import json; d=json.load(open('gpurun_out/r2g_ext_parity.json')); print(d.get('parity'))"
timeout 300 python scripts/ext_trace.py > gpurun_out/r2g_ext_trace.txt 2>&1; echo "trace rc=$?"; tail -6 gpurun_out/r2g_ext_trace.txt
