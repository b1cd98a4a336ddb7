#!/bin/bash
# round 2: ext kernel variants (K ring depth NK, K producer warps KW) on the mixed step
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
for V in "" kw2 nk6 nk6kw2 nk5kw2; do
  L=libspa.so; [ -n "$V" ] && L=libspa_$V.so
  SPA_LIB=$L timeout 300 python scripts/bench_extend.py --max-rows 128 --no-parity --cpu-seconds 0 > gpurun_out/r2j_ext_$V.json 2> gpurun_out/r2j_ext_$V.err; echo "ext $V rc=$?"
  python -c "import json,sys; d=json.load(open('gpurun_out/r2j_ext_$V.json')); print('$V', round(d['layer_us'],1), 'us', round(d['hbm_gbs_algorithmic']), 'GB/s', round(d['roofline']['frac'],3), round(d['tflops']), 'TF/s')"
done
