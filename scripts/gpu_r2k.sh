#!/bin/bash
# round 2: ncu full capture of the tcgen05 extend kernel (split rings, Q in TMEM) on the mixed step
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:ext_kernel -c 1 \
   -o /tmp/r2k_ext -f python scripts/bench_extend.py --max-rows 128 --profile > gpurun_out/r2k_ncu.log 2>&1; echo "ncu rc=$?"
python scripts/ncu_summary.py full /tmp/r2k_ext.ncu-rep --top 40 > gpurun_out/r2k_ext_full.txt 2>&1
ncu -i /tmp/r2k_ext.ncu-rep --page raw --csv > gpurun_out/r2k_ext_raw.csv 2>/dev/null
ncu -i /tmp/r2k_ext.ncu-rep --page source --csv --print-source sass > gpurun_out/r2k_ext_source.csv 2>/dev/null; gzip -f gpurun_out/r2k_ext_source.csv
head -n 60 gpurun_out/r2k_ext_full.txt
