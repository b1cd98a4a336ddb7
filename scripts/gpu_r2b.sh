#!/bin/bash
# ncu captures of the 16- and 32-row decode plans at B = 256, f = 0.75 (k = 3), summarised on the box
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
for R in 16 32; do
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:decode_kernel -c 1 \
   -o /tmp/r2b_rows$R -f python scripts/profile_small.py 256 0.75 $R > gpurun_out/r2b_ncu_rows$R.log 2>&1
echo "ncu rows=$R rc=$?"
python scripts/ncu_summary.py full /tmp/r2b_rows$R.ncu-rep --top 60 > gpurun_out/r2b_rows$R.txt 2>&1
ncu -i /tmp/r2b_rows$R.ncu-rep --page source --csv --print-source sass > gpurun_out/r2b_rows${R}_source.csv 2>/dev/null
gzip -f gpurun_out/r2b_rows${R}_source.csv
done
ls -la gpurun_out
