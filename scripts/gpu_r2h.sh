#!/bin/bash
# round 2: extend kernel timeline (item transitions) + ncu launch list of the mixed step
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 300 python scripts/ext_trace.py > gpurun_out/r2h_ext_trace.txt 2>&1; echo "trace rc=$?"; head -n 20 gpurun_out/r2h_ext_trace.txt
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/r2h_ext_launches.csv python scripts/bench_extend.py --max-rows 128 --profile > /dev/null 2>&1; echo "ncu rc=$?"
grep -E "gpu__time_duration|dram__bytes_read" gpurun_out/r2h_ext_launches.csv | cut -c1-300 | head -n 20
