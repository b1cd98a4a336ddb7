#!/bin/bash
# round 2: merge-tail variants on k = 3, the engine-load sweep (BJ config 3) on the current kernels, bench config 1
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
for W in 0 1; do
  SPA_MERGE_WHOLE=$W timeout 300 python scripts/trace_timeline.py sweep:256:0.75 --rows 0 --out gpurun_out/r2e_timeline_whole$W.jsonl > /dev/null 2>> gpurun_out/r2e_timeline.err; echo "timeline whole=$W rc=$?"
done
timeout 300 python scripts/trace_timeline.py sweep:256:1.0 --rows 0 --out gpurun_out/r2e_timeline_f1.jsonl > /dev/null 2>> gpurun_out/r2e_timeline.err
timeout 1200 python scripts/sweep_load.py --out gpurun_out/r2e_sweep.jsonl > gpurun_out/r2e_sweep.log 2>&1; echo "sweep rc=$?"; cat gpurun_out/r2e_sweep.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2e_bench.json 2> gpurun_out/r2e_bench.err; echo "bench rc=$?"; cut -c1-1500 gpurun_out/r2e_bench.json
