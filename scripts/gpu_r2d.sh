#!/bin/bash
# round 2: the KW=1 (no key split) 32-row variant: parity, sweep points, timeline
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity_full.py -m gpu -q -x -k "row_tile_warps or qwen_shaped" > gpurun_out/r2d_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2d_pytest.log
timeout 900 python scripts/sweep_load.py --batches 32,64,128,256 --fracs 0.75,1 --plans shared,shared32,shared32kw1 --out gpurun_out/r2d_sweep.jsonl > gpurun_out/r2d_sweep.log 2>&1; echo "sweep rc=$?"; cat gpurun_out/r2d_sweep.log
SPA_KW=1 timeout 300 python scripts/trace_timeline.py sweep:256:0.75 --rows 32 --out gpurun_out/r2d_timeline.jsonl > /dev/null 2>> gpurun_out/r2d_timeline.err; echo "timeline rc=$?"
