#!/bin/bash
# round 2 (re-entry): GPU suite on HEAD, bench config 1, engine-load sweep on the current kernels
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -rA -s > gpurun_out/r2f_pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|error" gpurun_out/r2f_pytest.log | tail -3
grep "fp8 vs bf16" gpurun_out/r2f_pytest.log | head
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err; echo "bench rc=$?"; cut -c1-1500 gpurun_out/r2f_bench.json
timeout 1200 python scripts/sweep_load.py --out gpurun_out/r2f_sweep.jsonl > gpurun_out/r2f_sweep.log 2>&1; echo "sweep rc=$?"; tail -40 gpurun_out/r2f_sweep.log
