#!/bin/bash
# round 2: GPU suite after the prefix-tree planner + full-precision/nested parity; timelines of k = 3 batches
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -rA -s -k "not fullsize" > gpurun_out/r2c_pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|error" gpurun_out/r2c_pytest.log | tail -3
grep "fp8 vs bf16" gpurun_out/r2c_pytest.log
for W in "sweep:256:0.75 --rows 16" "sweep:256:0.75 --rows 32" "qwen --rows 16"; do
  timeout 300 python scripts/trace_timeline.py $W --out gpurun_out/r2c_timeline.jsonl > /dev/null 2>> gpurun_out/r2c_timeline.err; echo "timeline $W rc=$?"
done
