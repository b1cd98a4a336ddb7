#!/bin/bash
# compute-sanitizer passes on small GPU parity cases
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-san}
SAN=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 900 $SAN --tool $tool --error-exitcode 9 --print-limit 20 \
     python -m pytest tests/test_gpu_parity.py -q -x -k "tiny_config or merge_paths_many_splits or window_one or single_key" \
     > gpurun_out/sanitize_${tool}_$TAG.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_${tool}_$TAG.log
done
