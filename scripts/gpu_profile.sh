#!/bin/bash
# ncu evidence for the decode step: bench line, launch list of 2 timed steps, one full capture of decode_kernel
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-r1}
if [ -z "$NOTEST" ]; then
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
tail -2 gpurun_out/pytest_gpu_$TAG.log
fi
timeout 900 python bench.py --steps 20 --warmup 5 $BENCH_ARGS > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 2 --profile $BENCH_ARGS > gpurun_out/ncu_launch_bench_$TAG.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:decode_kernel -c 2 \
   -o gpurun_out/prof_decode_$TAG -f python bench.py --steps 1 --warmup 2 --profile $BENCH_ARGS > gpurun_out/ncu_full_$TAG.log 2>&1
echo "full rc=$?"
tail -1 gpurun_out/bench_$TAG.log | cut -c1-3000
