#!/bin/bash
# GPU tests + bench sweep over split granularity (SPA_SPLIT_DIV), merge mode and PDL
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-sweep}
if [ -z "$NOTEST" ]; then
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
tail -3 gpurun_out/pytest_gpu_$TAG.log
fi
for mode in ${MODES:-separate fused nopdl}; do
for div in ${DIVS:-1 2}; do
  extra=""; envs=""
  [ "$mode" = fused ] && extra="--fused-merge"
  [ "$mode" = nopdl ] && envs="SPA_NO_PDL=1"
  env SPA_SPLIT_DIV=$div $envs timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-parity --cpu-seconds 1 $extra \
     > gpurun_out/bench_${TAG}_${mode}_div$div.log 2>&1
  python - "$mode div$div" gpurun_out/bench_${TAG}_${mode}_div$div.log <<'EOF'
import json, sys
for line in open(sys.argv[2]):
    if line.startswith("{"):
        r = json.loads(line)
        print(sys.argv[1], "tok/s %.0f" % r["value"], "ms/step %.3f" % r["ms_per_step"], "layer_ms %.4f" % r["layer_ms"],
              "GB/s %.0f" % r["roofline"]["achieved"], "frac %.3f" % r["roofline"]["frac"],
              "recs", r["plan"]["n_records"], "items", r["plan"]["n_items"], "sm_mhz", r["clocks"]["sm_mhz"])
EOF
done
done
