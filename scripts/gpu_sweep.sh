#!/bin/bash
# GPU tests + bench sweep: each CASES entry is "name|bench args|env"
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-sweep}
if [ -z "$NOTEST" ]; then
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
tail -3 gpurun_out/pytest_gpu_$TAG.log
fi
IFS=';' read -ra CS <<< "${CASES:-base||}"
for c in "${CS[@]}"; do
  IFS='|' read -r name args envs <<< "$c"
  env $envs timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-parity --cpu-seconds 1 $args \
     > gpurun_out/bench_${TAG}_${name}.log 2>&1
  python - "$name" gpurun_out/bench_${TAG}_${name}.log <<'EOF'
import json, sys
ok = False
for line in open(sys.argv[2]):
    if line.startswith("{"):
        r = json.loads(line); ok = True
        print(sys.argv[1], "tok/s %.0f" % r["value"], "ms/step %.3f" % r["ms_per_step"], "layer_ms %.4f" % r["layer_ms"],
              "GB/s %.0f" % r["roofline"]["achieved"], "frac %.3f" % r["roofline"]["frac"],
              "recs", r["plan"]["n_records"], "items", r["plan"]["n_items"], "sm_mhz", r["clocks"]["sm_mhz"])
if not ok:
    print(sys.argv[1], "FAILED:", open(sys.argv[2]).read()[-800:])
EOF
done
