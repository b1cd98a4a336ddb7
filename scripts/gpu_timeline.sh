# Timeline traces (scripts/trace_timeline.py) for a list of cases:
#   CASES="workload|args|env;..." OUT=gpurun_out/timeline.jsonl bash scripts/gpu_timeline.sh
set -u
OUT=${OUT:-gpurun_out/timeline.jsonl}
IFS=';' read -ra CS <<< "$CASES"
for c in "${CS[@]}"; do
  IFS='|' read -r w args envs <<< "$c"
  echo "== $w $args $envs" >&2
  env $envs timeout 300 python scripts/trace_timeline.py $w $args --out $OUT > /dev/null || echo "FAILED $c" >&2
done
