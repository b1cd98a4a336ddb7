#!/bin/bash
# A/B of library variants on one box: GPU suite on the main library (optional), then bench
# lines for each variant.  Usage: scripts/gpu_ab.sh "<variants>" [tests]
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out/ab; mkdir -p $O
if [ "$2" = "tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -n 3 $O/pytest_gpu.log
fi
summ() { python - "$1" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
except Exception as e:
    print(sys.argv[1], "unparsed", e); sys.exit()
r=d.get("roofline",{}); x=d.get("extra",{}) or {}
pw=d.get("per_window") or x.get("per_window")
print(f'{sys.argv[1]:44s} value={d["value"]:.1f} ms/step={d["ms_per_step"]:.3f} frac={r.get("frac")} achieved={r.get("achieved")} clocks={d.get("clocks",{}).get("sm_mhz")} per_window={pw}')
PY
}
for v in $1; do
  if [ "$v" = "main" ]; then export SPA_LIB=libspa.so; else export SPA_LIB=libspa_$v.so; fi
  for rep in 1 2; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e > $O/bench_${v}_$rep.json 2> $O/bench_${v}.err; summ $O/bench_${v}_$rep.json
  timeout 600 python bench.py --kv fp8 --steps 10 --warmup 3 --no-e2e > $O/fp8_${v}_$rep.json 2> $O/fp8_${v}.err; summ $O/fp8_${v}_$rep.json
  timeout 600 python bench.py --config gemma --steps 5 --warmup 3 --no-e2e > $O/gemma_${v}_$rep.json 2> $O/gemma_${v}.err; summ $O/gemma_${v}_$rep.json
  done
done
