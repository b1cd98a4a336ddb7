#!/bin/bash
# fp8 decode investigation: bench line, one full ncu capture with source-level stalls, timeline
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out/fp8prof; mkdir -p $O
timeout 600 python bench.py --kv fp8 --steps 10 --warmup 3 --no-e2e > $O/bench_fp8.json 2> $O/bench_fp8.err; echo "fp8 rc=$?"
timeout 600 python scripts/trace_timeline.py qwen --kv fp8 > $O/timeline_fp8.txt 2>&1; echo "tl rc=$?"
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:decode_kernel -c 1 \
   -o /tmp/fp8full -f python bench.py --kv fp8 --steps 1 --warmup 2 --profile --no-e2e > $O/ncu_full.log 2>&1; echo "full rc=$?"
python scripts/ncu_summary.py full /tmp/fp8full.ncu-rep --top 40 > $O/fp8_full.txt 2>&1
ncu -i /tmp/fp8full.ncu-rep --page source --csv --print-source sass > $O/fp8_source.csv 2>/dev/null
python scripts/ncu_stalls.py $O/fp8_source.csv x 70 > $O/fp8_stalls.txt 2>&1
gzip -f $O/fp8_source.csv
cut -c1-400 $O/bench_fp8.json
