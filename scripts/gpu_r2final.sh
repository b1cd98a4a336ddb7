#!/bin/bash
# round 2 final evidence on the final kernels: GPU suite, smoke, bench (both arms), other
# workloads (bf16 + fp8), extend, ncu launch lists and full captures (bf16 decode, fp8 decode,
# tcgen05 extend), engine-load sweep.  Outputs under gpurun_out/r02f (copied to profiles/r02_*).
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out/r02f; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -n 1 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -n 1 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?"
timeout 900 python bench.py --config gemma --steps 10 --warmup 3 > $O/bench_gemma.json 2> $O/bench_gemma.err; echo "gemma rc=$?"
timeout 900 python bench.py --config long --steps 5 --warmup 3 > $O/bench_long.json 2> $O/bench_long.err; echo "long rc=$?"
timeout 900 python bench.py --kv fp8 --steps 20 --warmup 5 > $O/bench_fp8_qwen.json 2> $O/bench_fp8.err; echo "fp8 rc=$?"
timeout 900 python bench.py --kv fp8 --config gemma --steps 10 --warmup 3 > $O/bench_fp8_gemma.json 2>> $O/bench_fp8.err; echo "fp8 gemma rc=$?"
timeout 900 python bench.py --kv fp8 --config long --steps 5 --warmup 3 > $O/bench_fp8_long.json 2>> $O/bench_fp8.err; echo "fp8 long rc=$?"
timeout 600 python scripts/bench_extend.py --max-rows 128 > $O/extend.json 2> $O/extend.err; echo "extend rc=$?"
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file $O/launches.csv python bench.py --steps 2 --warmup 2 --profile > $O/ncu_launch.log 2>&1; echo "launch list rc=$?"
python scripts/ncu_summary.py launches $O/launches.csv > $O/launches.txt 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:decode_kernel -c 2 \
   -o /tmp/r02_decode_full -f python bench.py --steps 1 --warmup 2 --profile > $O/ncu_full.log 2>&1; echo "full rc=$?"
python scripts/ncu_summary.py full /tmp/r02_decode_full.ncu-rep --top 40 > $O/decode_full.txt 2>&1
ncu -i /tmp/r02_decode_full.ncu-rep --page source --csv --print-source sass > $O/decode_source.csv 2>/dev/null
python scripts/ncu_stalls.py $O/decode_source.csv x 50 > $O/decode_stalls.txt 2>&1; gzip -f $O/decode_source.csv
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:decode_kernel -c 1 \
   -o /tmp/r02_fp8_full -f python bench.py --kv fp8 --steps 1 --warmup 2 --profile --no-e2e > $O/ncu_fp8.log 2>&1; echo "fp8 full rc=$?"
python scripts/ncu_summary.py full /tmp/r02_fp8_full.ncu-rep --top 40 > $O/fp8_full.txt 2>&1
ncu -i /tmp/r02_fp8_full.ncu-rep --page source --csv --print-source sass > $O/fp8_source.csv 2>/dev/null
python scripts/ncu_stalls.py $O/fp8_source.csv x 50 > $O/fp8_stalls.txt 2>&1; rm -f $O/fp8_source.csv
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file $O/fp8_launches.csv python bench.py --kv fp8 --steps 2 --warmup 2 --profile --no-e2e > /dev/null 2>&1
python scripts/ncu_summary.py launches $O/fp8_launches.csv > $O/fp8_launches.txt 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:ext_kernel -c 1 \
   -o /tmp/r02_ext_full -f python scripts/bench_extend.py --max-rows 128 --profile > $O/ncu_ext.log 2>&1; echo "ext full rc=$?"
python scripts/ncu_summary.py full /tmp/r02_ext_full.ncu-rep --top 40 > $O/ext_full.txt 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file $O/ext_launches.csv python scripts/bench_extend.py --max-rows 128 --profile > /dev/null 2>&1
python scripts/ncu_summary.py launches $O/ext_launches.csv > $O/ext_launches.txt 2>&1
timeout 1200 python scripts/sweep_load.py --out $O/sweep_load.jsonl > $O/sweep_load.txt 2>&1; echo "sweep rc=$?"
timeout 300 python scripts/trace_timeline.py qwen > $O/timeline_bf16.txt 2>&1
timeout 300 python scripts/trace_timeline.py qwen --kv fp8 > $O/timeline_fp8.txt 2>&1
for f in bench bench_gemma bench_long bench_fp8_qwen bench_fp8_gemma bench_fp8_long bench_reference; do cut -c1-200 $O/$f.json; echo; done
