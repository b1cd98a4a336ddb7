SPA_LIB=libspa_dbg.so timeout -s KILL 100 python scripts/bench_extend.py --max-rows 128 --no-parity --reps 2 > gpurun_out/ext_s54_dbg.txt 2>&1
timeout -s KILL 300 python -m pytest tests/test_gpu_extend_tc.py tests/test_gpu_extend.py -x -q 2>&1 | tail -3 > gpurun_out/ext_s54.log
timeout -s KILL 150 python scripts/bench_extend.py --max-rows 128 > gpurun_out/ext_s54.json 2>> gpurun_out/ext_s54.log
timeout -s KILL 100 python scripts/ext_trace.py > gpurun_out/ext_trace_s54.txt 2>&1
