timeout 300 python -m pytest tests/test_gpu_extend_tc.py -x -q -k "decode_rows_only" 2>&1 | tail -30 > gpurun_out/tc_s38.log
timeout 300 python -m pytest tests/test_gpu_extend_tc.py -x -q 2>&1 | tail -30 >> gpurun_out/tc_s38.log
