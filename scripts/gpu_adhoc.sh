./scripts/micro/hmma_bench > gpurun_out/hmma_bench.txt 2>&1
export OUT=gpurun_out/timeline_s34.jsonl
CASES="qwen||;qwen||SPA_LIB=libspa_qk2.so;qwen||SPA_LIB=libspa_qk4.so;sweep:1:0|--split 400|;sweep:1:0|--split 400|SPA_LIB=libspa_qk2.so;sweep:1:0|--split 400|SPA_LIB=libspa_qk4.so;sweep:8:0||;sweep:8:0||SPA_LIB=libspa_qk2.so;sweep:8:0||SPA_LIB=libspa_qk4.so" bash scripts/gpu_timeline.sh 2> gpurun_out/timeline_s34.err
