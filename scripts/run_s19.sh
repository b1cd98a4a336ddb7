set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -5 > gpurun_out/pytest_s19.log
export OUT=gpurun_out/timeline_s19.jsonl
CASES="qwen||;qwen|--merge 1|;sweep:1:0||;sweep:8:0||;sweep:64:0.5||;sweep:1:0||SPA_MAX_SPLITS=8;sweep:8:0||SPA_MAX_SPLITS=8;sweep:16:0.5||;sweep:32:0||;qwen||SPA_SPLIT_DIV=2;long||" bash scripts/gpu_timeline.sh 2> gpurun_out/timeline_s19.err
