set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -5 > gpurun_out/pytest_s20.log
export OUT=gpurun_out/timeline_s20.jsonl
CASES="qwen||;long||;sweep:1:0||;sweep:8:0||;sweep:32:0||;sweep:64:0.5||;sweep:256:0.5||;sweep:256:0.5||SPA_SPLIT_DIV=1;long||SPA_SPLIT_DIV=1;long||SPA_SPLIT_DIV=3" bash scripts/gpu_timeline.sh 2> gpurun_out/timeline_s20.err
