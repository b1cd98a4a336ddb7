timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3 > gpurun_out/pytest_s26.log
export OUT=gpurun_out/timeline_s26.jsonl
CASES="qwen||;sweep:256:0.5||;sweep:1:0||;sweep:8:0||;sweep:64:0.5||;long||;qwen|--merge 1|;qwen|--merge 2|" bash scripts/gpu_timeline.sh 2> gpurun_out/timeline_s26.err
