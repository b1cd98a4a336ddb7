timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3 > gpurun_out/pytest_s27.log
export OUT=gpurun_out/timeline_s27.jsonl
CASES="qwen||;sweep:256:0.5||;sweep:8:0||;sweep:64:0.5||" bash scripts/gpu_timeline.sh 2> gpurun_out/timeline_s27.err
