timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3 > gpurun_out/pytest_s28.log
export OUT=gpurun_out/timeline_s28.jsonl
CASES="qwen||;sweep:256:0.5||;long||;qwen|--split 70|" bash scripts/gpu_timeline.sh 2> gpurun_out/timeline_s28.err
