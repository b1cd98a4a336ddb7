timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3 > gpurun_out/pytest_s30.log
export OUT=gpurun_out/timeline_s30.jsonl
CASES="qwen||;sweep:256:0.5||;sweep:8:0||;sweep:1:0||;qwen||SPA_MERGE_WHOLE=1" bash scripts/gpu_timeline.sh 2> gpurun_out/timeline_s30.err
