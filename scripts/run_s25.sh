export OUT=gpurun_out/timeline_s25.jsonl
CASES="qwen||;sweep:256:0.5||;sweep:1:0||" bash scripts/gpu_timeline.sh 2> gpurun_out/timeline_s25.err
