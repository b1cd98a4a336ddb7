export OUT=gpurun_out/timeline_s24.jsonl
CASES="qwen||;sweep:256:0.5||;sweep:1:0||;sweep:1:0|--split 32|" bash scripts/gpu_timeline.sh 2> gpurun_out/timeline_s24.err
