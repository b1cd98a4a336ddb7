export OUT=gpurun_out/timeline_s22.jsonl
CASES="qwen||;sweep:256:0.5||;sweep:8:0||;qwen|--merge 2|;sweep:256:0.5|--merge 2|" bash scripts/gpu_timeline.sh 2> gpurun_out/timeline_s22.err
