cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out/tl; mkdir -p $O
for v in main nx1; do
  if [ "$v" = "main" ]; then export SPA_LIB=libspa.so; else export SPA_LIB=libspa_$v.so; fi
  timeout 300 python scripts/trace_timeline.py qwen --kv fp8 > $O/fp8_$v.txt 2>&1
  timeout 300 python scripts/trace_timeline.py qwen > $O/bf16_$v.txt 2>&1
done
