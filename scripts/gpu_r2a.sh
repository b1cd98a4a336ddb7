#!/bin/bash
# round 2, first GPU pass: the GPU suite on the current library, the R > 16 sweep point and
# full ncu captures of the 16- and 32-row decode plans at B = 256, f = 0.75 (k = 3)
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2a_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2a_pytest.log
timeout 600 python scripts/sweep_load.py --batches 64,256 --fracs 0.75 --out gpurun_out/r2a_sweep.jsonl > gpurun_out/r2a_sweep.log 2>&1; echo "sweep rc=$?"; cat gpurun_out/r2a_sweep.log | tail -3
for R in 16 32; do
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:decode_kernel -c 2 \
   -o gpurun_out/r2a_rows$R -f python scripts/profile_small.py 256 0.75 $R > gpurun_out/r2a_ncu_rows$R.log 2>&1
echo "ncu rows=$R rc=$?"
done
