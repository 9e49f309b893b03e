#!/bin/bash
# GPU tests + ncu launch list of bench.py + ncu --set full of both kernels.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$B > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_bench.log 2>&1
echo "launch list rc=$?"
P="python scripts/profile_kernels.py"
$P > gpurun_out/plain_profile.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:t3_bs_kernel -s 1 -c 1 -o gpurun_out/prof_bs_r1 $P bitslice > gpurun_out/ncu_full_bs.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:t3_sp_kernel -s 1 -c 1 -o gpurun_out/prof_sp_r1 $P sptable > gpurun_out/ncu_full_sp.log 2>&1
echo "ncu full rc=$?"
ls -la gpurun_out
