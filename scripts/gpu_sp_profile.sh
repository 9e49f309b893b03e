#!/bin/bash
# bench line + ncu --set full of the SP-table kernel (1 GiB launch).
# Usage: TAG=r1k bash scripts/gpu_sp_profile.sh
cd "$GRAFT_REPO_ROOT" || exit 1
TAG=${TAG:-run}
mkdir -p gpurun_out
timeout 600 python bench.py --steps 30 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
cat gpurun_out/bench_$TAG.json
P="python scripts/profile_kernels.py"
$P sptable > gpurun_out/plain_sp.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:t3_sp_kernel -s 1 -c 1 -o gpurun_out/prof_sp_$TAG $P sptable > gpurun_out/ncu_sp.log 2>&1
echo "ncu sp rc=$?"
cat gpurun_out/plain_sp.log
