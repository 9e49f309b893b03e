#!/bin/bash
# ncu --set full of one bitsliced variant (VARIANT=bitslice|bitslice_alu|...), TAG names the report.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
P="python scripts/profile_kernels.py $VARIANT"
$P > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:t3_bs_tma_kernel -s 1 -c 1 -o gpurun_out/prof_$TAG $P > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?"; cat gpurun_out/plain_$TAG.log
