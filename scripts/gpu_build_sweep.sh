#!/bin/bash
# Compile-time shape sweep of the shipped TMA kernel: rebuild the engine with
# each EXTRA_NVFLAGS set and time 1 GiB encrypts (3 launches, last printed).
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
while IFS= read -r FL; do
  make -B -s -C paper_1305_4376_b200/csrc EXTRA_NVFLAGS="$FL" > gpurun_out/sweep_make.log 2>&1 || { echo "build failed: $FL"; continue; }
  R=$(grep -A1 "t3_bs_tma_kernelILi5ELi48" paper_1305_4376_b200/csrc/build/ptxas.log | grep -o "Used [0-9]* registers\|[0-9]* bytes spill stores" | tr '\n' ' ')
  for rep in 1 2; do
    echo "[$FL] $R $(timeout 60 python scripts/profile_kernels.py bitslice 2>&1 | tail -1)"
  done
done <<'LIST'
-DT3_SWEEP_BASE
-DT3_BS_THREADS=256
-DT3_BS_THREADS=64 -DT3_BS_MIN_CTAS=8
-DT3_BS_MIN_CTAS=3
-DT3_BODY_ROUNDS=4
LIST
