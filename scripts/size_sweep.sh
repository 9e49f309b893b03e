#!/bin/bash
# Kernel time vs batch size for the shipped and the all-ALU round variants.
cd "$GRAFT_REPO_ROOT" || exit 1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv
for g in 1 2 4 8 16; do
  echo "GiB=$g $(T3_GIB=$g python scripts/profile_kernels.py bitslice bitslice_alu | grep 'launch 2' | tr '\n' ' ')"
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv
