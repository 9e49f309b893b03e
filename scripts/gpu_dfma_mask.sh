#!/bin/bash
# Which E-duplicate corrections should go to the FMA pipe: regenerate with
# T3_GEN_DFMA_MASK, rebuild, time 1 GiB encrypts.
cd "$GRAFT_REPO_ROOT" || exit 1
for M in 0xFFFF 0x5555 0x00FF 0xFF00 0x0F0F 0x3333; do
  T3_GEN_DFMA_MASK=$M python paper_1305_4376_b200/csrc/gen_bitslice.py 2>/dev/null
  make -s -C paper_1305_4376_b200/csrc > /dev/null 2>&1 || { echo "build failed $M"; continue; }
  for rep in 1 2; do echo "mask=$M $(timeout 60 python scripts/profile_kernels.py bitslice 2>&1 | tail -1)"; done
done
