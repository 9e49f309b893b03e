#!/bin/bash
# Time the shipped kernel at different grid sizes (CTAs per SM; the grid is
# also capped at one tile per warp).
cd "$GRAFT_REPO_ROOT" || exit 1
for c in ${CTAS:-4 16 32 48 64 96 128 160 221 256}; do
  echo "ctas_per_sm=$c $(T3DES_BS_CTAS_PER_SM=$c python scripts/profile_kernels.py bitslice bitslice_ldg | grep 'launch 2' | tr '\n' ' ')"
done
