#!/bin/bash
# Time the shipped kernel at different persistent-grid sizes.
cd "$GRAFT_REPO_ROOT" || exit 1
for c in 2 3 4 5 6 8 12 16 32; do
  echo "ctas_per_sm=$c $(T3DES_BS_CTAS_PER_SM=$c python scripts/profile_kernels.py bitslice | tail -1)"
done
