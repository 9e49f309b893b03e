#!/bin/bash
# Time the default bitsliced kernel under each compiled T3_OPT_* mask.
cd "$GRAFT_REPO_ROOT" || exit 1
for o in ${OPTS:-0 1 2 3 5 7}; do
  echo "opt=$o $(T3DES_BS_OPT=$o python scripts/profile_kernels.py bitslice bitslice | grep 'launch 2' | tr '\n' ' ')"
done
