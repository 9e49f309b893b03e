#!/bin/bash
# Pageable staging path: GPU tests of the host path, then e2e GB/s for a few
# copy-thread counts and stage sizes, with and without streaming stores.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "host_path or pipeline_shapes or pageable or python_api or multi" > gpurun_out/pageable_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pageable_pytest.log
for NT in 1 0; do for T in 8 12 16; do for S in 2 4 8; do
  echo "nt=$NT threads=$T stage=${S}MiB: $(T3DES_HOST_NT_COPY=$NT T3DES_HOST_COPY_THREADS=$T T3DES_HOST_STAGE_MIB=$S timeout 120 python scripts/e2e_pageable.py 2>&1 | grep '1024 MiB pageable')"
done; done; done
timeout 120 python scripts/e2e_pageable.py
lscpu | head -20
