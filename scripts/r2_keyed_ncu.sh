#!/bin/bash
# ncu --set full of the keyed kernel (one 1 GiB launch) next to the shipped TMA kernel
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 600 python scripts/keyed_probe.py > gpurun_out/keyed_probe_pre.txt 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:t3_keyed_kernel -s 2 -c 1 \
  -o gpurun_out/ncu_keyed python scripts/keyed_probe.py > gpurun_out/ncu_keyed.log 2>&1
echo "ncu rc=$?"
