#!/bin/bash
# keyed variant at HEAD: GPU tests, probe, ncu --set full of one keyed launch
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest tests/test_keyed.py -x -q -m gpu 2>&1 | tail -2
timeout 600 python scripts/keyed_probe.py > gpurun_out/keyed_probe.txt 2>&1; cat gpurun_out/keyed_probe.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:t3_keyed_kernel -s 2 -c 1 \
  -o gpurun_out/ncu_keyed python scripts/keyed_probe.py > gpurun_out/ncu_keyed.log 2>&1
echo "ncu rc=$?"
