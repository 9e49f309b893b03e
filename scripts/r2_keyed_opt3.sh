#!/bin/bash
# keyed variant after pinning the barriers: GPU tests, the probe (bench key), option-3 (16-round) spacing
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest tests/test_keyed.py -x -q -m gpu 2>&1 | tail -3
timeout 600 python scripts/keyed_probe.py > gpurun_out/keyed_probe.txt 2>&1; cat gpurun_out/keyed_probe.txt
O=gpurun_out/keyed_opt3.jsonl; : > $O
for se in "" "-DT3_KEYED_SYNC_EVERY=4" "-DT3_KEYED_SYNC_EVERY=12"; do
  T3DES_KEYED_NVRTC_OPTS="$se" T3_AB_KEY=0123456789ABCDEF timeout 300 python scripts/keyed_ab.py paper_1305_4376_b200/libt3des_b200.so opt3 >> $O 2>&1
done
cat $O
