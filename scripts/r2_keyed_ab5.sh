#!/bin/bash
# keyed kernel A/B, round 5: last pass spread over all SMs with idle warps taking only the barriers
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/keyed_ab5.jsonl; : > $O
for rep in 1 2; do
  for o in "" "-DT3_KEYED_SPREAD=1"; do
    T3DES_KEYED_NVRTC_OPTS="$o" timeout 300 python scripts/keyed_ab.py paper_1305_4376_b200/libt3des_b200.so rep$rep >> $O 2>&1
  done
done
timeout 900 python -m pytest tests/test_keyed.py -x -q -m gpu 2>&1 | tail -2
T3DES_KEYED_NVRTC_OPTS="-DT3_KEYED_SPREAD=1" timeout 900 python -m pytest tests/test_keyed.py -x -q -m gpu 2>&1 | tail -2
cat $O
