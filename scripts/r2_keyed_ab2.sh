#!/bin/bash
# keyed kernel A/B, round 2: barrier spacing with idle warps computing (free-top circuits)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/keyed_ab2.jsonl; : > $O
for rep in 1 2; do
  for se in 4 8 12 16 24 48; do
    T3DES_KEYED_NVRTC_OPTS="-DT3_KEYED_IDLE_COMPUTE=1 -DT3_KEYED_SYNC_EVERY=$se" timeout 300 python scripts/keyed_ab.py paper_1305_4376_b200/libt3des_b200.so ftop_rep$rep >> $O 2>&1
  done
done
cat $O
