#!/bin/bash
# keyed kernel A/B, round 4: pinned barrier spacing around 16 rounds
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/keyed_ab4.jsonl; : > $O
for rep in 1 2; do
  for se in 10 13 14 15 16 17 18 20; do
    T3DES_KEYED_NVRTC_OPTS="-DT3_KEYED_PIN=1 -DT3_KEYED_SYNC_EVERY=$se" timeout 300 python scripts/keyed_ab.py paper_1305_4376_b200/libt3des_b200.so pinned_rep$rep >> $O 2>&1
  done
done
cat $O
