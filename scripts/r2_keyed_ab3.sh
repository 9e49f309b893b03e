#!/bin/bash
# keyed kernel A/B, round 3: barriers pinned between rounds by a data dependency (T3_KEYED_PIN) vs the
# clustered barriers ptxas makes of plain __syncthreads
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/keyed_ab3.jsonl; : > $O
for rep in 1 2; do
  T3DES_KEYED_NVRTC_OPTS="" timeout 300 python scripts/keyed_ab.py paper_1305_4376_b200/libt3des_b200.so clustered12_rep$rep >> $O 2>&1
  for se in 2 3 4 6 8 12 16 24; do
    T3DES_KEYED_NVRTC_OPTS="-DT3_KEYED_PIN=1 -DT3_KEYED_SYNC_EVERY=$se" timeout 300 python scripts/keyed_ab.py paper_1305_4376_b200/libt3des_b200.so pinned_rep$rep >> $O 2>&1
  done
done
cat $O
