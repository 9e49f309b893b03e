#!/bin/bash
# keyed kernel A/B: circuits (shipped vs free-Feistel-top) x idle-warp policy x barrier spacing
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/keyed_ab.jsonl; : > $O
for lib in scripts/_ab/lib_keyed_base.so paper_1305_4376_b200/libt3des_b200.so; do
  for opts in "" "-DT3_KEYED_IDLE_COMPUTE=1" "-DT3_KEYED_SYNC_EVERY=2" "-DT3_KEYED_SYNC_EVERY=8" "-DT3_KEYED_IDLE_COMPUTE=1 -DT3_KEYED_SYNC_EVERY=8"; do
    T3DES_KEYED_NVRTC_OPTS="$opts" timeout 300 python scripts/keyed_ab.py $lib $(basename $lib) >> $O 2>&1
  done
done
cat $O
