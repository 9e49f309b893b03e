#!/bin/bash
# Stream path (t3des_cu_stream_fd via the CLI): 1 GiB file encrypt/decrypt
# with PKCS#7, timed by the shell, next to plain page-cache copy rates.
cd "$GRAFT_REPO_ROOT" || exit 1
python - <<'PY'
import numpy as np
np.random.default_rng(7).integers(0, 256, (1 << 30) + 11, dtype=np.uint8).tofile("/tmp/t3_in.bin")
PY
K=133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57
C=paper_1305_4376_b200/t3des_b200
cat /tmp/t3_in.bin > /dev/null
t() { local s=$(date +%s.%N); "$@"; local rc=$?; local e=$(date +%s.%N); echo "rc=$rc $(python -c "print(f'{(1<<30)/($e-$s)/1e9:.2f} GB/s ({$e-$s:.3f} s)')") : $*"; }
t cp /tmp/t3_in.bin /tmp/t3_cp.bin
t $C encrypt --key $K /tmp/t3_in.bin /tmp/t3_ct.bin --pkcs7
t $C decrypt --key $K /tmp/t3_ct.bin /tmp/t3_pt.bin --pkcs7
cmp /tmp/t3_in.bin /tmp/t3_pt.bin && echo "round trip identical"
t $C encrypt --key $K /tmp/t3_in.bin /tmp/t3_ct2.bin --pkcs7
t sh -c "$C encrypt --key $K --pkcs7 - - < /tmp/t3_in.bin > /tmp/t3_ct3.bin"
cmp /tmp/t3_ct.bin /tmp/t3_ct3.bin && echo "pipe == file"
ls -la /tmp/t3_*.bin
rm -f /tmp/t3_*.bin
