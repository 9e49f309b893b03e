#!/bin/bash
# The paper's Table I/II/IV sweeps on the B200 through the CLI (reference CSV
# format), 512 MiB payload (the paper's file size), device-resident and end to
# end, plus the reference's own CPU workers sweep on the same host.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/tables
CLI=paper_1305_4376_b200/t3des_b200
for mode in device host; do
  $CLI bench --mode $mode --sweep workgroup --values 32,64,128,256,512,1024 --variant sptable --payload-mb 512 --reps 3 --format csv --out gpurun_out/tables/table1_workgroup_sptable_$mode.csv
  $CLI bench --mode $mode --sweep workgroup --values 32,64,128 --variant bitslice --payload-mb 512 --reps 3 --format csv --out gpurun_out/tables/table1_workgroup_bitslice_$mode.csv
  $CLI bench --mode $mode --sweep chunk --values 1024,16384,131072,1048576,16777216,67108864 --payload-mb 512 --reps 3 --format csv --out gpurun_out/tables/table2_chunk_$mode.csv
done
$CLI bench --mode host --sweep workers --values 1,2,4 --payload-mb 512 --reps 3 --format csv --out gpurun_out/tables/table4_workers_host.csv
python - <<'PY' > gpurun_out/tables/table4_reference_cpu_workers.csv
import sys, time
sys.path.insert(0, ".")
import numpy as np
from tests.oracle_util import Oracle
o = Oracle.load()
s = o.schedule_hex("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57")
x = o.payload(512 << 20, 0x3DE5C0DE)
y = np.empty_like(x)
print("backend,workers,chunk_blocks,work_group,payload_bytes,compute_seconds,throughput_mb_s")
for w in (1, 2, 4, 8, 16):
    n = x.nbytes if w >= 4 else (64 << 20)
    o.ref.ref_ecb(x.ctypes.data, y.ctypes.data, 8 << 20, s, 0, 1, w, 0, 0)
    t0 = time.perf_counter(); o.ref.ref_ecb(x.ctypes.data, y.ctypes.data, n, s, 0, 1, w, 0, 0); dt = time.perf_counter() - t0
    print(f"threaded,{w},131072,256,{n},{dt:.6f},{n / dt / (1 << 20):.3f}", flush=True)
PY
ls -la gpurun_out/tables
