#!/usr/bin/env python3
"""Pageable host batches of 1-64 MiB: the round-1 staging (lock-step loop,
streaming stores both ways; scripts/_ab/libt3des_b200_lockstep.so) against
the current one (decoupled fill/drain, cached slot stores), one subprocess
per measurement, interleaved rounds, median us per in-place call."""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, time, json, statistics
sys.path.insert(0, sys.argv[1])
from paper_1305_4376_b200 import _native as N
if sys.argv[2] != "-":
    N.LIB_PATH = sys.argv[2]
import numpy as np
import paper_1305_4376_b200 as t3
e = t3.Engine(0)
e.set_schedule(t3.triple_schedule(t3.parse_hex_key("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57")))
out = {}
for mib in (1, 4, 16, 64):
    n = mib << 20
    a = np.random.default_rng(0).integers(0, 256, n, dtype=np.uint8)
    for _ in range(10): e.ecb_host(0, a.ctypes.data, a.ctypes.data, n)
    v = []
    for _ in range(40):
        t0 = time.perf_counter(); e.ecb_host(0, a.ctypes.data, a.ctypes.data, n); v.append(time.perf_counter() - t0)
    out[mib] = statistics.median(v) * 1e6
print(json.dumps(out))
'''
libs = {"lockstep_r1": os.path.join(ROOT, "scripts", "_ab", "libt3des_b200_lockstep.so"), "current": "-"}
res = {k: {} for k in libs}
for r in range(4):
    for k, lib in libs.items():
        p = subprocess.run([sys.executable, "-c", CHILD, ROOT, lib], capture_output=True, text=True, timeout=300)
        if p.returncode:
            print(k, "failed", p.stderr[-300:], flush=True)
            continue
        for mib, us in json.loads(p.stdout.strip().splitlines()[-1]).items():
            res[k].setdefault(mib, []).append(us)
for k, d in res.items():
    print(json.dumps({"lib": k, **{f"{m}MiB_us": round(statistics.median(v), 1) for m, v in d.items()}}), flush=True)
