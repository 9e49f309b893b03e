#!/usr/bin/env python3
"""Pageable 4-64 MiB batches (the regime between the single-stage path and
the 1 GiB default): stage size x slot-store policy, one subprocess per
policy (the copy pools read T3DES_HOST_NT_IN at creation), median us per
in-place call."""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, time, json, statistics
sys.path.insert(0, sys.argv[1])
import numpy as np
import paper_1305_4376_b200 as t3
e = t3.Engine(0)
e.set_schedule(t3.triple_schedule(t3.parse_hex_key("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57")))
out = {}
for mib in (4, 16, 64):
    n = mib << 20
    a = np.random.default_rng(0).integers(0, 256, n, dtype=np.uint8)
    for st in ("default", "1", "2", "4", "8"):
        if st == "default": os.environ.pop("T3DES_HOST_STAGE_MIB", None)
        else: os.environ["T3DES_HOST_STAGE_MIB"] = st
        if st != "default" and int(st) > mib: continue
        for _ in range(5): e.ecb_host(0, a.ctypes.data, a.ctypes.data, n)
        v = []
        for _ in range(25):
            t0 = time.perf_counter(); e.ecb_host(0, a.ctypes.data, a.ctypes.data, n); v.append(time.perf_counter() - t0)
        out[f"{mib}MiB_stage{st}"] = round(n / statistics.median(v) / 1e9, 2)
print(json.dumps(out))
'''
for nt_in in ("0", "1"):
    p = subprocess.run([sys.executable, "-c", CHILD, ROOT], capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, T3DES_HOST_NT_IN=nt_in))
    print(json.dumps({"nt_in": nt_in, "GBps": json.loads(p.stdout.strip().splitlines()[-1]) if not p.returncode else p.stderr[-300:]}), flush=True)
