#!/usr/bin/env python3
"""Slot-store policy (T3DES_HOST_NT_IN 0 = cached, 1 = streaming) against
pageable batch size with the engine's default stage choice: 16 MiB .. 1 GiB,
in place, 3 interleaved rounds of one subprocess per policy, median GB/s."""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, time, json, statistics
sys.path.insert(0, sys.argv[1])
import numpy as np
import paper_1305_4376_b200 as t3
e = t3.Engine(0)
e.set_schedule(t3.triple_schedule(t3.parse_hex_key("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57")))
out = {}
big = np.random.default_rng(0).integers(0, 256, 1 << 30, dtype=np.uint8)
for mib in (16, 64, 128, 256, 512, 1024):
    n = mib << 20
    a = big[:n]
    for _ in range(3): e.ecb_host(0, a.ctypes.data, a.ctypes.data, n)
    v = []
    for _ in range(max(5, 2048 // mib)):
        t0 = time.perf_counter(); e.ecb_host(0, a.ctypes.data, a.ctypes.data, n); v.append(time.perf_counter() - t0)
    out[mib] = n / statistics.median(v) / 1e9
print(json.dumps(out))
'''
res = {"0": {}, "1": {}, "default": {}}
for r in range(3):
    for nt in ("0", "1", "default"):
        env = dict(os.environ)
        env.pop("T3DES_HOST_NT_IN", None)
        if nt != "default":
            env["T3DES_HOST_NT_IN"] = nt
        p = subprocess.run([sys.executable, "-c", CHILD, ROOT], capture_output=True, text=True, timeout=600, env=env)
        if p.returncode:
            print(nt, p.stderr[-300:])
            continue
        for k, v in json.loads(p.stdout.strip().splitlines()[-1]).items():
            res[nt].setdefault(k, []).append(v)
for nt, d in res.items():
    print(json.dumps({"nt_in": nt, **{f"{k}MiB": round(statistics.median(v), 2) for k, v in d.items()}}), flush=True)
