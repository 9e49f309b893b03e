#!/usr/bin/env python3
"""Pageable 1 GiB: split of the copy threads between the fill side (into the
slots) and the drain side (out of them), total 14 (and 12, 16), interleaved
rounds of one subprocess per split, median GB/s in place and out of place."""
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
n = 1 << 30
x = np.random.default_rng(0).integers(0, 256, n, dtype=np.uint8)
y = np.empty_like(x)
out = {}
for name, (s, d) in (("ip", (x, x)), ("oop", (x, y))):
    for _ in range(2): e.ecb_host(0, s.ctypes.data, d.ctypes.data, n)
    v = []
    for _ in range(5):
        t0 = time.perf_counter(); e.ecb_host(0, s.ctypes.data, d.ctypes.data, n); v.append(time.perf_counter() - t0)
    out[name] = n / statistics.median(v) / 1e9
print(json.dumps(out))
'''
cfgs = [(14, 7), (14, 6), (14, 8), (14, 5), (14, 9), (12, 6), (16, 8)]
res = {c: {"ip": [], "oop": []} for c in cfgs}
for r in range(3):
    for total, nin in cfgs:
        env = dict(os.environ, T3DES_HOST_COPY_THREADS=str(total), T3DES_HOST_IN_THREADS=str(nin))
        p = subprocess.run([sys.executable, "-c", CHILD, ROOT], capture_output=True, text=True, timeout=300, env=env)
        if p.returncode:
            print(total, nin, p.stderr[-200:])
            continue
        d = json.loads(p.stdout.strip().splitlines()[-1])
        res[(total, nin)]["ip"].append(d["ip"])
        res[(total, nin)]["oop"].append(d["oop"])
for (total, nin), d in res.items():
    print(json.dumps({"total": total, "in": nin, "in_place": round(statistics.median(d["ip"]), 2),
                      "out_of_place": round(statistics.median(d["oop"]), 2)}), flush=True)
