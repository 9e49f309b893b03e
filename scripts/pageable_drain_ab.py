#!/usr/bin/env python3
"""A/B: round-1 lock-step pageable staging loop (libt3des_b200_lockstep.so,
built from the previous commit into scripts/_ab/) against the decoupled
fill/drain ring, for ring depths 4/6/8; interleaved rounds, one subprocess
per measurement (a process loads one engine library)."""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, time, json
sys.path.insert(0, sys.argv[1])
from paper_1305_4376_b200 import _native as N
if sys.argv[2] != "-":
    N.LIB_PATH = sys.argv[2]
import numpy as np
import paper_1305_4376_b200 as t3
GiB = 1 << 30
x = np.random.default_rng(1).integers(0, 256, GiB, dtype=np.uint8)
y = np.empty_like(x)
e = t3.Engine(0)
e.set_schedule(t3.triple_schedule(t3.parse_hex_key("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57")))
def timed(src, dst):
    e.ecb_host(0, src.ctypes.data, dst.ctypes.data, GiB)
    best = 1e9
    for _ in range(4):
        t0 = time.perf_counter(); e.ecb_host(0, src.ctypes.data, dst.ctypes.data, GiB); best = min(best, time.perf_counter() - t0)
    return GiB / best / 1e9
print(json.dumps({"ip": timed(x, x), "oop": timed(x, y)}))
'''
VARIANTS = {
    "lockstep_4": ("scripts/_ab/libt3des_b200_lockstep.so", {}),
    "drain_4": ("-", {"T3DES_HOST_SLOTS": "4"}),
    "drain_6": ("-", {"T3DES_HOST_SLOTS": "6"}),
    "drain_8": ("-", {"T3DES_HOST_SLOTS": "8"}),
    "drain_6_s4": ("-", {"T3DES_HOST_SLOTS": "6", "T3DES_HOST_STAGE_MIB": "4"}),
    "drain_8_s4": ("-", {"T3DES_HOST_SLOTS": "8", "T3DES_HOST_STAGE_MIB": "4"}),
}
res = {k: {"ip": [], "oop": []} for k in VARIANTS}
for r in range(4):
    for name, (lib, env) in VARIANTS.items():
        lib = lib if lib == "-" else os.path.join(ROOT, lib)
        p = subprocess.run([sys.executable, "-c", CHILD, ROOT, lib], capture_output=True, text=True,
                           env=dict(os.environ, **env), timeout=300)
        if p.returncode:
            print(name, "failed", p.stderr[-500:], flush=True)
            continue
        d = json.loads(p.stdout.strip().splitlines()[-1])
        res[name]["ip"].append(d["ip"])
        res[name]["oop"].append(d["oop"])
for name, v in res.items():
    if v["ip"]:
        print(json.dumps({"variant": name, "in_place_median": round(statistics.median(v["ip"]), 2),
                          "out_of_place_median": round(statistics.median(v["oop"]), 2),
                          "in_place_all": [round(a, 1) for a in v["ip"]]}), flush=True)
