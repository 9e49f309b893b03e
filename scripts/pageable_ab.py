#!/usr/bin/env python3
"""Interleaved A/B of the pageable staging settings that pageable_cache_sweep.py
flagged (cached stores into the pinned slots): 5 rounds x configs, 1 GiB in
place and out of place, median per config."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1305_4376_b200 as t3  # noqa: E402

GiB = 1 << 30
KEY = "133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57"
x = np.random.default_rng(1).integers(0, 256, GiB, dtype=np.uint8)
y = np.empty_like(x)
ts = t3.triple_schedule(t3.parse_hex_key(KEY))
CONFIGS = [(1, 1, 4, 12), (1, 1, 6, 14), (0, 1, 6, 14), (0, 1, 4, 12),
           (0, 0, 6, 14)]
engines = {}
for c in CONFIGS:
    nt_in, nt_out, stage, th = c
    os.environ.update(T3DES_HOST_NT_IN=str(nt_in), T3DES_HOST_NT_OUT=str(nt_out), T3DES_HOST_COPY_THREADS=str(th))
    e = t3.Engine(0)
    e.set_schedule(ts)
    os.environ["T3DES_HOST_STAGE_MIB"] = str(stage)
    e.ecb_host(0, x.ctypes.data, y.ctypes.data, 64 << 20)  # creates the copy pools with this config's env
    engines[c] = e


def timed(c, src, dst, reps=3):
    os.environ["T3DES_HOST_STAGE_MIB"] = str(c[2])
    e = engines[c]
    e.ecb_host(0, src.ctypes.data, dst.ctypes.data, GiB)
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        e.ecb_host(0, src.ctypes.data, dst.ctypes.data, GiB)
        best = min(best, time.perf_counter() - t0)
    return GiB / best / 1e9


res = {c: {"ip": [], "oop": []} for c in CONFIGS}
for r in range(5):
    for c in CONFIGS:
        res[c]["ip"].append(timed(c, x, x))
        res[c]["oop"].append(timed(c, x, y))
for c in CONFIGS:
    print(json.dumps({"nt_in": c[0], "nt_out": c[1], "stage_mib": c[2], "threads": c[3],
                      "in_place_median": round(statistics.median(res[c]["ip"]), 2),
                      "out_of_place_median": round(statistics.median(res[c]["oop"]), 2),
                      "in_place_all": [round(v, 1) for v in res[c]["ip"]]}), flush=True)
