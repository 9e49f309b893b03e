#!/usr/bin/env python3
"""Pageable (std::vector-style) e2e: streaming vs cached stores per copy
direction, stage size and copy threads.  Cached stores into the pinned slots
could keep a slot in the CPU's last-level cache for the H2D DMA read (DDIO),
saving two of the six host-DRAM crossings per byte; cached stores out to the
caller pay a read-for-ownership.  1 GiB, in place and out of place."""
import itertools
import json
import os
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


def timed(e, src, dst, reps=4):
    e.ecb_host(0, src.ctypes.data, dst.ctypes.data, GiB)
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        e.ecb_host(0, src.ctypes.data, dst.ctypes.data, GiB)
        best = min(best, time.perf_counter() - t0)
    return round(GiB / best / 1e9, 2)


for nt_in, nt_out, stage, th in itertools.product((1, 0), (1, 0), (1, 2, 4), (12, 16)):
    os.environ.update(T3DES_HOST_NT_IN=str(nt_in), T3DES_HOST_NT_OUT=str(nt_out), T3DES_HOST_STAGE_MIB=str(stage),
                      T3DES_HOST_COPY_THREADS=str(th))
    e = t3.Engine(0)
    e.set_schedule(ts)
    row = {"nt_in": nt_in, "nt_out": nt_out, "stage_mib": stage, "threads": th,
           "in_place": timed(e, x, x), "out_of_place": timed(e, x, y)}
    e.close()
    print(json.dumps(row), flush=True)
