#!/usr/bin/env python3
"""Median wall time per t3des_cu_ecb_host call for small host batches (the
reference's default stream chunk is 1 MiB), pageable and pinned, in place,
through the Python Engine (ctypes overhead ~1-2 us included)."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1305_4376_b200 as t3  # noqa: E402

e = t3.Engine(0)
e.set_schedule(t3.triple_schedule(t3.parse_hex_key("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57")))
for kib in (8, 64, 256, 512, 1024, 2048, 4096, 16384):
    n = kib << 10
    row = {"KiB": kib}
    for kind in ("pageable", "pinned"):
        if kind == "pinned":
            t = torch.empty(n, dtype=torch.uint8).pin_memory()
            p = t.data_ptr()
        else:
            a = np.random.default_rng(0).integers(0, 256, n, dtype=np.uint8)
            p = a.ctypes.data
        for _ in range(20):
            e.ecb_host(0, p, p, n)
        v = []
        for _ in range(200):
            t0 = time.perf_counter()
            e.ecb_host(0, p, p, n)
            v.append(time.perf_counter() - t0)
        row[kind + "_us"] = round(statistics.median(v) * 1e6, 1)
    print(json.dumps(row), flush=True)
