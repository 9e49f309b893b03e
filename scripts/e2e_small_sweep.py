#!/usr/bin/env python3
"""Small/mid host batches through t3des_cu_ecb_host: per-call time vs
pipeline stage size, pinned and pageable buffers (in place).  Decides the
stage size the engine picks below 8 MiB."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1305_4376_b200 as t3  # noqa: E402

e = t3.Engine(0)
e.set_schedule(t3.triple_schedule(t3.parse_hex_key("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57")))
KIB = 1 << 10
for size in (256 * KIB, 1024 * KIB, 4096 * KIB, 16384 * KIB):
    pinned = torch.empty(size, dtype=torch.uint8).pin_memory()
    page = np.random.default_rng(0).integers(0, 256, size, dtype=np.uint8)
    for kind, ptr in (("pinned", pinned.data_ptr()), ("pageable", page.ctypes.data)):
        row = []
        d = t3.Engine(0)  # default stage choice (no set_pipeline)
        d.set_schedule(t3.triple_schedule(t3.parse_hex_key("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57")))
        for _ in range(5):
            d.ecb_host(0, ptr, ptr, size)
        ts = []
        for _ in range(30):
            t0 = time.perf_counter()
            d.ecb_host(0, ptr, ptr, size)
            ts.append(time.perf_counter() - t0)
        d.close()
        row.append(f"default:{np.median(ts) * 1e6:7.1f}us |")
        for stage in (64 * KIB, 128 * KIB, 256 * KIB, 512 * KIB, 1024 * KIB, 2048 * KIB, 4096 * KIB, 8192 * KIB):
            if stage > size:
                continue
            e.set_pipeline(stage, 3)
            for _ in range(5):
                e.ecb_host(0, ptr, ptr, size)
            ts = []
            for _ in range(30):
                t0 = time.perf_counter()
                e.ecb_host(0, ptr, ptr, size)
                ts.append(time.perf_counter() - t0)
            row.append(f"{stage // KIB}K:{np.median(ts) * 1e6:7.1f}us")
        print(f"{size // KIB:6d} KiB {kind:8s} " + " ".join(row), flush=True)
