#!/usr/bin/env python3
"""End-to-end (pinned host -> device -> host) GB/s vs batch size for a few
pipeline stage sizes (t3des_cu_set_pipeline)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_4376_b200 as t3  # noqa: E402

e = t3.Engine(0)
e.set_schedule(t3.triple_schedule(t3.parse_hex_key("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57")))
for mib in (1, 8, 32, 64, 256, 1024):
    n = mib << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    o = torch.empty(n, dtype=torch.uint8).pin_memory()
    row = []
    for stage in (0, 2, 4, 8, 32):
        if stage == 0:
            e.set_pipeline(max(8, ((n // 8) // 8) * 8) if n >= (16 << 20) else n, 3)  # n/8 per stage
            label = "n/8"
        else:
            e.set_pipeline(stage << 20, 3)
            label = f"{stage}M"
        e.ecb_host(0, h.data_ptr(), o.data_ptr(), n)
        reps = 20 if mib <= 64 else 3
        t0 = time.perf_counter()
        for _ in range(reps):
            e.ecb_host(0, h.data_ptr(), o.data_ptr(), n)
        row.append(f"{label}:{reps * n / (time.perf_counter() - t0) / 1e9:5.1f}")
    print(f"{mib:5d} MiB  " + "  ".join(row), flush=True)
