#!/usr/bin/env python3
"""Pinned 1 GiB / 256 MiB end to end through t3des_cu_ecb_host: DMA pipeline
with and without the fill/drain ramp (T3DES_RAMP_KIB), alternating runs."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_4376_b200 as t3  # noqa: E402

KEY = "133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57"
for mib in (256, 1024):
    n = mib << 20
    x = torch.empty(n, dtype=torch.uint8).pin_memory()
    for rep in range(2):
        row = []
        for ramp in ("0", "1024", "2048", "4096", "8192"):
            os.environ["T3DES_RAMP_KIB"] = ramp
            e = t3.Engine(0)
            e.set_schedule(t3.triple_schedule(t3.parse_hex_key(KEY)))
            e.ecb_host(0, x.data_ptr(), x.data_ptr(), n)
            reps = 5
            t0 = time.perf_counter()
            for _ in range(reps):
                e.ecb_host(0, x.data_ptr(), x.data_ptr(), n)
            row.append(f"ramp {ramp}K: {reps * n / (time.perf_counter() - t0) / 1e9:5.1f}")
            e.close()
        print(f"{mib} MiB pinned: " + " | ".join(row), flush=True)
