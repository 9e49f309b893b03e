#!/usr/bin/env python3
"""Per-call wall time of the Python batch API (encrypt_batch) for small
device-resident and host batches: what a caller pays per call on top of
the kernel (schedule install, launch, synchronisation)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1305_4376_b200 as t3  # noqa: E402

ts = t3.triple_schedule(t3.parse_hex_key("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57"))
for kib in (8, 1024):
    n = kib << 10
    d = torch.randint(0, 255, (n,), dtype=torch.uint8, device="cuda")
    h = np.random.default_rng(0).integers(0, 256, n, dtype=np.uint8)
    for name, buf in (("device", d), ("host", h)):
        for _ in range(20):
            t3.encrypt_batch(buf, buf, ts)
        torch.cuda.synchronize()
        reps = 500
        t0 = time.perf_counter()
        for _ in range(reps):
            t3.encrypt_batch(buf, buf, ts)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / reps
        print(f"{kib:5d} KiB {name:6s}: {dt * 1e6:8.1f} us per encrypt_batch call", flush=True)
