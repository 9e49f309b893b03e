#!/usr/bin/env python3
"""Pinned host batches through t3des_cu_ecb_host: DMA pipeline vs zero-copy
(SP-table kernel on the mapped host pages), per-call median wall time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1305_4376_b200 as t3  # noqa: E402

KEY = "133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57"
for kib in (8, 64, 256, 512, 1024):
    n = kib << 10
    buf = torch.empty(n, dtype=torch.uint8).pin_memory()
    buf.numpy()[:] = np.random.default_rng(kib).integers(0, 256, n, dtype=np.uint8)
    ref = None
    row = []
    for mode, zc in (("dma", "0"), ("zero-copy", str(1 << 30))):
        os.environ["T3DES_ZEROCOPY_MAX"] = zc
        e = t3.Engine(0)
        e.set_schedule(t3.triple_schedule(t3.parse_hex_key(KEY)))
        x = buf.clone().pin_memory()
        e.ecb_host(0, x.data_ptr(), x.data_ptr(), n)
        if ref is None:
            ref = x.numpy().copy()
        ok = np.array_equal(x.numpy(), ref)
        ts = []
        for _ in range(200):
            t0 = time.perf_counter()
            e.ecb_host(0, x.data_ptr(), x.data_ptr(), n)
            ts.append(time.perf_counter() - t0)
        row.append(f"{mode} {np.median(ts) * 1e6:7.1f} us{'' if ok else ' MISMATCH'}")
        e.close()
    print(f"{kib:5d} KiB pinned: " + " | ".join(row), flush=True)
