#!/usr/bin/env python3
"""Per-call wall time of t3des_cu_ecb_multi (host spans, block-range shards)
on repeated calls: the first call creates the per-device contexts and their
staging buffers, later calls reuse them from the context pool.  On a 1-GPU
box the shards all go to device 0 (several contexts on one device)."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1305_4376_b200 as t3  # noqa: E402
from paper_1305_4376_b200 import _native as N  # noqa: E402

ts = t3.triple_schedule(t3.parse_hex_key("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57"))
sub = ts.sub48()
ndev = torch.cuda.device_count()
for mib in (8, 64):
    n = mib << 20
    for kind in ("pinned", "pageable"):
        if kind == "pinned":
            buf = torch.empty(n, dtype=torch.uint8).pin_memory()
            ptr = buf.data_ptr()
        else:
            arr = np.random.default_rng(0).integers(0, 256, n, dtype=np.uint8)
            ptr = arr.ctypes.data
        for g in (1, 4):
            devs = (ctypes.c_int * g)(*[i % ndev for i in range(g)])
            times = []
            for _ in range(6):
                t0 = time.perf_counter()
                rc = N.lib().t3des_cu_ecb_multi(devs, g, sub, 0, ctypes.c_void_p(ptr), ctypes.c_void_p(ptr), n)
                times.append(time.perf_counter() - t0)
                assert rc == 0, rc
            print(f"{mib:3d} MiB {kind:8s} shards={g}: first call {times[0] * 1e3:7.2f} ms, "
                  f"later calls {min(times[1:]) * 1e3:7.2f} ms ({n / min(times[1:]) / 1e9:5.1f} GB/s)", flush=True)
