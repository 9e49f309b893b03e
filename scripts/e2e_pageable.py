#!/usr/bin/env python3
"""End-to-end GB/s of t3des_cu_ecb_host from pageable vs pinned host
buffers (1 GiB and 64 MiB), plus the raw pageable/pinned copy rates."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1305_4376_b200 as t3  # noqa: E402

e = t3.Engine(0)
e.set_schedule(t3.triple_schedule(t3.parse_hex_key("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57")))
for mib in (64, 1024):
    n = mib << 20
    page_in = np.random.default_rng(1).integers(0, 256, n, dtype=np.uint8)
    page_out = np.empty_like(page_in)
    pin_in = torch.from_numpy(page_in).pin_memory()
    pin_out = torch.empty(n, dtype=torch.uint8).pin_memory()
    for label, src, dst in (("pageable", page_in.ctypes.data, page_out.ctypes.data),
                            ("pinned", pin_in.data_ptr(), pin_out.data_ptr())):
        e.ecb_host(0, src, dst, n)
        reps = 3
        t0 = time.perf_counter()
        for _ in range(reps):
            e.ecb_host(0, src, dst, n)
        print(f"{mib} MiB {label}: {reps * n / (time.perf_counter() - t0) / 1e9:.1f} GB/s", flush=True)
    assert np.array_equal(page_out, pin_out.numpy())
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    tp = torch.from_numpy(page_in)
    for label, h in (("pageable", tp), ("pinned", pin_in)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            d.copy_(h)
        torch.cuda.synchronize()
        h2d = 3 * n / (time.perf_counter() - t0) / 1e9
        t0 = time.perf_counter()
        for _ in range(3):
            h.copy_(d)
        torch.cuda.synchronize()
        d2h = 3 * n / (time.perf_counter() - t0) / 1e9
        print(f"{mib} MiB raw {label} copy: H2D {h2d:.1f} GB/s, D2H {d2h:.1f} GB/s", flush=True)
print("host threads:", os.cpu_count())
