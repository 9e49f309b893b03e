#!/usr/bin/env python3
"""Per-launch time of each variant for small batches (CUDA events, 200 reps)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_4376_b200 as t3  # noqa: E402

e = t3.Engine(0)
e.set_schedule(t3.triple_schedule(t3.parse_hex_key("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57")))
s = torch.cuda.current_stream().cuda_stream
for kib in (8, 64, 256, 1024, 4096, 16384, 65536):
    n = kib * 1024
    src = torch.randint(0, 255, (n,), dtype=torch.uint8, device="cuda")
    dst = torch.empty_like(src)
    row = []
    for name, v in (("bitslice", t3.VARIANT_BITSLICE), ("sptable", t3.VARIANT_SPTABLE)):
        e.set_variant(v)
        for _ in range(10):
            e.ecb_device(0, src.data_ptr(), dst.data_ptr(), n, s)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 200 if kib <= 4096 else 20
        a.record()
        for _ in range(reps):
            e.ecb_device(0, src.data_ptr(), dst.data_ptr(), n, s)
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) * 1e3 / reps
        row.append(f"{name} {us:8.1f} us ({n / us / 1e3:7.1f} GB/s)")
    print(f"{kib:6d} KiB: " + " | ".join(row), flush=True)

# odd sizes: full tiles + a partial tile (AUTO runs the tail concurrently)
for mib in (16, 64):
    n = (mib << 20) + 8 * 517
    src = torch.randint(0, 255, (n,), dtype=torch.uint8, device="cuda")
    dst = torch.empty_like(src)
    row = []
    for name, v in (("auto", t3.VARIANT_AUTO), ("bitslice", t3.VARIANT_BITSLICE)):
        e.set_variant(v)
        for _ in range(5):
            e.ecb_device(0, src.data_ptr(), dst.data_ptr(), n, s)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            e.ecb_device(0, src.data_ptr(), dst.data_ptr(), n, s)
        b.record()
        torch.cuda.synchronize()
        row.append(f"{name} {a.elapsed_time(b) * 1e3 / 20:8.1f} us")
    print(f"{mib} MiB + 517 blocks: " + " | ".join(row), flush=True)
