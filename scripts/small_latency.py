#!/usr/bin/env python3
"""GPU time per launch (CUDA events, back-to-back launches) of each variant
for small and mid-size batches, and the BASELINE configs[0] loop (1 MiB
encrypt + decrypt)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_4376_b200 as t3  # noqa: E402

e = t3.Engine(0)
e.set_schedule(t3.triple_schedule(t3.parse_hex_key("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57")))
s = torch.cuda.current_stream().cuda_stream
V = (("bitslice", t3.VARIANT_BITSLICE), ("sptable", t3.VARIANT_SPTABLE),
     ("auto", t3.VARIANT_AUTO))
for kib in (8, 64, 256, 1024, 2048, 4096, 8192, 16384, 65536):
    n = kib * 1024
    src = torch.randint(0, 255, (n,), dtype=torch.uint8, device="cuda")
    dst = torch.empty_like(src)
    row = []
    for name, v in V:
        e.set_variant(v)
        for _ in range(5):
            e.ecb_device(0, src.data_ptr(), dst.data_ptr(), n, s)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 100 if kib <= 4096 else 20
        a.record()
        for _ in range(reps):
            e.ecb_device(0, src.data_ptr(), dst.data_ptr(), n, s)
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) * 1e3 / reps
        row.append(f"{name} {us:7.1f} us ({n / us / 1e3:6.1f} GB/s)")
    print(f"{kib:6d} KiB: " + " | ".join(row), flush=True)
n = 1 << 20
d = torch.randint(0, 255, (n,), dtype=torch.uint8, device="cuda")
y, z = torch.empty_like(d), torch.empty_like(d)
for name, v in V:
    e.set_variant(v)
    for _ in range(3):
        e.ecb_device(0, d.data_ptr(), y.data_ptr(), n, s)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50):
        e.ecb_device(0, d.data_ptr(), y.data_ptr(), n, s)
        e.ecb_device(1, y.data_ptr(), z.data_ptr(), n, s)
    b.record()
    torch.cuda.synchronize()
    assert torch.equal(z, d)
    print(f"configs[0] 1 MiB enc+dec {name}: {a.elapsed_time(b) * 1e3 / 50:.1f} us", flush=True)
