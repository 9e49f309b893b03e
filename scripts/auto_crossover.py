#!/usr/bin/env python3
"""Per-launch time of the bitsliced and SP-table kernels around the AUTO
threshold (1-3 MiB), 200 launches each."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1305_4376_b200 as t3
e = t3.Engine(0)
e.set_schedule(t3.triple_schedule(t3.parse_hex_key("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57")))
s = torch.cuda.current_stream().cuda_stream
for kib in (1024, 1536, 2048, 2560, 3072):
    n = kib * 1024
    src = torch.randint(0, 255, (n,), dtype=torch.uint8, device="cuda"); dst = torch.empty_like(src)
    row = []
    for name, v in (("bitslice", t3.VARIANT_BITSLICE), ("sptable", t3.VARIANT_SPTABLE)):
        e.set_variant(v)
        for _ in range(10): e.ecb_device(0, src.data_ptr(), dst.data_ptr(), n, s)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(200): e.ecb_device(0, src.data_ptr(), dst.data_ptr(), n, s)
        b.record(); torch.cuda.synchronize()
        row.append(f"{name} {a.elapsed_time(b) * 5:6.1f} us")
    print(kib, "KiB:", " | ".join(row), flush=True)
