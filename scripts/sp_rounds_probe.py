#!/usr/bin/env python3
"""SP-table kernel GPU time for a tiny batch with 48 rounds (3-key) vs 16
rounds (option 3 collapses to single DES): separates per-round latency from
the fixed cost (launch, 64 KiB shared-table fill)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_4376_b200 as t3  # noqa: E402

s = torch.cuda.current_stream().cuda_stream
for key in ("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57", "0123456789ABCDEF"):
    e = t3.Engine(0)
    e.set_schedule(t3.triple_schedule(t3.parse_hex_key(key)))
    e.set_variant(t3.VARIANT_SPTABLE)
    for kib in (8, 1024):
        n = kib * 1024
        src = torch.randint(0, 255, (n,), dtype=torch.uint8, device="cuda")
        dst = torch.empty_like(src)
        for _ in range(5):
            e.ecb_device(0, src.data_ptr(), dst.data_ptr(), n, s)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(100):
            e.ecb_device(0, src.data_ptr(), dst.data_ptr(), n, s)
        b.record()
        torch.cuda.synchronize()
        print(f"{len(key) * 4}-bit key, {kib} KiB: {a.elapsed_time(b) * 10:.1f} us/launch", flush=True)
    e.close()
