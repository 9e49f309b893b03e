#!/usr/bin/env python3
"""Small driver for ncu captures: 1 GiB device-resident encrypt with the
bench key, a few launches of each kernel variant (bitsliced, SP-table)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_4376_b200 as t3  # noqa: E402

n = (int(os.environ.get("T3_GIB", "1")) << 30) // 8
e = t3.Engine(0)
e.set_schedule(t3.triple_schedule(t3.parse_hex_key("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57")))
src = torch.empty(8 * n, dtype=torch.uint8, device="cuda")
dst = torch.empty_like(src)
s = torch.cuda.current_stream().cuda_stream
e.fill_splitmix(src.data_ptr(), 0, n, 0x3DE5C0DE, s)
variants = sys.argv[1:] or ["bitslice", "sptable"]
for v in variants:
    e.set_variant({"sptable": t3.VARIANT_SPTABLE, "bitslice_ldg": t3.VARIANT_BITSLICE_LDG,
                   "bitslice_alu": t3.VARIANT_BITSLICE_ALU}.get(v, t3.VARIANT_BITSLICE))
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for i in range(3):
        ev[0].record()
        e.ecb_device(0, src.data_ptr(), dst.data_ptr(), 8 * n, s)
        ev[1].record()
        torch.cuda.synchronize()
        print(f"{v} launch {i}: {ev[0].elapsed_time(ev[1]):.3f} ms", flush=True)
