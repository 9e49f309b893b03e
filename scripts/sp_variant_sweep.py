#!/usr/bin/env python3
"""SP-table kernel code-generation masks (T3_SPV_*, env T3DES_SP_VAR):
1 GiB encrypt GB/s, small-launch latency, and bit-identity with mask 0."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_4376_b200 as t3  # noqa: E402

KEY = "133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57"
masks = [int(a) for a in sys.argv[1:]] or [0, 234]
wgs = [int(w) for w in os.environ.get("SP_WG", "0").split(",")]
masks = [(m, w) for m in masks for w in wgs]
s = torch.cuda.current_stream().cuda_stream
n = (1 << 30) // 8
src = torch.empty(8 * n, dtype=torch.uint8, device="cuda")
ref = torch.empty_like(src)
dst = torch.empty_like(src)
small = torch.randint(0, 255, (1 << 20,), dtype=torch.uint8, device="cuda")
sdst = torch.empty_like(small)
for k, (m, wg) in enumerate(masks):
    os.environ["T3DES_SP_VAR"] = str(m)
    e = t3.Engine(0)
    e.set_launch(0, wg)
    e.set_schedule(t3.triple_schedule(t3.parse_hex_key(KEY)))
    e.set_variant(t3.VARIANT_SPTABLE)
    if k == 0:
        e.fill_splitmix(src.data_ptr(), 0, n, 0x3DE5C0DE, s)
    out = ref if k == 0 else dst
    e.ecb_device(0, src.data_ptr(), out.data_ptr(), 8 * n, s)
    torch.cuda.synchronize()
    same = bool(torch.equal(out, ref))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        e.ecb_device(0, src.data_ptr(), out.data_ptr(), 8 * n, s)
    b.record()
    torch.cuda.synchronize()
    gbs = 3 * 8 * n / (a.elapsed_time(b) / 1e3) / 1e9
    lat = {}
    for kib in (8, 1024):
        for _ in range(5):
            e.ecb_device(0, small.data_ptr(), sdst.data_ptr(), kib * 1024, s)
        a.record()
        for _ in range(100):
            e.ecb_device(0, small.data_ptr(), sdst.data_ptr(), kib * 1024, s)
        b.record()
        torch.cuda.synchronize()
        lat[kib] = a.elapsed_time(b) * 10
    print(f"SPV={m:2d} wg={wg:4d}: 1 GiB {gbs:6.1f} GB/s | 8 KiB {lat[8]:5.1f} us | 1 MiB {lat[1024]:5.1f} us | "
          f"identical to SPV=0: {same}", flush=True)
    e.close()
