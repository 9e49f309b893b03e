#!/usr/bin/env python3
"""Host time per ecb_device call vs GPU time (events) for tiny batches; run
under ncu for the kernels' own durations."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_4376_b200 as t3  # noqa: E402

e = t3.Engine(0)
e.set_schedule(t3.triple_schedule(t3.parse_hex_key("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57")))
s = torch.cuda.current_stream().cuda_stream
reps = int(os.environ.get("REPS", "200"))
for kib in (8, 1024):
    n = kib * 1024
    src = torch.randint(0, 255, (n,), dtype=torch.uint8, device="cuda")
    dst = torch.empty_like(src)
    for name, v in (("bitslice", t3.VARIANT_BITSLICE), ("sptable", t3.VARIANT_SPTABLE)):
        e.set_variant(v)
        for _ in range(3):
            e.ecb_device(0, src.data_ptr(), dst.data_ptr(), n, s)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record()
        for _ in range(reps):
            e.ecb_device(0, src.data_ptr(), dst.data_ptr(), n, s)
        b.record()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        print(f"{kib} KiB {name}: host {1e6 * (t1 - t0) / reps:.1f} us/call, gpu {a.elapsed_time(b) * 1e3 / reps:.1f} us/launch", flush=True)
