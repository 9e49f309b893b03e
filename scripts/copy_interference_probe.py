#!/usr/bin/env python3
"""Do PCIe copies slow down while a kernel runs?  (scripts/e2e_timeline_probe.py
showed the 32 MiB stage copies taking 0.72-0.82 ms instead of 0.69 once any
kernel sits between H2D and D2H.)

  1. bidirectional pinned copies alone (8 x 256 MiB each way);
  2. the same while another stream runs a device-resident kernel back to back
     (bitsliced 3DES / SP-table / a torch memory-bound pass);
  3. the split-queue pipeline (H2D stream, kernel stream, D2H stream chained by
     events, ring of R buffers) with the bitsliced kernel, against the
     engine's per-stage-stream pattern.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_4376_b200 as t3  # noqa: E402

MiB = 1 << 20
C = 256 * MiB
IT = 8
h_in = torch.empty(C, dtype=torch.uint8).pin_memory()
h_out = torch.empty(C, dtype=torch.uint8).pin_memory()
d_a = torch.empty(C, dtype=torch.uint8, device="cuda")
d_b = torch.empty(C, dtype=torch.uint8, device="cuda")
s_in, s_out, s_k = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
e = t3.Engine(0)
e.set_schedule(t3.triple_schedule(t3.parse_hex_key("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57")))
big = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")
big2 = torch.empty_like(big)
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def copies(h2d=True, d2h=True):
    t0, e1, e2 = ev(), ev(), ev()
    t0.record(s_in)
    s_out.wait_event(t0)
    for _ in range(IT):
        if h2d:
            with torch.cuda.stream(s_in):
                d_a.copy_(h_in, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s_out):
                h_out.copy_(d_b, non_blocking=True)
    e1.record(s_in)
    e2.record(s_out)
    return t0, e1, e2


def background(kind, n):
    with torch.cuda.stream(s_k):
        for _ in range(n):
            if kind == "bitslice":
                e.set_variant(t3.VARIANT_BITSLICE)
                e.ecb_device(0, big.data_ptr(), big2.data_ptr(), big.numel(), s_k.cuda_stream)
            elif kind == "sptable":
                e.set_variant(t3.VARIANT_SPTABLE)
                e.ecb_device(0, big.data_ptr(), big2.data_ptr(), big.numel() // 2, s_k.cuda_stream)
            elif kind == "torch":
                torch.bitwise_not(big, out=big2)


def main():
    res = {}
    for kind in ("none", "bitslice", "sptable", "torch"):
        for h2d, d2h, name in ((True, False, "h2d"), (False, True, "d2h"), (True, True, "bidir")):
            torch.cuda.synchronize()
            kb0 = ev()
            kb0.record(s_k)
            background(kind, {"none": 0, "bitslice": 6, "sptable": 6, "torch": 40}[kind])
            kb1 = ev()
            kb1.record(s_k)
            t0, e1, e2 = copies(h2d, d2h)
            torch.cuda.synchronize()
            ms = max(t0.elapsed_time(e1) if h2d else 0, t0.elapsed_time(e2) if d2h else 0)
            res[f"{kind}:{name}"] = {"GBps_each_way": round(IT * C / ms / 1e6, 2),
                                     "background_ms": round(kb0.elapsed_time(kb1), 2), "copy_ms": round(ms, 2)}
            print(kind, name, json.dumps(res[f"{kind}:{name}"]), flush=True)
    # kernel alone for reference
    for kind in ("bitslice", "sptable", "torch"):
        torch.cuda.synchronize()
        kb0 = ev()
        kb0.record(s_k)
        background(kind, 3)
        kb1 = ev()
        kb1.record(s_k)
        torch.cuda.synchronize()
        print(kind, "alone_ms_per_launch", round(kb0.elapsed_time(kb1) / 3, 3), flush=True)


if __name__ == "__main__":
    main()
