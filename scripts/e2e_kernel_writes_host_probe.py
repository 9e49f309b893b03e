#!/usr/bin/env python3
"""Pinned e2e with the kernel writing its output straight into the host
buffer (UVA, posted PCIe writes spread over the kernel) instead of a D2H
copy: stage k = H2D copy (copy engine) -> kernel(device buf -> host out) on
stream k % S.  Against the engine's H2D -> kernel -> D2H pipeline."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_4376_b200 as t3  # noqa: E402

GiB = 1 << 30
nbytes = GiB
h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
h.random_(0, 255)
ref = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
e = t3.Engine(0)
e.set_schedule(t3.triple_schedule(t3.parse_hex_key("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57")))
d = h.cuda()
e.set_variant(t3.VARIANT_BITSLICE)
e.ecb_device(0, d.data_ptr(), ref.data_ptr(), nbytes, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
del d
out = torch.empty(nbytes, dtype=torch.uint8).pin_memory()


def run(C, S, variant, streams, bufs):
    e.set_variant(variant)
    for k, off in enumerate(range(0, nbytes, C)):
        n = min(C, nbytes - off)
        s = streams[k % S]
        b = bufs[k % S]
        with torch.cuda.stream(s):
            b[:n].copy_(h[off:off + n], non_blocking=True)
            e.ecb_device(0, b.data_ptr(), out.data_ptr() + off, n, s.cuda_stream)


def main():
    for C_mib in (16, 32, 64):
        C = C_mib << 20
        for S in (2, 3, 4):
            streams = [torch.cuda.Stream() for _ in range(S)]
            bufs = [torch.empty(C, dtype=torch.uint8, device="cuda") for _ in range(S)]
            row = {"chunk_mib": C_mib, "S": S}
            for name, v in (("bitslice_ldg", t3.VARIANT_BITSLICE_LDG), ("bitslice_tma", t3.VARIANT_BITSLICE),
                            ("sptable", t3.VARIANT_SPTABLE)):
                f = lambda: run(C, S, v, streams, bufs)  # noqa: E731
                f()
                torch.cuda.synchronize()
                best = 1e9
                for _ in range(5):
                    t0 = time.perf_counter()
                    f()
                    torch.cuda.synchronize()
                    best = min(best, time.perf_counter() - t0)
                ok = torch.equal(out.cuda(), ref)
                row[name] = [round(nbytes / best / 1e9, 2), bool(ok)]
            print(json.dumps(row), flush=True)
    e.set_variant(t3.VARIANT_AUTO)
    best = 1e9
    for _ in range(6):
        t0 = time.perf_counter()
        e.ecb_host(0, h.data_ptr(), out.data_ptr(), nbytes)
        best = min(best, time.perf_counter() - t0)
    print(json.dumps({"engine_pipeline": round(nbytes / best / 1e9, 2)}), flush=True)


if __name__ == "__main__":
    main()
