#!/usr/bin/env python3
"""A/B on one box, interleaved, for the pinned 1 GiB e2e path:
  A  engine pipeline (t3des_cu_ecb_host: H2D -> kernel -> D2H, 3 streams)
  B  H2D copy -> kernel writing its output straight into the pinned host buffer
     (no D2H copy), C MiB stages on S streams, SP-table / bitsliced kernels
  C  kernel reading the pinned input over PCIe (no H2D copy) -> D2H copy
plus the bidirectional copy ceiling.  5 rounds."""
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
out = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
e = t3.Engine(0)
e.set_schedule(t3.triple_schedule(t3.parse_hex_key("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57")))
ref = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
d = h.cuda()
e.set_variant(t3.VARIANT_BITSLICE)
e.ecb_device(0, d.data_ptr(), ref.data_ptr(), nbytes, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
del d
S = 3
streams = [torch.cuda.Stream() for _ in range(4)]
bufs = [torch.empty(64 << 20, dtype=torch.uint8, device="cuda") for _ in range(4)]
d_a = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
d_b = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
hb = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()


def B(C, variant, S=2):
    def run():
        e.set_variant(variant)
        for k, off in enumerate(range(0, nbytes, C)):
            n = min(C, nbytes - off)
            s = streams[k % S]
            b = bufs[k % S]
            with torch.cuda.stream(s):
                b[:n].copy_(h[off:off + n], non_blocking=True)
                e.ecb_device(0, b.data_ptr(), out.data_ptr() + off, n, s.cuda_stream)
    return run


def Cv(C, variant, S=2):
    def run():
        e.set_variant(variant)
        for k, off in enumerate(range(0, nbytes, C)):
            n = min(C, nbytes - off)
            s = streams[k % S]
            b = bufs[k % S]
            with torch.cuda.stream(s):
                e.ecb_device(0, h.data_ptr() + off, b.data_ptr(), n, s.cuda_stream)
                out[off:off + n].copy_(b[:n], non_blocking=True)
    return run


def A():
    e.set_variant(t3.VARIANT_AUTO)
    e.ecb_host(0, h.data_ptr(), out.data_ptr(), nbytes)


def bidir():
    for i in range(4):
        with torch.cuda.stream(streams[0]):
            d_a.copy_(h[i << 28:(i + 1) << 28], non_blocking=True)
        with torch.cuda.stream(streams[1]):
            hb.copy_(d_b, non_blocking=True)


def timed(fn, check=True):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(4):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    ok = bool(torch.equal(out.cuda(), ref)) if check else None
    return [round(nbytes / best / 1e9, 2), ok]


def main():
    cases = {"A_engine": A, "bidir_ceiling": bidir,
             "B_sp_16": B(16 << 20, t3.VARIANT_SPTABLE), "B_sp_32": B(32 << 20, t3.VARIANT_SPTABLE),
             "B_bs_16": B(16 << 20, t3.VARIANT_BITSLICE), "B_sp_8_s3": B(8 << 20, t3.VARIANT_SPTABLE, 3),
             "C_sp_16": Cv(16 << 20, t3.VARIANT_SPTABLE), "C_bs_16": Cv(16 << 20, t3.VARIANT_BITSLICE)}
    for r in range(5):
        row = {"round": r}
        for name, fn in cases.items():
            out.zero_()
            row[name] = timed(fn, check=name != "bidir_ceiling")
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
