#!/usr/bin/env python3
"""Zero-copy with the bitsliced kernels: run t3des_cu_ecb_device directly on
page-locked host memory (UVA: a cudaHostAlloc pointer is a valid device
address), so the SMs read and write the payload over PCIe themselves — no
copy engines, no staging.  Compares against the copy-engine pipeline
(t3des_cu_ecb_host) for pinned batches, checks the output."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_4376_b200 as t3  # noqa: E402

KEY = "133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57"
e = t3.Engine(0)
e.set_schedule(t3.triple_schedule(t3.parse_hex_key(KEY)))
s = torch.cuda.Stream()


def timed(fn, reps=4):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


def main():
    for mib in (64, 256, 1024):
        n = mib << 20
        h = torch.empty(n, dtype=torch.uint8).pin_memory()
        h.random_(0, 255)
        o = torch.empty(n, dtype=torch.uint8).pin_memory()
        ref = torch.empty(n, dtype=torch.uint8, device="cuda")
        e.set_variant(t3.VARIANT_BITSLICE)
        d = h.cuda()
        e.ecb_device(0, d.data_ptr(), ref.data_ptr(), n, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        row = {"MiB": mib}
        for name, var in (("bitslice_tma", t3.VARIANT_BITSLICE), ("bitslice_ldg", t3.VARIANT_BITSLICE_LDG),
                          ("sptable", t3.VARIANT_SPTABLE)):
            e.set_variant(var)
            try:
                dt = timed(lambda: e.ecb_device(0, h.data_ptr(), o.data_ptr(), n, s.cuda_stream))
                ok = torch.equal(o.cuda(), ref)
                row[name] = {"GBps": round(n / dt / 1e9, 2), "ok": bool(ok)}
            except Exception as exc:  # noqa: BLE001
                row[name] = {"error": str(exc)}
            print(json.dumps(row), flush=True)
        e.set_variant(t3.VARIANT_AUTO)
        dt = timed(lambda: e.ecb_host(0, h.data_ptr(), o.data_ptr(), n))
        row["ecb_host_pipeline"] = {"GBps": round(n / dt / 1e9, 2), "ok": bool(torch.equal(o.cuda(), ref))}
        print(json.dumps(row), flush=True)
        del h, o, ref, d


if __name__ == "__main__":
    main()
