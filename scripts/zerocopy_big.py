#!/usr/bin/env python3
"""Host batches through t3des_cu_ecb_host: DMA pipeline (AUTO) vs zero-copy
with the SP-table kernel on mapped pages, GB/s end to end; pinned buffers, or
pageable ones with ZC_PAGEABLE=1.  Usage: zerocopy_big.py [MiB ...]"""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1305_4376_b200 as t3
KEY = "133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57"
for mib in [int(a) for a in sys.argv[1:]] or (4, 64, 1024):
    n = mib << 20
    pageable = os.environ.get("ZC_PAGEABLE") == "1"
    xp = np.zeros(n, dtype=np.uint8)
    x = None if pageable else torch.empty(n, dtype=torch.uint8).pin_memory()
    ptr = xp.ctypes.data if pageable else x.data_ptr()
    row = []
    for mode, zc, var in (("dma", "0", t3.VARIANT_AUTO), ("zc-sp", str(1 << 40), t3.VARIANT_SPTABLE)):
        os.environ["T3DES_ZEROCOPY_MAX"] = zc
        e = t3.Engine(0); e.set_schedule(t3.triple_schedule(t3.parse_hex_key(KEY))); e.set_variant(var)
        e.ecb_host(0, ptr, ptr, n)
        reps = 20 if mib < 1024 else 3
        t0 = time.perf_counter()
        for _ in range(reps): e.ecb_host(0, ptr, ptr, n)
        dt = (time.perf_counter() - t0) / reps
        row.append(f"{mode} {n / dt / 1e9:6.1f} GB/s")
        e.close()
    print(f"{mib} MiB {'pageable' if pageable else 'pinned'}: " + " | ".join(row), flush=True)
