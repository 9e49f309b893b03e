#!/usr/bin/env python3
"""Sweep the host-path pipeline shape (t3des_cu_set_pipeline) on 1 GiB of
pinned host memory; also reports raw PCIe copy rates for context."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_4376_b200 as t3  # noqa: E402

nbytes = 1 << 30
h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
h2 = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
res = {}
for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    res[name] = round(3 * nbytes / (time.perf_counter() - t0) / 1e9, 2)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
h2.copy_(h)
torch.cuda.synchronize()
d2 = torch.empty_like(d)
t0 = time.perf_counter()
for _ in range(3):
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
res["bidir_each_way"] = round(3 * nbytes / (time.perf_counter() - t0) / 1e9, 2)
del d, d2
torch.cuda.empty_cache()
e = t3.Engine(0)
e.set_schedule(t3.triple_schedule(t3.parse_hex_key("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57")))
sweep = {}
for chunk_mib in (8, 16, 32, 64, 128):
    for streams in (2, 3, 4, 6):
        e.set_pipeline(chunk_mib << 20, streams)
        e.ecb_host(0, h.data_ptr(), h.data_ptr(), nbytes)
        t0 = time.perf_counter()
        for _ in range(3):
            e.ecb_host(0, h.data_ptr(), h.data_ptr(), nbytes)
        sweep[f"{chunk_mib}MiBx{streams}"] = round(3 * nbytes / (time.perf_counter() - t0) / 1e9, 2)
        print(chunk_mib, streams, sweep[f"{chunk_mib}MiBx{streams}"], flush=True)
res["ecb_host_GBps"] = sweep
print(json.dumps(res))
