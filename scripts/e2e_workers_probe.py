#!/usr/bin/env python3
"""Pinned and pageable 1 GiB end to end: one pipeline (t3des_cu_ecb_host)
against 2-3 concurrent pipelines on the same GPU (t3des_cu_ecb_workers: the
batch split into block ranges, one context + host thread each).  Several
pipelines interleave their copy bursts; does that close the gap to the
bidirectional copy ceiling?  Interleaved rounds, medians."""
import ctypes
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1305_4376_b200 as t3  # noqa: E402
from paper_1305_4376_b200 import _native as N  # noqa: E402

GiB = 1 << 30
ts = t3.triple_schedule(t3.parse_hex_key("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57"))
sub = ts.sub48()
pin = torch.empty(GiB, dtype=torch.uint8).pin_memory()
pin.random_(0, 255)
page = np.random.default_rng(1).integers(0, 256, GiB, dtype=np.uint8)
e = t3.Engine(0)
e.set_schedule(ts)


def workers(w, p):
    rc = N.lib().t3des_cu_ecb_workers(w, 0, sub, 0, p, p, GiB)
    assert rc == 0, rc


cases = {
    "pinned_ecb_host": lambda: e.ecb_host(0, pin.data_ptr(), pin.data_ptr(), GiB),
    "pinned_workers1": lambda: workers(1, pin.data_ptr()),
    "pinned_workers2": lambda: workers(2, pin.data_ptr()),
    "pinned_workers3": lambda: workers(3, pin.data_ptr()),
    "pinned_workers4": lambda: workers(4, pin.data_ptr()),
    "pageable_ecb_host": lambda: e.ecb_host(0, page.ctypes.data, page.ctypes.data, GiB),
    "pageable_workers2": lambda: workers(2, page.ctypes.data),
    "pageable_workers3": lambda: workers(3, page.ctypes.data),
}
res = {k: [] for k in cases}
for f in cases.values():
    f()
for r in range(4):
    for k, f in cases.items():
        best = 1e9
        for _ in range(3):
            t0 = time.perf_counter()
            f()
            best = min(best, time.perf_counter() - t0)
        res[k].append(GiB / best / 1e9)
print(json.dumps({k: round(statistics.median(v), 2) for k, v in res.items()}))
