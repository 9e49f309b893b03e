#!/usr/bin/env python3
"""A/B of the keyed kernel's build choices, one process per configuration:
keyed_ab.py <lib.so> [label] — T3DES_KEYED_NVRTC_OPTS carries the NVRTC
defines under test.  Prints one JSON line: 1 GiB encrypt, keyed vs AUTO,
CUDA events, median of 10 after 2 warm-ups."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1305_4376_b200 import _native as N  # noqa: E402

N.LIB_PATH = os.path.abspath(sys.argv[1])
import torch  # noqa: E402

import paper_1305_4376_b200 as t3  # noqa: E402

n = (1 << 30) // 8
e = t3.Engine(0)
e.set_schedule(t3.triple_schedule(t3.parse_hex_key(os.environ.get("T3_AB_KEY", "133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57"))))
x = torch.empty(8 * n, dtype=torch.uint8, device="cuda")
e.fill_splitmix(x.data_ptr(), 0, n, 0x3DE5C0DE)
s = torch.cuda.Stream()
res = {"label": sys.argv[2] if len(sys.argv) > 2 else "", "opts": os.environ.get("T3DES_KEYED_NVRTC_OPTS", "")}
outs = {}
e.set_variant(N.VARIANT_KEYED)
res["prepare_s"] = round(e.keyed_prepare(0), 3)
for name, v in (("auto", N.VARIANT_AUTO), ("keyed", N.VARIANT_KEYED)):
    e.set_variant(v)
    y = torch.empty_like(x)
    ts = []
    for i in range(12):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        e.ecb_device(0, x.data_ptr(), y.data_ptr(), 8 * n, s.cuda_stream)
        b.record(s)
        b.synchronize()
        if i >= 2:
            ts.append(a.elapsed_time(b))
    ts.sort()
    res[name + "_ms"] = round(ts[len(ts) // 2], 4)
    outs[name] = y
res["equal"] = bool(torch.equal(outs["auto"], outs["keyed"]))
res["keyed_gbps"] = round(8 * n / res["keyed_ms"] / 1e6, 2)
res["auto_gbps"] = round(8 * n / res["auto_ms"] / 1e6, 2)
print(json.dumps(res))
