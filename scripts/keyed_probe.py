#!/usr/bin/env python3
"""VARIANT_KEYED on the GPU: NVRTC compile + load time (t3des_cu_keyed_prepare,
first use and cache hit) and 1 GiB device-resident throughput of the keyed
kernel next to the shipped table-driven kernel (AUTO), CUDA events on the
launching stream, L2 flushed between launches; outputs compared."""
import json
import sys
import time

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_4376_b200 as t3  # noqa: E402
from paper_1305_4376_b200 import _native as N  # noqa: E402

KEY = "133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57"
n = (1 << 30) // 8
e = t3.Engine(0)
e.set_schedule(t3.triple_schedule(t3.parse_hex_key(sys.argv[1] if len(sys.argv) > 1 else KEY)))
x = torch.empty(8 * n, dtype=torch.uint8, device="cuda")
e.fill_splitmix(x.data_ptr(), 0, n, 0x3DE5C0DE)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
res = {}
e.set_variant(N.VARIANT_KEYED)
t0 = time.perf_counter()
res["prepare_first_s"] = e.keyed_prepare(0)
res["prepare_first_wall_s"] = time.perf_counter() - t0
res["prepare_again_s"] = e.keyed_prepare(0)
res["prepare_decrypt_s"] = e.keyed_prepare(1)
outs = {}
for name, v in (("auto", N.VARIANT_AUTO), ("keyed", N.VARIANT_KEYED), ("auto2", N.VARIANT_AUTO), ("keyed2", N.VARIANT_KEYED)):
    e.set_variant(v)
    y = torch.empty_like(x)
    ts = []
    with torch.cuda.stream(s):
        for i in range(12):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            e.ecb_device(0, x.data_ptr(), y.data_ptr(), 8 * n, s.cuda_stream)
            b.record(s)
            b.synchronize()
            if i >= 2:
                ts.append(a.elapsed_time(b))
    ts.sort()
    res[name] = {"ms_min": ts[0], "ms_median": ts[len(ts) // 2], "gbps_median": 8 * n / ts[len(ts) // 2] / 1e6}
    outs[name] = y
res["keyed_equals_auto"] = bool(torch.equal(outs["auto"], outs["keyed"]))
e.set_variant(N.VARIANT_KEYED)
z = torch.empty_like(x)
e.ecb_device(1, outs["keyed"].data_ptr(), z.data_ptr(), 8 * n, 0)
torch.cuda.synchronize()
res["keyed_roundtrip"] = bool(torch.equal(z, x))
print(json.dumps(res, indent=1))
