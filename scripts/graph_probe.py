#!/usr/bin/env python3
"""configs[0] (1 MiB encrypt + decrypt) launched eagerly vs captured once in
a CUDA graph and replayed (t3des_cu_ecb_device is stream-ordered and
capture-safe: the AUTO side-stream tail forks/joins with events), plus a
bit-exactness check of the replayed graph."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_4376_b200 as t3  # noqa: E402

e = t3.Engine(0)
e.set_schedule(t3.triple_schedule(t3.parse_hex_key("0123456789ABCDEF23456789ABCDEF01456789ABCDEF0123")))
res = {}
for nbytes in (1 << 20, (1 << 20) + 8 * 517, 64 << 10):
    x = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    e.fill_splitmix(x.data_ptr(), 0, nbytes // 8, 7)
    y, z = torch.empty_like(x), torch.empty_like(x)
    s = torch.cuda.Stream()
    reps = 50

    def pair(st):
        e.ecb_device(0, x.data_ptr(), y.data_ptr(), nbytes, st.cuda_stream)
        e.ecb_device(1, y.data_ptr(), z.data_ptr(), nbytes, st.cuda_stream)

    with torch.cuda.stream(s):
        for _ in range(5):
            pair(s)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    with torch.cuda.stream(s):
        for _ in range(reps):
            pair(s)
    b.record(s)
    torch.cuda.synchronize()
    eager = a.elapsed_time(b) * 1e3 / reps
    g = torch.cuda.CUDAGraph()
    z.zero_()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            pair(s)
    torch.cuda.synchronize()
    z.zero_()
    g.replay()
    torch.cuda.synchronize()
    ok = bool(torch.equal(z, x))
    a.record(s)
    with torch.cuda.stream(s):
        g.replay()
    b.record(s)
    torch.cuda.synchronize()
    res[nbytes] = {"eager_us_per_pair": round(eager, 2), "graph_us_per_pair": round(a.elapsed_time(b) * 1e3 / reps, 2),
                   "graph_round_trip_ok": ok}
    print(nbytes, json.dumps(res[nbytes]), flush=True)
