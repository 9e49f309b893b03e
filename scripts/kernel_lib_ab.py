#!/usr/bin/env python3
"""A/B of engine builds (scripts/_ab/*.so, e.g. S-box emission orders from
T3_GEN_ORDER) on the shipped bitsliced kernel: 1 GiB device-resident encrypt,
20 launches timed with CUDA events per measurement, one subprocess per
measurement (a process loads one engine library), interleaved rounds."""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json
sys.path.insert(0, sys.argv[1])
from paper_1305_4376_b200 import _native as N
if sys.argv[2] != "-":
    N.LIB_PATH = sys.argv[2]
import torch
import paper_1305_4376_b200 as t3
n = 1 << 30
e = t3.Engine(0)
e.set_schedule(t3.triple_schedule(t3.parse_hex_key("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57")))
e.set_variant(t3.VARIANT_BITSLICE)
src = torch.empty(n, dtype=torch.uint8, device="cuda"); dst = torch.empty_like(src)
s = torch.cuda.current_stream().cuda_stream
e.fill_splitmix(src.data_ptr(), 0, n // 8, 0x3DE5C0DE, s)
for _ in range(5): e.ecb_device(0, src.data_ptr(), dst.data_ptr(), n, s)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); a.record()
for _ in range(20): e.ecb_device(0, src.data_ptr(), dst.data_ptr(), n, s)
b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b) / 20
ref = e.checksum(dst.data_ptr(), 0, n // 8, s)
print(json.dumps({"GBps": n / ms / 1e6, "checksum": ref}))
'''
libs = {"default": "-"}
for f in sorted(os.listdir(os.path.join(ROOT, "scripts", "_ab"))):
    if f.startswith("lib_") and f.endswith(".so"):
        libs[f[4:-3]] = os.path.join(ROOT, "scripts", "_ab", f)
res = {k: [] for k in libs}
sums = {}
for r in range(int(os.environ.get("AB_ROUNDS", "5"))):
    for k, lib in libs.items():
        p = subprocess.run([sys.executable, "-c", CHILD, ROOT, lib], capture_output=True, text=True, timeout=300)
        if p.returncode:
            print(k, "failed", p.stderr[-400:], flush=True)
            continue
        d = json.loads(p.stdout.strip().splitlines()[-1])
        res[k].append(d["GBps"])
        sums.setdefault(k, set()).add(d["checksum"])
ref = sums.get("default")
for k, v in res.items():
    if v:
        print(json.dumps({"lib": k, "median_GBps": round(statistics.median(v), 2), "all": [round(x, 1) for x in v],
                          "output_equals_default": sums.get(k) == ref}), flush=True)
