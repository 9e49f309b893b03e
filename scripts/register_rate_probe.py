#!/usr/bin/env python3
"""How fast can pageable memory be page-locked (cudaHostRegister via
t3des_cu_host_register) — single thread and several threads on disjoint
chunks — and unregistered?  Decides whether a register-on-the-fly pipeline
could beat the staged pageable path (24.5 GB/s, host-DRAM-bound)."""
import ctypes
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1305_4376_b200 import _native as N  # noqa: E402

L = N.lib()
torch.cuda.init()
GiB = 1 << 30
buf = np.ones(GiB, dtype=np.uint8)  # faulted in
base = buf.ctypes.data
try:
    from cuda.bindings import runtime as rt  # cuda-python
    for a in ("cudaDevAttrPageableMemoryAccess", "cudaDevAttrPageableMemoryAccessUsesHostPageTables",
              "cudaDevAttrHostRegisterSupported"):
        err, v = rt.cudaDeviceGetAttribute(getattr(rt.cudaDeviceAttr, a), 0)
        print(a, int(v))
except Exception as exc:  # noqa: BLE001
    print("cuda-python:", exc)

for chunk_mib in (4, 16, 64):
    C = chunk_mib << 20
    for nth in (1, 2, 4, 8):
        offs = list(range(0, GiB, C))

        def work(i):
            for o in offs[i::nth]:
                assert L.t3des_cu_host_register(base + o, C) == 0

        def unwork(i):
            for o in offs[i::nth]:
                assert L.t3des_cu_host_unregister(base + o) == 0

        for phase, fn in (("register", work), ("unregister", unwork)):
            ths = [threading.Thread(target=fn, args=(i,)) for i in range(nth)]
            t0 = time.perf_counter()
            for t in ths:
                t.start()
            for t in ths:
                t.join()
            dt = time.perf_counter() - t0
            print(json.dumps({"chunk_mib": chunk_mib, "threads": nth, "phase": phase, "GBps": round(GiB / dt / 1e9, 2)}),
                  flush=True)
