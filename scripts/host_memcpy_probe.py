#!/usr/bin/env python3
"""Host memory ceiling for the pageable path: aggregate memcpy rate of T
threads (numpy copyto releases the GIL) over 1 GiB buffers — the pageable
e2e needs two host copies per byte (in to the pinned slot, out of it)."""
import json
import threading
import time

import numpy as np

GiB = 1 << 30
src = np.ones(GiB, np.uint8)
dst = np.empty_like(src)
dst[:] = 0
for T in (1, 2, 4, 7, 8, 12, 14, 16):
    per = GiB // T

    def work(i):
        np.copyto(dst[i * per:(i + 1) * per], src[i * per:(i + 1) * per])

    best = 1e9
    for _ in range(3):
        th = [threading.Thread(target=work, args=(i,)) for i in range(T)]
        t0 = time.perf_counter()
        for t in th:
            t.start()
        for t in th:
            t.join()
        best = min(best, time.perf_counter() - t0)
    print(json.dumps({"threads": T, "copy_GBps": round(per * T / best / 1e9, 2)}), flush=True)
