#!/usr/bin/env python3
"""Soak test of the host-buffer paths: 4 threads issue random batches for
T seconds — pageable / pinned, 0 B .. 64 MiB, in place or not, workers 0/2/3,
encrypt then decrypt — checking the round trip of every batch and the
oracle on sampled blocks.  Prints counts and any mismatch."""
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1305_4376_b200 as t3  # noqa: E402
from tests.oracle_util import Oracle  # noqa: E402

SECS = float(os.environ.get("SOAK_S", "60"))
KEYS = ["133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57", "0123456789ABCDEF23456789ABCDEF01", "0123456789ABCDEF"]
o = Oracle.load()
stats = {"batches": 0, "bytes": 0, "errors": []}
lock = threading.Lock()
t_end = time.time() + SECS


def work(tid):
    rng = np.random.default_rng(1000 + tid)
    while time.time() < t_end:
        n = int(rng.choice([0, 1, 17, 1024, 1025, int(rng.integers(1, 1 << 20)), int(rng.integers(1, 8 << 20))]))
        key = KEYS[int(rng.integers(0, 3))]
        ts = t3.triple_schedule(t3.parse_hex_key(key))
        s = o.schedule_hex(key)
        pinned = bool(rng.integers(0, 2))
        if pinned:
            buf = torch.empty(8 * n, dtype=torch.uint8).pin_memory()
            x = buf.numpy()
        else:
            x = np.empty(8 * n, np.uint8)
        x[:] = rng.integers(0, 256, 8 * n, dtype=np.uint8)
        orig = x.copy()
        y = x if rng.integers(0, 2) else np.empty_like(x)
        cfg = t3.DispatchConfig(workers=int(rng.choice([0, 0, 2, 3])))
        try:
            t3.encrypt_batch(x, y, ts, cfg)
            if n:
                idx = rng.integers(0, n, min(n, 256))
                blocks = orig.reshape(-1, 8)[idx].reshape(-1)
                want = o.ecb(blocks, s, 0).reshape(-1, 8)
                if not np.array_equal(y.reshape(-1, 8)[idx], want):
                    raise AssertionError("oracle mismatch")
            z = np.empty_like(y)
            t3.decrypt_batch(y, z, ts, cfg)
            if not np.array_equal(z, orig):
                raise AssertionError("round trip mismatch")
        except Exception as exc:  # noqa: BLE001
            with lock:
                stats["errors"].append(f"t{tid} n={n} pinned={pinned} {exc!r}"[:200])
        with lock:
            stats["batches"] += 1
            stats["bytes"] += 16 * n


th = [threading.Thread(target=work, args=(i,)) for i in range(4)]
for t in th:
    t.start()
for t in th:
    t.join()
print(json.dumps({"seconds": SECS, **stats, "errors": stats["errors"][:10], "n_errors": len(stats["errors"])}))
