#!/usr/bin/env python3
"""Generate tests/golden/c3_checksum.json: the checksum of BASELINE
configs[3]'s 64 GiB ciphertext, computed by the UNMODIFIED reference library.

Workload (the same one bench.py shards over N ranks and the configs[3] leg
encrypts on one GPU): block i of 8,589,934,592 = splitmix64(0x3DE5C0DE ^ i)
serialised big-endian, encrypted under the reference bench key
(proj/src/bench.cpp:15-16) with the reference's own encrypt_batch,
Backend::Threaded (oracle/_ref/libt3des_ref.so).  The checksum is the
shard-additive t3_checksum_kernel sum (oracle_checksum), so the value is the
sum over any block-range split — N ranks' per-shard checksums must add up to
it, and so must the single-GPU run.  Per-GiB piece checksums are kept too:
piece 0 is BASELINE configs[1] (the N = 1 bench workload), and the shard
boundaries of N = 2, 4, 8 fall on piece boundaries.

Needs oracle/_ref (built where /root/reference exists; the .so travels with
the gpurun snapshot).  ~64 x (reference 1 GiB encrypt) — about 3-4 min on a
16-thread GPU host, much longer on a small build container.  Usage:

    python tests/golden/make_c3_checksum.py [--gib 64] [--out tests/golden/c3_checksum.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

BENCH_KEY = "133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57"
SEED = 0x3DE5C0DE


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gib", type=float, default=64)
    ap.add_argument("--piece-mib", type=int, default=1024)
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "c3_checksum.json"))
    args = ap.parse_args()
    import numpy as np

    from tests.oracle_util import Oracle

    o = Oracle.load()
    if o.ref is None:
        sys.exit("oracle/_ref/libt3des_ref.so is missing (build it with make -C oracle where /root/reference exists)")
    s = o.schedule_hex(BENCH_KEY)
    total = int(args.gib * (1 << 30)) // 8
    piece = (args.piece_mib << 20) // 8
    acc_ct = acc_pt = 0
    pieces_ct, pieces_pt = [], []
    ct = np.empty(8 * piece, dtype=np.uint8)
    t0 = time.time()
    for first in range(0, total, piece):
        n = min(piece, total - first)
        pt = o.splitmix(first, n, SEED)
        out = ct[: 8 * n]
        rc = o.ref.ref_ecb(pt.ctypes.data, out.ctypes.data, pt.nbytes, s, 0, 1, 0, 0, 0)
        assert rc == 0, rc
        pieces_pt.append(o.checksum(pt, first))
        pieces_ct.append(o.checksum(out, first))
        acc_pt = (acc_pt + pieces_pt[-1]) % 2**64
        acc_ct = (acc_ct + pieces_ct[-1]) % 2**64
        print(f"{(first + n) * 8 >> 20} MiB  {time.time() - t0:.0f} s", file=sys.stderr, flush=True)
    rec = {
        "what": "BASELINE configs[3]: encrypt of the 64 GiB splitmix payload, shard-additive checksum",
        "key": BENCH_KEY, "seed": SEED, "nblocks": total, "direction": "encrypt",
        "payload": "block i = splitmix64(seed ^ i), big-endian (t3des_cu_fill_splitmix / oracle_splitmix_payload)",
        "checksum_fn": "sum_i splitmix64(0x3DE5C0DE ^ le64(block i) ^ i) mod 2^64 (t3_checksum_kernel / oracle_checksum)",
        "plaintext_checksum": f"{acc_pt:016x}",
        "ciphertext_checksum": f"{acc_ct:016x}",
        "piece_blocks": piece,
        "piece_plaintext_checksums": [f"{v:016x}" for v in pieces_pt],
        "piece_ciphertext_checksums": [f"{v:016x}" for v in pieces_ct],
        "generator": "tests/golden/make_c3_checksum.py: reference encrypt_batch, Backend::Threaded "
                     f"(oracle/_ref), {ref_threads(o)} threads, {args.piece_mib} MiB pieces, {time.time() - t0:.0f} s",
    }
    with open(args.out, "w") as f:
        json.dump(rec, f, indent=1)
        f.write("\n")
    print(json.dumps(rec))


def ref_threads(o) -> int:
    return int(o.ref.ref_resolve_workers(0))


if __name__ == "__main__":
    main()
