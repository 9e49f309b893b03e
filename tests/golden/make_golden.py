#!/usr/bin/env python3
"""Generate tests/golden/golden.json from the UNMODIFIED reference library.

Run in the build container (needs /root/reference and oracle/_ref built by
`make -C oracle`).  The JSON it writes is committed; the tests read only the
JSON, so they also run where /root/reference does not exist (the GPU box).

Contents
  kats            the reference's embedded vectors (proj/src/verify.cpp:15-40)
                  plus the 3-block NIST SP 800-67 example, re-derived through
                  the reference's encrypt_batch (ScalarReference backend)
  walkthrough     16 subkeys of key 133457799BBCDFF1 from reference key_schedule
  batches         encrypt/decrypt of make_payload-style inputs for the keying
                  options and the edge-case block counts of BASELINE configs
                  [0] and [4]: small outputs in full (hex), larger ones as
                  SHA-256 of the output (plus first/last block)
"""
from __future__ import annotations

import ctypes
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF = os.path.join(ROOT, "oracle", "_ref", "libt3des_ref.so")

DES_KATS = [  # verify.cpp:15-22
    (0x133457799BBCDFF1, 0x0123456789ABCDEF, 0x85E813540F0AB405),
    (0x0E329232EA6D0D73, 0x8787878787878787, 0x0000000000000000),
    (0x0101010101010101, 0x0000000000000000, 0x8CA64DE9C1B123A7),
    (0x8001010101010101, 0x0000000000000000, 0x95A8D72813DAA94D),
    (0x7CA110454A1A6E57, 0x01A1D6D039776742, 0x690F5B0D9A26939B),
    (0x0131D9619DC1376E, 0x5CD54CA83DEF57DA, 0x7A389D10354BD271),
]
TDES_KATS = [  # verify.cpp:25-33
    ("0123456789ABCDEF23456789ABCDEF01456789ABCDEF0123", "5468652071756663", "A826FD8CE53B855F"),
    ("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57", "0123456789ABCDEF", "1A493D768C1B9432"),
    ("0123456789ABCDEF23456789ABCDEF01", "4E6F772069732074", "B7835779EE26ACB7"),
    ("0123456789ABCDEF", "4E6F772069732074", "3FA40E8A984D4815"),
]
WALKTHROUGH = [  # verify.cpp:35-40
    0x1B02EFFC7072, 0x79AED9DBC9E5, 0x55FC8A42CF99, 0x72ADD6DB351D,
    0x7CEC07EB53A8, 0x63A53E507B2F, 0xEC84B7F618BC, 0xF78A3AC13BFB,
    0xE0DBEBEDE781, 0xB1F347BA464F, 0x215FD3DED386, 0x7571F59467E9,
    0x97C5D1FABA41, 0x5F43B7F2E73A, 0xBF918D3D3F0A, 0xCB3D8B0E17F5,
]
# NIST SP 800-67 Rev.1 App. B: 3 blocks, plaintext "The qufck brown fox jump"
SP80067 = ("0123456789ABCDEF23456789ABCDEF01456789ABCDEF0123",
           "5468652071756663" "6B2062726F776E20" "666F78206A756D70")

BENCH_KEY = "133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57"  # bench.cpp:15-16
KEYS = {
    "opt1_bench": BENCH_KEY,
    "opt1_nist": "0123456789ABCDEF23456789ABCDEF01456789ABCDEF0123",
    "opt2": "0123456789ABCDEF23456789ABCDEF01",
    "opt3": "0123456789ABCDEF",
}
SIZES = [0, 1, 2, 31, 32, 33, 63, 64, 1023, 1024, 1025, 8195, 131071, 131072]


def main() -> None:
    r = ctypes.CDLL(REF)
    U64 = ctypes.c_uint64
    r.ref_ecb.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(U64),
                          ctypes.c_int, ctypes.c_int, ctypes.c_uint, ctypes.c_size_t, ctypes.c_size_t]
    r.ref_make_payload.argtypes = [ctypes.c_void_p, U64, U64]

    def sched(hexkey):
        s = (U64 * 48)()
        opt = ctypes.c_int()
        assert r.ref_schedule_hex(hexkey.encode(), s, ctypes.byref(opt)) == 0
        return s, opt.value

    def ecb(s, data: bytes, dec: int, backend: int = 1) -> bytes:
        x = np.frombuffer(data, dtype=np.uint8).copy()
        y = np.zeros_like(x)
        rc = r.ref_ecb(x.ctypes.data, y.ctypes.data, x.nbytes, s, dec, backend, 0, 0, 0)
        assert rc == 0
        return y.tobytes()

    def payload(nbytes, seed):
        buf = np.zeros(max(nbytes, 1), dtype=np.uint8)
        r.ref_make_payload(buf.ctypes.data, nbytes, seed)
        return buf[:nbytes].tobytes()

    out = {"generator": "tests/golden/make_golden.py (reference library oracle/_ref)", "kats": {}, "batches": []}
    des = []
    for key, pt, ct in DES_KATS:  # DES via option-3 key (EDE collapses to DES)
        s, _ = sched(f"{key:016X}")
        got_ct = ecb(s, pt.to_bytes(8, "big"), 0, 0)
        assert got_ct == ct.to_bytes(8, "big"), "reference disagrees with its own DES KAT"
        des.append({"key": f"{key:016X}", "plaintext": f"{pt:016X}", "ciphertext": f"{ct:016X}"})
    out["kats"]["des"] = des
    tdes = []
    for key, pt, ct in TDES_KATS:
        s, opt = sched(key)
        assert ecb(s, bytes.fromhex(pt), 0, 0).hex().upper() == ct
        tdes.append({"key": key, "option": opt, "plaintext": pt, "ciphertext": ct})
    s, _ = sched(SP80067[0])
    ct3 = ecb(s, bytes.fromhex(SP80067[1]), 0, 0).hex().upper()
    tdes.append({"key": SP80067[0], "option": 1, "plaintext": SP80067[1], "ciphertext": ct3,
                 "source": "NIST SP 800-67 App. B (3 blocks), ciphertext from the reference"})
    out["kats"]["tdes"] = tdes
    s, _ = sched("133457799BBCDFF1")
    out["walkthrough"] = {"key": "133457799BBCDFF1", "subkeys": [f"{v:012X}" for v in list(s)[:16]]}
    assert list(s)[:16] == WALKTHROUGH
    sched_out = {}
    for name, key in KEYS.items():
        s, opt = sched(key)
        sched_out[name] = {"key": key, "option": opt, "sub48": [f"{v:012X}" for v in s]}
    out["schedules"] = sched_out
    for name, key in KEYS.items():
        s, _ = sched(key)
        for n in SIZES:
            pt = payload(8 * n, 0x3DE5C0DE)
            for dec in (0, 1):
                ct = ecb(s, pt, dec, 1)
                rec = {"key": name, "nblocks": n, "decrypt": dec, "payload_seed": 0x3DE5C0DE,
                       "sha256": hashlib.sha256(ct).hexdigest()}
                if n <= 64:
                    rec["output_hex"] = ct.hex()
                elif n:
                    rec["first"] = ct[:8].hex()
                    rec["last"] = ct[-8:].hex()
                out["batches"].append(rec)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(f"wrote {path}: {len(out['batches'])} batch vectors; SP800-67 3-block ct = {ct3}", file=sys.stderr)


if __name__ == "__main__":
    main()
