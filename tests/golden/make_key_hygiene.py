#!/usr/bin/env python3
"""Generate tests/golden/key_hygiene.json from the UNMODIFIED reference
library (oracle/_ref/libt3des_ref.so, built by `make -C oracle` where
/root/reference exists): has_odd_parity / is_weak_key / is_semiweak_key /
normalize_parity (des.cpp:159-207) and to_hex(parse_hex_key(...))
(tdes.cpp:32-81) on

  - keys whose PC-1 registers C, D are each constant, 2-periodic or
    4-periodic (the weak, semi-weak and "possibly weak" families), built
    by inverting PC-1, with random parity bits;
  - random keys;
  - hex keys of all three keying options, in upper and lower case.

The JSON is committed; tests/test_capi_host.py reads only the JSON (the GPU
box has no /root/reference) and compares the engine library with it.
"""
from __future__ import annotations

import ctypes
import json
import os
import random

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF = os.path.join(ROOT, "oracle", "_ref", "libt3des_ref.so")

# FIPS 46-3 PC-1 (1-based key bit positions, MSB = bit 1): C = first 28, D = last 28
PC1 = [57, 49, 41, 33, 25, 17, 9, 1, 58, 50, 42, 34, 26, 18, 10, 2, 59, 51, 43, 35, 27, 19, 11, 3, 60, 52, 44, 36,
       63, 55, 47, 39, 31, 23, 15, 7, 62, 54, 46, 38, 30, 22, 14, 6, 61, 53, 45, 37, 29, 21, 13, 5, 28, 20, 12, 4]

PATTERNS = [0x0000000, 0xFFFFFFF, 0x5555555, 0xAAAAAAA,  # constant, 2-periodic
            0x1111111, 0x2222222, 0x4444444, 0x8888888, 0x3333333, 0x6666666, 0xCCCCCCC, 0x9999999,
            0x7777777, 0xBBBBBBB, 0xDDDDDDD, 0xEEEEEEE]  # 4-periodic


def key_from_registers(c: int, d: int, parity: int) -> int:
    cd = (c << 28) | d
    key = 0
    for i, pos in enumerate(PC1):
        if (cd >> (55 - i)) & 1:
            key |= 1 << (64 - pos)
    return key | (parity & 0x0101010101010101)


def main() -> None:
    ref = ctypes.CDLL(REF)
    ref.ref_key_flags.argtypes = [ctypes.c_uint64]
    ref.ref_key_flags.restype = ctypes.c_int
    ref.ref_normalize_parity.argtypes = [ctypes.c_uint64]
    ref.ref_normalize_parity.restype = ctypes.c_uint64
    ref.ref_to_hex.argtypes = [ctypes.c_char_p, ctypes.c_char_p]
    ref.ref_to_hex.restype = ctypes.c_int
    rng = random.Random(0x7E57)
    keys = []
    for c in PATTERNS:
        for d in PATTERNS:
            for _ in range(3):
                keys.append(key_from_registers(c, d, rng.getrandbits(64)))
    keys += [rng.getrandbits(64) for _ in range(500)]
    keys += [0x0101010101010101, 0xFEFEFEFEFEFEFEFE, 0x133457799BBCDFF1, 0, 0xFFFFFFFFFFFFFFFF]
    cases = [[f"{k:016X}", ref.ref_key_flags(k), f"{ref.ref_normalize_parity(k):016X}"] for k in keys]
    hexes = []
    for n in (16, 32, 48):
        for _ in range(4):
            h = "".join(rng.choice("0123456789abcdefABCDEF") for _ in range(n))
            buf = ctypes.create_string_buffer(64)
            assert ref.ref_to_hex(h.encode(), buf) == 0
            hexes.append({"in": h, "to_hex": buf.value.decode()})
    out = {"source": "reference des.cpp:159-207 / tdes.cpp:32-81 via oracle/_ref (tests/golden/make_key_hygiene.py)",
           "keys_format": "[key, flags, normalize_parity(key)]; flags bit 0 has_odd_parity, bit 1 is_weak_key, "
                          "bit 2 is_semiweak_key",
           "keys": cases, "to_hex": hexes}
    with open(os.path.join(ROOT, "tests", "golden", "key_hygiene.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))
    weak = sum(1 for c in cases if c[1] & 2)
    semi = sum(1 for c in cases if c[1] & 4)
    print(f"{len(cases)} keys ({weak} weak, {semi} semi-weak), {len(hexes)} hex keys")


if __name__ == "__main__":
    main()
