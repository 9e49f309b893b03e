"""Pin the C oracle (oracle/des_oracle.c) before trusting it: the
reference's own known-answer vectors, golden batches produced by the
reference library, and (when oracle/_ref is built) the reference itself."""
import ctypes
import hashlib

import numpy as np
import pytest

from tests.oracle_util import U64, sub48_from_hex_list


def test_des_kats(oracle, golden):
    # reference verify.cpp:15-22, test_des.cpp:47-54
    for kat in golden["kats"]["des"]:
        k, p, c = (int(kat[x], 16) for x in ("key", "plaintext", "ciphertext"))
        assert oracle.lib.oracle_des_block(p, k, 0) == c
        assert oracle.lib.oracle_des_block(c, k, 1) == p


@pytest.mark.parametrize("route", [0, 1])
def test_tdes_kats_both_routes(oracle, golden, route):
    # reference verify.cpp:25-33 through the plain (0) and fused SP (1) routes
    # (test_tdes.cpp:68-79), plus the 3-block NIST SP 800-67 example.
    for kat in golden["kats"]["tdes"]:
        s = oracle.schedule_hex(kat["key"])
        pt = bytes.fromhex(kat["plaintext"])
        ct = oracle.ecb(pt, s, 0, route=route)
        assert ct.tobytes().hex().upper() == kat["ciphertext"]
        assert oracle.ecb(ct, s, 1, route=route).tobytes() == pt


def test_walkthrough_subkeys(oracle, golden):
    ks = (U64 * 16)()
    oracle.lib.oracle_key_schedule(int(golden["walkthrough"]["key"], 16), ks)
    assert [f"{v:012X}" for v in ks] == golden["walkthrough"]["subkeys"]


def test_schedules_match_reference(oracle, golden):
    for name, rec in golden["schedules"].items():
        assert list(oracle.schedule_hex(rec["key"])) == [int(v, 16) for v in rec["sub48"]], name


def test_golden_batches(oracle, golden):
    # make_payload restatement (mt19937_64) + fused route vs the reference's
    # Threaded backend outputs, every keying option, edge block counts.
    for rec in golden["batches"]:
        s = sub48_from_hex_list(golden["schedules"][rec["key"]]["sub48"])
        pt = oracle.payload(8 * rec["nblocks"], rec["payload_seed"])
        out = oracle.ecb(pt, s, rec["decrypt"])
        assert hashlib.sha256(out.tobytes()).hexdigest() == rec["sha256"], rec


def test_plain_route_equals_fused_route(oracle):
    rng = np.random.default_rng(7)
    for _ in range(20):
        keys = rng.integers(0, 2**63, 3, dtype=np.uint64)
        s = (U64 * 48)()
        oracle.lib.oracle_triple_schedule(int(keys[0]), int(keys[1]), int(keys[2]), s)
        x = rng.integers(0, 256, 8 * 64, dtype=np.uint8)
        for d in (0, 1):
            assert np.array_equal(oracle.ecb(x, s, d, route=0), oracle.ecb(x, s, d, route=1))


def test_option3_is_single_des(oracle):
    # acceptance.cpp:104-116
    rng = np.random.default_rng(3)
    for _ in range(200):
        k = int(rng.integers(0, 2**63, dtype=np.uint64))
        p = int(rng.integers(0, 2**63, dtype=np.uint64))
        s = oracle.schedule_hex(f"{k:016X}")
        assert oracle.lib.oracle_tdes_block(p, s, 0) == oracle.lib.oracle_des_block(p, k, 0)


def test_error_codes(oracle):
    s = oracle.schedule_hex("0123456789ABCDEF")
    x = np.zeros(16, dtype=np.uint8)
    assert oracle.lib.oracle_ecb(x.ctypes.data, x.ctypes.data, 12, s, 0, 1, 1) == 1
    assert oracle.lib.oracle_ecb(x.ctypes.data, x.ctypes.data + 8, 8 + 8, s, 0, 1, 1) == 3
    assert oracle.lib.oracle_ecb(x.ctypes.data, x.ctypes.data, 16, s, 0, 1, 1) == 0  # in place ok


def test_splitmix_payload(oracle):
    a = oracle.splitmix(1000, 50, 0xABCDEF)
    for i in (0, 17, 49):
        v = oracle.lib.oracle_splitmix_block(0xABCDEF, 1000 + i)
        assert a[8 * i: 8 * i + 8].tobytes() == int(v).to_bytes(8, "big")


@pytest.mark.skipif("not __import__('os').path.exists(__import__('tests.oracle_util', fromlist=['REF_SO']).REF_SO)")
def test_oracle_vs_reference_library(oracle):
    rng = np.random.default_rng(11)
    for keyhex in ("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57", "0123456789ABCDEF23456789ABCDEF01",
                   "0123456789ABCDEF"):
        s = oracle.schedule_hex(keyhex)
        s_ref = (U64 * 48)()
        opt = ctypes.c_int()
        assert oracle.ref.ref_schedule_hex(keyhex.encode(), s_ref, ctypes.byref(opt)) == 0
        assert list(s) == list(s_ref)
        x = rng.integers(0, 256, 8 * 8195, dtype=np.uint8)
        for d in (0, 1):
            assert np.array_equal(oracle.ecb(x, s, d), oracle.ref_ecb(x, s_ref, d))
    p1 = oracle.payload(4096)
    p2 = np.empty(4096, dtype=np.uint8)
    oracle.ref.ref_make_payload(p2.ctypes.data, 4096, 0x3DE5C0DE)
    assert np.array_equal(p1, p2)
