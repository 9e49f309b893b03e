"""CPU checks of the kernel design, before any GPU time:
  * every generated S-box circuit, exhaustively (64 inputs x 4 outputs);
  * the committed generated headers are what gen_bitslice.py produces;
  * the bitsliced core (t3des_core.cuh: transposes, IP/FP renaming, 48
    rounds, whitening tables) compiled for the host, against the oracle;
  * the SP-table kernel's index/IP/FP arithmetic, restated in Python.
"""
import ctypes
import os
import subprocess
import sys

import numpy as np
import pytest

from tests.oracle_util import ROOT, U64, bs_host

CSRC = os.path.join(ROOT, "paper_1305_4376_b200", "csrc")
sys.path.insert(0, CSRC)
import gen_bitslice as G  # noqa: E402

KEYS = ["133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57", "0123456789ABCDEF23456789ABCDEF01456789ABCDEF0123",
        "0123456789ABCDEF23456789ABCDEF01", "0123456789ABCDEF"]


@pytest.mark.parametrize("box", range(8))
def test_sbox_circuit_exhaustive(box):
    gates, outs = G.load_circuit(box)
    G.verify_circuit(box, gates, outs)  # raises on any mismatch
    assert len(gates) <= 40


def test_generated_headers_up_to_date(tmp_path):
    with open(os.path.join(CSRC, "generated", "bitslice_rounds.cuh")) as f:
        before = f.read()
    subprocess.check_call([sys.executable, os.path.join(CSRC, "gen_bitslice.py")], stderr=subprocess.DEVNULL)
    with open(os.path.join(CSRC, "generated", "bitslice_rounds.cuh")) as f:
        assert f.read() == before, "generated/bitslice_rounds.cuh is stale: rerun gen_bitslice.py"


@pytest.mark.parametrize("keyhex", KEYS)
def test_bitsliced_core_host_build(oracle, keyhex):
    lib = bs_host()
    s = oracle.schedule_hex(keyhex)
    x = oracle.payload(8 * 32 * 40)
    for d in (0, 1):
        y = np.empty_like(x)
        assert lib.bs_host_ecb(x.ctypes.data, y.ctypes.data, 32 * 40, s, d) == 0
        assert np.array_equal(y, oracle.ecb(x, s, d)), (keyhex, d)


def test_bitsliced_core_random_keys(oracle):
    # fast == reference on random 3-key cases (test_tdes.cpp:110-122)
    lib = bs_host()
    rng = np.random.default_rng(5)
    for _ in range(40):
        k = rng.integers(0, 2**63, 3, dtype=np.uint64)
        s = (U64 * 48)()
        oracle.lib.oracle_triple_schedule(int(k[0]), int(k[1]), int(k[2]), s)
        x = rng.integers(0, 256, 8 * 64, dtype=np.uint8)
        for d in (0, 1):
            y = np.empty_like(x)
            lib.bs_host_ecb(x.ctypes.data, y.ctypes.data, 64, s, d)
            assert np.array_equal(y, oracle.ecb(x, s, d, route=0))


def test_whitening_table_primary_slots(oracle):
    """Every R-role half must arrive at each round whitened with that round's
    primary-slot key bits (the kernel reads primary slots unmodified).
    Re-simulate the kernel's XOR sequence symbolically from the table."""
    lib = bs_host()
    s = oracle.schedule_hex(KEYS[0])
    w = (ctypes.c_uint32 * 8192)()
    nw = lib.bs_host_table(s, 0, w)
    # layout (t3des_core.cuh T3_TAB_*): PRE 64 | 48 rounds x 64 | RW1 32 | RW2 32 | POST 64 | S words 192
    # | t3_cfix constants 2, 1
    stride = 64
    rw1 = 64 + 48 * stride
    rw2, post, ws = rw1 + 32, rw1 + 64, rw1 + 128
    assert nw == ws + 192 + 2
    assert list(w[ws + 192: ws + 194]) == [2, 1]
    w = np.array(w[:nw], dtype=np.uint64)
    for dst, src, n in ((ws, 0, 64), (ws + 64, rw1, 32), (ws + 96, rw2, 32), (ws + 128, post, 64)):
        assert np.array_equal(w[dst:dst + n], w[src:src + n] | 1)  # FMA multipliers S = D | 1
    for t in range(48):
        d = w[64 + stride * t + 32: 64 + stride * t + 48]
        assert np.array_equal(w[64 + stride * t + 48: 64 + stride * t + 64], d | 1)
    w = w & 1
    seq = [s[i] for i in range(16)] + [s[31 - i] for i in range(16)] + [s[32 + i] for i in range(16)]
    prim = G.e_slot_maps()[0]

    def kp(t):
        return np.array([(seq[t] >> (47 - prim[q])) & 1 for q in range(32)], dtype=np.uint64)

    wh = [w[0:32].copy(), w[32:64].copy()]  # whitening carried by A, B
    for t in range(48):
        p, loc = divmod(t, 16)
        lh = (loc % 2) if p != 1 else 1 - (loc % 2)
        rh = 1 - lh
        if t == 16:
            wh[0] ^= w[rw1: rw1 + 32]
        if t == 32:
            wh[1] ^= w[rw2: rw2 + 32]
        assert np.array_equal(wh[rh], kp(t)), t
        wh[lh] ^= w[64 + stride * t: 64 + stride * t + 32]
    wh[0] ^= w[post: post + 32]
    wh[1] ^= w[post + 32: post + 64]
    assert not wh[0].any() and not wh[1].any()


# ---- SP-table kernel arithmetic (kernels.cuh t3_sp_kernel) restated ------
M32 = 0xFFFFFFFF


def _dswap(a, b, s, m):
    w = ((a >> s) ^ b) & m
    return a ^ ((w << s) & M32), b ^ w


def _rotr(x, s):
    s &= 31
    return ((x >> s) | (x << (32 - s))) & M32


def test_sp_kernel_arithmetic(oracle):
    sp = [[0] * 64 for _ in range(8)]
    for i in range(8):
        for x in range(64):
            v = G.sbox_value(i, x) << (28 - 4 * i)
            sp[i][x] = sum(((v >> (32 - G.P[p])) & 1) << (31 - p) for p in range(32))
    s = oracle.schedule_hex(KEYS[0])
    enc = [s[i] for i in range(16)] + [s[31 - i] for i in range(16)] + [s[32 + i] for i in range(16)]
    blocks = oracle.payload(8 * 16)
    expect = oracle.ecb(blocks, s, 0)
    for b in range(16):
        v = int.from_bytes(blocks[8 * b: 8 * b + 8].tobytes(), "big")
        x, y = v >> 32, v & M32
        x, y = _dswap(x, y, 4, 0x0F0F0F0F)
        x, y = _dswap(x, y, 16, 0x0000FFFF)
        y, x = _dswap(y, x, 2, 0x33333333)
        y, x = _dswap(y, x, 8, 0x00FF00FF)
        x, y = _dswap(x, y, 1, 0x55555555)

        def f(r, k48):
            out = 0
            for i in range(8):
                kk = ((k48 >> (42 - 6 * i)) & 0x3F) << 7
                off = (_rotr(r, 20 - 4 * i) ^ kk) & 0x1F80
                out |= sp[i][off >> 7]
            return out

        for t in range(0, 16, 2):
            x ^= f(y, enc[t]); y ^= f(x, enc[t + 1])
        for t in range(16, 32, 2):
            y ^= f(x, enc[t]); x ^= f(y, enc[t + 1])
        for t in range(32, 48, 2):
            x ^= f(y, enc[t]); y ^= f(x, enc[t + 1])
        hi, lo = y, x
        hi, lo = _dswap(hi, lo, 1, 0x55555555)
        lo, hi = _dswap(lo, hi, 8, 0x00FF00FF)
        lo, hi = _dswap(lo, hi, 2, 0x33333333)
        hi, lo = _dswap(hi, lo, 16, 0x0000FFFF)
        hi, lo = _dswap(hi, lo, 4, 0x0F0F0F0F)
        assert ((hi << 32) | lo).to_bytes(8, "big") == expect[8 * b: 8 * b + 8].tobytes()


def test_ip_delta_swaps_match_fips(oracle):
    rng = np.random.default_rng(2)
    for _ in range(200):
        v = int(rng.integers(0, 2**63, dtype=np.uint64)) * 2 + 1
        x, y = v >> 32, v & M32
        x, y = _dswap(x, y, 4, 0x0F0F0F0F)
        x, y = _dswap(x, y, 16, 0x0000FFFF)
        y, x = _dswap(y, x, 2, 0x33333333)
        y, x = _dswap(y, x, 8, 0x00FF00FF)
        x, y = _dswap(x, y, 1, 0x55555555)
        assert (x << 32) | y == oracle.lib.oracle_permute(v, 64, 0)


@pytest.mark.parametrize("keyhex,expect_rounds", [
    ("0123456789ABCDEF", 16),                                           # option 3
    ("0123456789ABCDEF0123456789ABCDEF456789ABCDEF0123", 16),           # K1 = K2
    ("0123456789ABCDEF23456789ABCDEF0123456789ABCDEF01", 16),           # K2 = K3
    ("0023456789ABCDEF0123456789ABCDEF456789ABCDEF0123", 16),           # K1, K2 differ only in parity
    ("0123456789ABCDEF23456789ABCDEF01", 48),                           # option 2: no collapse
    (KEYS[0], 48),
])
def test_collapsed_single_des_path(oracle, keyhex, expect_rounds):
    """K1 = K2 or K2 = K3 (schedules equal): EDE = single DES, run as 16
    bitsliced rounds; bit-exact with the full 48-round oracle."""
    lib = bs_host()
    s = oracle.schedule_hex(keyhex)
    x = oracle.payload(8 * 32 * 12)
    for d in (0, 1):
        y = np.empty_like(x)
        assert lib.bs_host_ecb_collapse(x.ctypes.data, y.ctypes.data, 32 * 12, s, d) == expect_rounds
        assert np.array_equal(y, oracle.ecb(x, s, d, route=0)), (keyhex, d)
