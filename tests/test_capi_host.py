"""C-ABI library checks that need no GPU: it loads, exports every symbol
include/t3des_cu.h declares, host keying matches the reference, argument
errors are reported as the reference reports them, and — without a
device — the cipher fails loudly instead of falling back to a CPU."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1305_4376_b200 as t3
from paper_1305_4376_b200 import _native as N
from tests.oracle_util import ROOT

HEADER = os.path.join(ROOT, "include", "t3des_cu.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(t3des_cu_[a-z_0-9]+)\s*\(", txt)))


def test_exports_every_declared_symbol(engine_lib):
    syms = declared_symbols()
    assert len(syms) >= 15
    out = subprocess.check_output(["nm", "-D", "--defined-only", N.LIB_PATH], text=True)
    exported = set(re.findall(r" T (t3des_cu_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    assert set(syms) == set(N.SIGNATURES), "ctypes signature table out of sync with the header"


def test_library_is_sm100a_only(engine_lib):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", N.LIB_PATH], text=True)
    assert "sm_100a" in out
    assert re.search(r"sm_(?!100a)\d+", out) is None


def test_parse_hex_key_options(engine_lib):
    k = t3.parse_hex_key("0123456789ABCDEF23456789ABCDEF01456789ABCDEF0123")
    assert k.option is t3.KeyingOption.Option1 and k.k3.raw == 0x456789ABCDEF0123
    k = t3.parse_hex_key("0123456789abcdef23456789ABCDEF01")
    assert k.option is t3.KeyingOption.Option2 and k.k3 == k.k1
    k = t3.parse_hex_key("0123456789ABCDEF")
    assert k.option is t3.KeyingOption.Option3 and k.k1 == k.k2 == k.k3
    assert t3.to_hex(t3.parse_hex_key("0123456789abcdef23456789ABCDEF01")) == "0123456789ABCDEF23456789ABCDEF01"
    for bad in ("", "0123", "0123456789ABCDEF0", "0123456789ABCDEG", "z" * 48):
        with pytest.raises(t3.KeyFormatError):
            t3.parse_hex_key(bad)


def test_schedules_match_golden(engine_lib, golden):
    for rec in golden["schedules"].values():
        ts = t3.triple_schedule(t3.parse_hex_key(rec["key"]))
        got = [f"{v:012X}" for v in ts.pass1 + ts.pass2 + ts.pass3]
        assert got == rec["sub48"]
    ks = t3.key_schedule(int(golden["walkthrough"]["key"], 16))
    assert [f"{v:012X}" for v in ks] == golden["walkthrough"]["subkeys"]
    # parity bits are ignored by PC-1 (test_des.cpp:29-40)
    assert t3.key_schedule(0x133457799BBCDFF1) == t3.key_schedule(0x133457799BBCDFF1 ^ 0x0101010101010101)


def test_plan_dispatch_matches_reference_semantics():
    cfg = t3.DispatchConfig(chunk_blocks=131072)
    assert t3.plan_dispatch(0, cfg) == []
    assert [(s.offset, s.length) for s in t3.plan_dispatch(300000, cfg)] == [
        (0, 131072), (131072, 131072), (262144, 37856)]
    for chunk in (1, 7, 64):
        cfg.chunk_blocks = chunk
        for total in range(0, 500, 37):
            spans = t3.plan_dispatch(total, cfg)
            assert sum(s.length for s in spans) == total
            assert all(s.length == chunk for s in spans[:-1])


def test_argument_errors_before_device(engine_lib):
    ts = t3.triple_schedule(t3.parse_hex_key("0123456789ABCDEF"))
    with pytest.raises(t3.InputLengthError):
        t3.encrypt_batch(b"\0" * 12, bytearray(12), ts)
    with pytest.raises(t3.InputLengthError):
        t3.encrypt_batch(b"\0" * 16, bytearray(24), ts)
    with pytest.raises(NotImplementedError):
        t3.encrypt_batch(b"\0" * 16, bytearray(16), ts, t3.DispatchConfig(backend=t3.Backend.Threaded))
    out = bytearray(16)
    t3.encrypt_batch(b"\1" * 16, out, ts, t3.DispatchConfig(backend=t3.Backend.NoOpCopy))
    assert bytes(out) == b"\1" * 16
    t3.encrypt_batch(b"", bytearray(), ts)  # N = 0 is a no-op


def test_c_abi_status_codes(engine_lib):
    L = engine_lib
    assert L.t3des_cu_version() >= 10000
    for code in range(0, 8):
        assert L.t3des_cu_strerror(code)
    n = ctypes.c_int(-1)
    assert L.t3des_cu_device_count(ctypes.byref(n)) == 0
    keys = (ctypes.c_uint64 * 3)()
    assert L.t3des_cu_parse_hex_key(b"00", 2, keys, None) == N.ERR_KEY
    assert L.t3des_cu_ecb_device(None, 0, None, None, 0, None) == N.ERR_ARG
    sub = (ctypes.c_uint64 * 48)()
    buf = ctypes.create_string_buffer(24)
    assert L.t3des_cu_ecb_workers(2, 0, None, 0, buf, buf, 16) == N.ERR_ARG
    assert L.t3des_cu_ecb_workers(2, 0, sub, 2, buf, buf, 16) == N.ERR_ARG
    assert L.t3des_cu_ecb_workers(2, 0, sub, 0, buf, buf, 12) == N.ERR_LENGTH
    assert L.t3des_cu_ecb_workers(2, 0, sub, 0, ctypes.addressof(buf), ctypes.addressof(buf) + 8, 16) == N.ERR_OVERLAP


@pytest.mark.skipif("__import__('torch').cuda.is_available()")
def test_no_device_is_an_error_not_a_fallback(engine_lib):
    h = ctypes.c_void_p()
    assert engine_lib.t3des_cu_create(0, ctypes.byref(h)) == N.ERR_NO_DEVICE
    ts = t3.triple_schedule(t3.parse_hex_key("0123456789ABCDEF"))
    with pytest.raises(t3.CudaError):
        t3.encrypt_batch(b"\0" * 64, bytearray(64), ts)
    with pytest.raises(t3.CudaError):  # the workers axis too
        t3.encrypt_batch(b"\0" * 64, bytearray(64), ts, t3.DispatchConfig(workers=2))


def test_cpp_api_compiles_and_reports_errors(engine_lib, tmp_path):
    """The C++ mirror of the reference API (include/t3des_b200/t3des.hpp)
    builds against the library; keying and argument errors work host-side."""
    src = tmp_path / "t.cpp"
    src.write_text(r'''
#include <cstdio>
#include <vector>
#include "t3des_b200/t3des.hpp"
using namespace t3des;
int main() {
    auto k = parse_hex_key("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57");
    auto ts = triple_schedule(k);
    if (ts.pass1[0] != key_schedule(k.k1)[0]) return 2;
    if (key_schedule(DesKey{0x133457799BBCDFF1ull})[0] != 0x1B02EFFC7072ull) return 3;
    try { parse_hex_key("12"); return 4; } catch (const KeyFormatError&) {}
    std::vector<std::uint8_t> in(12), out(12);
    try { encrypt_batch(in, out, ts, DispatchConfig{}); return 5; } catch (const InputLengthError&) {}
    std::vector<std::uint8_t> a(16), b(16);
    try { encrypt_batch(a, b, ts, DispatchConfig{.backend = Backend::Threaded}); return 6; }
    catch (const std::invalid_argument&) {}
    std::uint8_t blk[8] = {1,2,3,4,5,6,7,8};
    if (load_block(std::span<const std::uint8_t, 8>(blk, 8)) != 0x0102030405060708ull) return 7;
    std::puts("ok");
    return 0;
}
''')
    exe = tmp_path / "t"
    subprocess.check_call(["/usr/bin/g++", "-std=c++20", "-I" + os.path.join(ROOT, "include"), str(src),
                           N.LIB_PATH, "-Wl,-rpath," + os.path.dirname(N.LIB_PATH), "-o", str(exe)])
    assert subprocess.run([str(exe)], capture_output=True, text=True).stdout.strip() == "ok"


def test_pipeline_and_launch_argument_checks(engine_lib):
    L = engine_lib
    assert L.t3des_cu_set_pipeline(None, 1 << 20, 3) == N.ERR_ARG
    assert L.t3des_cu_set_launch(None, 0, 0) == N.ERR_ARG
    assert L.t3des_cu_set_variant(None, 0) == N.ERR_ARG
    first, count = ctypes.c_uint64(), ctypes.c_uint64()
    assert L.t3des_cu_shard_range(100, 0, 0, ctypes.byref(first), ctypes.byref(count)) == N.ERR_ARG
    assert L.t3des_cu_shard_range(100, 2, 1, ctypes.byref(first), ctypes.byref(count)) == 0
    assert (first.value, count.value) == (0, 100)  # 100 blocks < one tile: all in the last shard
    rep = N.StreamReportC()
    assert L.t3des_cu_stream_fd(None, 0, 0, 1, 16, 0, ctypes.byref(rep)) == N.ERR_ARG
    assert L.t3des_cu_ecb_multi(None, 0, None, 0, None, None, 0) == N.ERR_ARG
    devs = (ctypes.c_int * 1)(0)
    sub = (ctypes.c_uint64 * 48)()
    assert L.t3des_cu_ecb_multi(devs, 1, sub, 0, None, None, 12) == N.ERR_LENGTH
    assert L.t3des_cu_ecb_multi_device(devs, 1, sub, 0, 0, None, None, 12, 0) == N.ERR_LENGTH


def _key_hygiene_golden():
    import json

    with open(os.path.join(ROOT, "tests", "golden", "key_hygiene.json")) as f:
        return json.load(f)


def test_key_hygiene_matches_reference_golden(engine_lib):
    """has_odd_parity / is_weak_key / is_semiweak_key / normalize_parity
    (reference des.cpp:159-207) against the reference's own answers
    (tests/golden/make_key_hygiene.py): the weak, semi-weak and 4-periodic
    "possibly weak" register families with random parity bits, random keys."""
    g = _key_hygiene_golden()
    assert len(g["keys"]) > 1000
    for hexkey, flags, normalized in g["keys"]:
        k = int(hexkey, 16)
        assert engine_lib.t3des_cu_des_key_flags(k) == flags, hexkey
        assert engine_lib.t3des_cu_normalize_parity(k) == int(normalized, 16), hexkey
        assert t3.has_odd_parity(k) == bool(flags & 1)
        assert t3.is_weak_key(t3.DesKey(k)) == bool(flags & 2)
        assert t3.is_semiweak_key(k) == bool(flags & 4)
        assert t3.normalize_parity(k).raw == int(normalized, 16)
        assert t3.has_odd_parity(t3.normalize_parity(k))
    for case in g["to_hex"]:
        assert t3.to_hex(t3.parse_hex_key(case["in"])) == case["to_hex"]


def test_key_hygiene_matches_reference_library(engine_lib):
    """The same against the reference library itself on fresh random keys
    (skipped where oracle/_ref was not built)."""
    from tests.oracle_util import REF_SO

    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (no /root/reference here)")
    ref = ctypes.CDLL(REF_SO)
    ref.ref_key_flags.argtypes = [ctypes.c_uint64]
    ref.ref_key_flags.restype = ctypes.c_int
    ref.ref_normalize_parity.argtypes = [ctypes.c_uint64]
    ref.ref_normalize_parity.restype = ctypes.c_uint64
    rng = np.random.default_rng(0xB200)
    keys = [int(x) for x in rng.integers(0, 2**63, size=20000, dtype=np.uint64)]
    keys += [k | (1 << 63) for k in keys[:100]]
    for k in keys:
        assert engine_lib.t3des_cu_des_key_flags(k) == ref.ref_key_flags(k), hex(k)
        assert engine_lib.t3des_cu_normalize_parity(k) == ref.ref_normalize_parity(k), hex(k)


def test_cpp_api_reference_surface(engine_lib, tmp_path):
    """The rest of the reference's host API in the C++ mirror: to_hex,
    ParityError, the key hygiene helpers, resolve_workers and the KAT
    accessors compile, link and answer like the reference (no device)."""
    g = _key_hygiene_golden()
    src = tmp_path / "surface.cpp"
    src.write_text(r'''
#include <cstdio>
#include <string>
#include "t3des_b200/t3des.hpp"
using namespace t3des;
int main(int argc, char** argv) {
    if (to_hex(parse_hex_key(argv[1])) != argv[2]) return 2;
    const DesKey k{std::stoull(argv[3], nullptr, 16)};
    const int flags = (has_odd_parity(k) ? 1 : 0) | (is_weak_key(k) ? 2 : 0) | (is_semiweak_key(k) ? 4 : 0);
    if (flags != std::atoi(argv[4])) return 3;
    if (normalize_parity(k).raw != std::stoull(argv[5], nullptr, 16)) return 4;
    try { throw ParityError("x"); } catch (const std::runtime_error&) {}
    DispatchConfig cfg;
    if (resolve_workers(cfg) != 1) return 5;
    cfg.workers = 3;
    if (resolve_workers(cfg) != 3) return 6;
    if (des_kats().size() != 6 || tdes_kats().size() != 4 || walkthrough_subkeys().size() != 16) return 7;
    const auto ks = key_schedule(DesKey{kWalkthroughKey});
    for (int i = 0; i < 16; ++i) if (ks[i] != walkthrough_subkeys()[i]) return 8;
    std::puts("ok");
    return 0;
}
''')
    exe = tmp_path / "surface"
    subprocess.check_call(["/usr/bin/g++", "-std=c++20", "-I" + os.path.join(ROOT, "include"), str(src),
                           N.LIB_PATH, "-Wl,-rpath," + os.path.dirname(N.LIB_PATH), "-o", str(exe)])
    weak = next(c for c in g["keys"] if c[1] & 2)
    semi = next(c for c in g["keys"] if c[1] & 4)
    plain = next(c for c in g["keys"] if c[1] == 0)
    for case, key in zip(g["to_hex"][::4], (weak, semi, plain)):
        p = subprocess.run([str(exe), case["in"], case["to_hex"], key[0], str(key[1]), key[2]],
                           capture_output=True, text=True)
        assert p.returncode == 0 and p.stdout.strip() == "ok", (p.returncode, case, key)
