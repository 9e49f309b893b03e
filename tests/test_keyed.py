"""SURVEY §8f-4, key-specialised kernels: T3DES_CU_VARIANT_KEYED.

The round keys of one execution sequence are folded into the LOP3
immediates (generated/keyed_rounds.cuh, t3_keyed_round<K>); NVRTC compiles
keyed_kernel.cuh for the installed schedule at run time (csrc/keyed.cpp).

CPU (no GPU needed):
  * the same templates compiled by g++ for one key sequence
    (tests/native/keyed_host.cpp) equal the oracle — options 1/2/3 (option 3
    as the collapsed 16-round sequence), both directions, random keys;
  * t3des_cu_keyed_compile builds the sm_100a CUBIN through NVRTC, and its
    SASS has the keyed kernel's shape: no local memory, >= 48 x 186 LOP3,
    the CTA barriers that hold the warps together, TMA bulk copies.
GPU: the engine's keyed variant against the oracle (tile/grid edges, tails,
in place, unaligned spans), against the reference at 64 MiB, and the
module cache across schedule changes.
"""
import os
import random
import subprocess

import numpy as np
import pytest

from tests.oracle_util import ROOT

CSRC = os.path.join(ROOT, "paper_1305_4376_b200", "csrc")
BUILD = os.path.join(ROOT, "tests", "native", "_build", "keyed")
BENCH_KEY = "133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57"
KEYS = {"option1": BENCH_KEY, "option2": "0123456789ABCDEF23456789ABCDEF01", "option3": "0123456789ABCDEF"}


def sub48_of(hexkey: str) -> list[int]:
    import paper_1305_4376_b200 as t3

    return list(t3.triple_schedule(t3.parse_hex_key(hexkey)).sub48())


def exec_sequence(sub: list[int], decrypt: bool) -> list[int]:
    """The round keys in execution order (tdes.cpp:177-185): encrypt = k1
    fwd, k2 rev, k3 fwd; decrypt the reverse.  When k1 = k2 (or k2 = k3) the
    EDE collapses to single DES under k3 (k1): 16 keys."""
    k1, k2, k3 = sub[0:16], sub[16:32], sub[32:48]
    if k1 == k2 or k2 == k3:
        seq = list(k3 if k1 == k2 else k1)
    else:
        seq = k1 + k2[::-1] + k3
    return seq[::-1] if decrypt else seq


def host_keyed(seq: list[int], name: str) -> str:
    os.makedirs(BUILD, exist_ok=True)
    exe = os.path.join(BUILD, name)
    subprocess.check_call(["/usr/bin/g++", "-std=c++17", "-O0", "-I" + CSRC,  # -O0: 2.5 s vs 9 s per key
                           "-DT3K_SEQ=" + ",".join(f"0x{k:012x}ull" for k in seq), f"-DT3K_ROUNDS={len(seq)}",
                           os.path.join(ROOT, "tests", "native", "keyed_host.cpp"), "-o", exe])
    return exe


@pytest.mark.parametrize("direction", [0, 1], ids=["encrypt", "decrypt"])
@pytest.mark.parametrize("which", ["option1", "option2", "option3", "random1", "random2"])
def test_keyed_rounds_on_host_equal_oracle(oracle, which, direction):
    if which.startswith("random"):
        rng = random.Random(which)
        hexkey = "".join(rng.choice("0123456789ABCDEF") for _ in range(48))
    else:
        hexkey = KEYS[which]
    seq = exec_sequence(sub48_of(hexkey), bool(direction))
    assert len(seq) == (16 if which == "option3" else 48)
    exe = host_keyed(seq, f"{which}_{direction}")
    x = oracle.splitmix(0, 32 * 64, 0x4B + direction)
    got = np.frombuffer(subprocess.run([exe], input=x.tobytes(), capture_output=True, check=True).stdout, np.uint8)
    assert np.array_equal(got, oracle.ecb(x, oracle.schedule_hex(hexkey), direction))


def _cubin(lib, hexkey: str, direction: int) -> bytes:
    import ctypes

    sub = (ctypes.c_uint64 * 48)(*sub48_of(hexkey))
    size, secs = ctypes.c_size_t(), ctypes.c_double()
    cap = 16 << 20  # one compile (~1.6 MB CUBIN with line info)
    buf = ctypes.create_string_buffer(cap)
    rc = lib.t3des_cu_keyed_compile(sub, direction, buf, cap, ctypes.byref(size), ctypes.byref(secs))
    if rc == 10:
        pytest.skip("NVRTC not available")
    assert rc == 0 and 0 < size.value <= cap
    return buf.raw[: size.value]


def test_keyed_compile_sm100a_cubin(engine_lib, tmp_path):
    """NVRTC builds the keyed kernel for sm_100a in this container (no GPU):
    no local memory, 48 rounds x 186 S-box gates of LOP3 at least, the CTA
    barriers that keep its warps in one window of the code, TMA copies."""
    import ctypes

    lib = engine_lib
    sub = (ctypes.c_uint64 * 48)(*sub48_of(BENCH_KEY))
    size = ctypes.c_size_t()
    assert lib.t3des_cu_keyed_compile(sub, 2, None, 0, ctypes.byref(size), None) == 4  # bad direction
    assert lib.t3des_cu_keyed_compile(None, 0, None, 0, ctypes.byref(size), None) == 4
    path = tmp_path / "keyed.cubin"
    path.write_bytes(_cubin(lib, BENCH_KEY, 0))
    res = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-res-usage", str(path)], capture_output=True,
                         text=True, check=True).stdout
    assert "t3_keyed_kernel" in res and "LOCAL:0" in res and "STACK:0" in res, res
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", str(path)], capture_output=True, text=True,
                          check=True).stdout
    ops = [ln.split()[1].split(".")[0] for ln in sass.splitlines() if ln.strip().startswith("/*") and "*/" in ln
           and len(ln.split()) > 1]
    assert ops.count("LOP3") >= 48 * 186
    assert ops.count("BAR") >= 2  # the CTA barriers pinned at the pass boundaries
    assert "UBLKCP" in ops


# ---- GPU ----------------------------------------------------------------

torch = None


@pytest.fixture(scope="module")
def keng(engine_lib):
    global torch
    import torch as _torch

    torch = _torch
    import paper_1305_4376_b200 as t3

    e = t3.Engine(0)
    yield e
    e.close()


def _run(e, hexkey, x_dev, direction, out=None, stream=None):
    import paper_1305_4376_b200 as t3
    from paper_1305_4376_b200 import _native as N

    e.set_schedule(t3.triple_schedule(t3.parse_hex_key(hexkey)))
    e.set_variant(N.VARIANT_KEYED)
    e.set_launch(0, 0)
    out = torch.empty_like(x_dev) if out is None else out
    e.ecb_device(direction, x_dev.data_ptr(), out.data_ptr(), x_dev.numel(),
                 stream if stream is not None else torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("direction", [0, 1], ids=["encrypt", "decrypt"])
@pytest.mark.parametrize("which", ["option1", "option2", "option3"])
def test_keyed_variant_vs_oracle(keng, oracle, which, direction):
    """Sizes around the keyed kernel's shapes: no full tile (table-driven
    tail only), one tile, a grid of a few CTAs with idle warps, more tiles
    than one pass of 148 x 16 warps (last pass partly idle) plus a tail on
    the side stream; then in place and an unaligned span."""
    hexkey = KEYS[which]
    s = oracle.schedule_hex(hexkey)
    for n in (1000, 1024, 1024 * 37 + 1, 148 * 16 * 1024 * 2 + 5 * 1024 + 3):
        x = oracle.splitmix(0, n, 0x600D + n + direction)
        want = oracle.ecb(x, s, direction)
        got = _run(keng, hexkey, torch.from_numpy(x).cuda(), direction).cpu().numpy()
        assert np.array_equal(got, want), f"n={n}"
    x = oracle.splitmix(0, 5000, 7)
    xd = torch.from_numpy(x).cuda()
    _run(keng, hexkey, xd, direction, out=xd)  # in place
    assert np.array_equal(xd.cpu().numpy(), oracle.ecb(x, s, direction))
    raw = torch.zeros(8 * 4096 + 16, dtype=torch.uint8, device="cuda")
    x = oracle.splitmix(0, 4096, 9)
    src = raw[8: 8 + x.nbytes]  # 8-byte aligned, not 16: the table-driven kernels
    src.copy_(torch.from_numpy(x))
    got = _run(keng, hexkey, src, direction).cpu().numpy()
    assert np.array_equal(got, oracle.ecb(x, s, direction))


@pytest.mark.gpu
def test_keyed_variant_64mib_vs_reference(keng, oracle):
    """64 MiB (the reference acceptance size, acceptance.cpp:119-152) through
    the keyed kernel, whole output against the reference library."""
    x = oracle.payload(64 << 20, seed=0x3DE5C0DE)
    s = oracle.schedule_hex(BENCH_KEY)
    want = oracle.ref_ecb(x, s, 0, backend=1, workers=0) if oracle.ref is not None else oracle.ecb(x, s, 0)
    got = _run(keng, BENCH_KEY, torch.from_numpy(x).cuda(), 0).cpu().numpy()
    assert np.array_equal(got, want)
    back = _run(keng, BENCH_KEY, torch.from_numpy(got).cuda(), 1).cpu().numpy()
    assert np.array_equal(back, x)


@pytest.mark.gpu
def test_keyed_module_cache_follows_the_schedule(keng, oracle):
    """prepare compiles once per key sequence: a second prepare is a cache
    hit, a new schedule gets its own module (its output is that key's), and
    the first key's module is still cached when the schedule switches back."""
    import paper_1305_4376_b200 as t3

    ka, kb = "0123456789ABCDEFFEDCBA98765432100F1E2D3C4B5A6978", "F0E1D2C3B4A5968778695A4B3C2D1E0F0123456789ABCDEF"
    keng.set_schedule(t3.triple_schedule(t3.parse_hex_key(ka)))
    first = keng.keyed_prepare(0)
    assert keng.keyed_prepare(0) < min(0.05, first / 10)
    x = oracle.splitmix(0, 1024 * 300, 11)
    xd = torch.from_numpy(x).cuda()
    for k in (kb, ka, kb):
        got = _run(keng, k, xd, 0).cpu().numpy()
        assert np.array_equal(got, oracle.ecb(x, oracle.schedule_hex(k), 0)), k
    keng.set_schedule(t3.triple_schedule(t3.parse_hex_key(ka)))
    assert keng.keyed_prepare(0) < 0.05


@pytest.mark.gpu
def test_keyed_variant_in_a_cuda_graph(keng, oracle):
    """Prepared up front, the keyed kernel captures into a CUDA graph (the
    C ABI is stream-ordered) and replays with the right output; the capture
    itself compiles nothing."""
    import paper_1305_4376_b200 as t3
    from paper_1305_4376_b200 import _native as N

    key = "0123456789ABCDEF23456789ABCDEF01456789ABCDEF0123"
    keng.set_schedule(t3.triple_schedule(t3.parse_hex_key(key)))
    keng.set_variant(N.VARIANT_KEYED)
    keng.keyed_prepare(0)
    keng.keyed_prepare(1)
    x = oracle.splitmix(0, 1024 * 500 + 17, 21)
    xd = torch.from_numpy(x).cuda()
    y, z = torch.empty_like(xd), torch.empty_like(xd)
    gs = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=gs):
        keng.ecb_device(0, xd.data_ptr(), y.data_ptr(), xd.numel(), gs.cuda_stream)
        keng.ecb_device(1, y.data_ptr(), z.data_ptr(), xd.numel(), gs.cuda_stream)
    with torch.cuda.stream(gs):
        g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy(), oracle.ecb(x, oracle.schedule_hex(key), 0))
    assert torch.equal(z, xd)


@pytest.mark.gpu
def test_keyed_variant_fuzz(keng, oracle):
    """Random keys of all three keying shapes, random sizes (whole tiles,
    passes with idle warps, tails), random 16-byte-aligned offsets, both
    directions, in place or not — the keyed variant against the oracle."""
    rng = random.Random(0xF4)
    for trial in range(6):
        nhex = rng.choice([16, 32, 48])
        key = "".join(rng.choice("0123456789ABCDEF") for _ in range(nhex))
        s = oracle.schedule_hex(key)
        for _ in range(3):
            n = rng.choice([1024 * rng.randint(1, 3000), rng.randint(1, 4_000_000)])
            direction = rng.randint(0, 1)
            off = 16 * rng.randint(0, 8)  # blocks stay 16-byte aligned: the keyed kernel runs
            x = oracle.splitmix(0, n, rng.getrandbits(32))
            buf = torch.zeros(off + x.nbytes + 64, dtype=torch.uint8, device="cuda")
            src = buf[off: off + x.nbytes]
            src.copy_(torch.from_numpy(x))
            if rng.random() < 0.5:
                _run(keng, key, src, direction, out=src)
                got = src.cpu().numpy()
            else:
                got = _run(keng, key, src, direction).cpu().numpy()
            assert np.array_equal(got, oracle.ecb(x, s, direction)), (trial, key, n, direction, off)
            assert not buf[off + x.nbytes:].any()  # nothing written past the batch


def _kernel_names(fn):
    """Names of the CUDA kernels `fn` launches (torch.profiler / CUPTI sees
    the engine library's launches too)."""
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    return {e.name for e in prof.events()}


@pytest.mark.gpu
def test_auto_runs_a_prepared_keyed_module(keng, oracle):
    """AUTO never compiles a keyed kernel, but once t3des_cu_keyed_prepare
    has built one for the installed schedule and a direction, AUTO's
    bitsliced launches in that direction run it (small launches stay on the
    SP-table kernel, the other direction on the table-driven kernel), and a
    new schedule drops it.  Bytes equal the oracle throughout."""
    import paper_1305_4376_b200 as t3
    from paper_1305_4376_b200 import _native as N

    hexkey = KEYS["option1"]
    s = oracle.schedule_hex(hexkey)
    n = 1024 * 300 + 5  # > T3DES_CU_AUTO_SMALL_BLOCKS: bitsliced + side-stream tail
    x = oracle.splitmix(0, n, 0xA070)
    xd = torch.from_numpy(x).cuda()
    out = torch.empty_like(xd)
    st = torch.cuda.current_stream().cuda_stream
    keng.set_schedule(t3.triple_schedule(t3.parse_hex_key(hexkey)))
    keng.set_variant(N.VARIANT_AUTO)
    keng.set_launch(0, 0)

    def enc():
        keng.ecb_device(0, xd.data_ptr(), out.data_ptr(), x.nbytes, st)

    names = _kernel_names(enc)
    assert not any("keyed" in k for k in names), names  # not prepared: table-driven
    assert np.array_equal(out.cpu().numpy(), oracle.ecb(x, s, 0))
    keng.keyed_prepare(0)
    names = _kernel_names(enc)
    assert any("t3_keyed_kernel" in k for k in names), names
    assert np.array_equal(out.cpu().numpy(), oracle.ecb(x, s, 0))
    back = torch.empty_like(xd)
    names = _kernel_names(lambda: keng.ecb_device(1, out.data_ptr(), back.data_ptr(), x.nbytes, st))
    assert not any("keyed" in k for k in names), names  # decrypt was not prepared
    assert torch.equal(back, xd)
    other = KEYS["option2"]
    keng.set_schedule(t3.triple_schedule(t3.parse_hex_key(other)))
    names = _kernel_names(enc)
    assert not any("keyed" in k for k in names), names  # a new schedule drops it
    assert np.array_equal(out.cpu().numpy(), oracle.ecb(x, oracle.schedule_hex(other), 0))
