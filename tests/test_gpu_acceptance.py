"""GPU mirrors of the reference's acceptance criteria and randomized
equivalence tests (proj/tests/acceptance.cpp:104-152,284-300;
test_tdes.cpp:81-90,110-122), against the CPU oracle."""
import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import paper_1305_4376_b200 as t3  # noqa: E402
from paper_1305_4376_b200 import _native as N  # noqa: E402
from tests.oracle_util import U64  # noqa: E402

pytestmark = pytest.mark.gpu
BENCH_KEY = "133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57"


@pytest.fixture(scope="module")
def eng(engine_lib):
    e = t3.Engine(0)
    yield e
    e.close()


def _run(eng, sub48, x, d, variant=N.VARIANT_AUTO):
    eng.set_sub48(sub48)
    eng.set_variant(variant)
    src = torch.from_numpy(x).cuda()
    dst = torch.empty_like(src)
    eng.ecb_device(d, src.data_ptr(), dst.data_ptr(), x.nbytes, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return dst.cpu().numpy()


def test_random_three_key_cases(eng, oracle):
    # fast == reference on random 3-key cases (test_tdes.cpp:110-122)
    rng = np.random.default_rng(1234)
    for i in range(300):
        k = rng.integers(0, 2**63, 3, dtype=np.uint64)
        s = (U64 * 48)()
        oracle.lib.oracle_triple_schedule(int(k[0]), int(k[1]), int(k[2]), s)
        x = rng.integers(0, 256, 8 * (1 + 97 * (i % 23)), dtype=np.uint8)
        v = (N.VARIANT_BITSLICE, N.VARIANT_SPTABLE)[i % 2]
        for d in (0, 1):
            assert np.array_equal(_run(eng, s, x, d, v), oracle.ecb(x, s, d, route=0)), (i, d)


def test_option3_collapses_to_single_des(eng, oracle):
    # acceptance.cpp:104-116 (c3): K1 = K2 = K3 is single DES
    rng = np.random.default_rng(99)
    for i in range(200):
        k = int(rng.integers(0, 2**63, dtype=np.uint64))
        s = oracle.schedule_hex(f"{k:016X}")
        x = rng.integers(0, 256, 8 * 1025, dtype=np.uint8)
        y = _run(eng, s, x, 0, (N.VARIANT_BITSLICE, N.VARIANT_SPTABLE)[i % 2])
        for b in (0, 511, 1024):
            blk = int.from_bytes(x[8 * b: 8 * b + 8].tobytes(), "big")
            assert int.from_bytes(y[8 * b: 8 * b + 8].tobytes(), "big") == oracle.lib.oracle_des_block(blk, k, 0)


def test_identical_blocks(eng, oracle):
    # acceptance.cpp:284-300 (c9): 1000 identical blocks -> 1000 identical outputs
    s = oracle.schedule_hex(BENCH_KEY)
    x = np.tile(np.frombuffer(bytes.fromhex("0123456789ABCDEF"), np.uint8), 1000)
    for v in (N.VARIANT_BITSLICE, N.VARIANT_SPTABLE):
        y = _run(eng, s, x, 0, v).reshape(1000, 8)
        assert (y == y[0]).all() and y[0].tobytes() == oracle.ecb(x[:8], s, 0).tobytes()


def test_backend_equivalence_64mib(eng, oracle):
    """acceptance.cpp:119-152 (c4): 64 MiB, output independent of GPU count
    {1,2,4,8}, blocks per launch {1024, 131072} and CTA size {32, 64, 128};
    multiple GPUs are emulated by contexts on device 0 when only one exists."""
    s = oracle.schedule_hex(BENCH_KEY)
    x = oracle.payload(64 << 20)
    want = oracle.ecb(x, s, 0)
    ts = t3.triple_schedule(t3.parse_hex_key(BENCH_KEY))
    for chunk in (1024, 131072):
        for wg in (32, 64, 128):
            out = np.empty_like(x)
            t3.encrypt_batch(x, out, ts, t3.DispatchConfig(chunk_blocks=chunk, work_group=wg, gpu_chunked=True,
                                                            variant=N.VARIANT_BITSLICE))
            assert np.array_equal(out, want), (chunk, wg)
    ngpu = torch.cuda.device_count()
    for g in (1, 2, 4, 8):
        devs = [i % ngpu for i in range(g)]
        out = np.empty_like(x)
        arr = (ctypes.c_int * g)(*devs)
        assert N.lib().t3des_cu_ecb_multi(arr, g, s, 0, x.ctypes.data, out.ctypes.data, x.nbytes) == 0
        assert np.array_equal(out, want), g
