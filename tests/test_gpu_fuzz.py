"""Randomised parity of the host-buffer paths (the drop-in surface a reference
caller uses): random block counts (0 .. ~5 MiB, ragged), keying options,
directions, in place or not, pageable / pinned / registered memory on either
side, byte offsets that break 8- and 16-byte alignment, and the workers axis —
every output byte against the C oracle.  Seeded, so a failure reproduces."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
import paper_1305_4376_b200 as t3  # noqa: E402

pytestmark = pytest.mark.gpu

KEYS = ["133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57", "0123456789ABCDEF23456789ABCDEF01", "0123456789ABCDEF",
        "0123456789ABCDEF0123456789ABCDEF456789ABCDEF0123"]


def buffer(kind: str, nbytes: int, offset: int, rng):
    """(array view of nbytes at `offset` into a fresh allocation, keepalive)."""
    if kind == "pinned":
        base = torch.empty(nbytes + 64, dtype=torch.uint8).pin_memory()
        arr = base.numpy()
    else:
        arr = np.empty(nbytes + 64, dtype=np.uint8)
        base = arr
    view = arr[offset:offset + nbytes]
    view[:] = rng.integers(0, 256, nbytes, dtype=np.uint8)
    return view, base


@pytest.mark.parametrize("seed", range(6))
def test_random_host_batches(oracle, seed):
    rng = np.random.default_rng(1000 + seed)
    for case in range(25):
        n = int(rng.choice([0, 1, 7, 1023, 1024, 1025, int(rng.integers(1, 700_000))]))
        key = KEYS[int(rng.integers(0, len(KEYS)))]
        d = int(rng.integers(0, 2))
        kin = str(rng.choice(["pageable", "pinned", "registered"]))
        kout = str(rng.choice(["pageable", "pinned", "registered"]))
        if 8 * n < (1 << 20):  # registration page-locks whole pages: only separate mmap'd buffers
            kin = "pageable" if kin == "registered" else kin
            kout = "pageable" if kout == "registered" else kout
        inplace = bool(rng.integers(0, 3) == 0)
        off_in = int(rng.choice([0, 8, 16, 3]))
        off_out = int(rng.choice([0, 8, 24, 5]))
        workers = int(rng.choice([0, 0, 0, 2, 3]))
        x, keep_x = buffer("pinned" if kin == "pinned" else "pageable", 8 * n, off_in, rng)
        want = oracle.ecb(x.copy(), oracle.schedule_hex(key), d)
        regs = []
        if inplace:
            y, keep_y = x, keep_x
        else:
            y, keep_y = buffer("pinned" if kout == "pinned" else "pageable", 8 * n, off_out, rng)
            if kout == "registered" and n:
                regs.append(t3.HostRegistration(y))
        if kin == "registered" and n:
            regs.append(t3.HostRegistration(x))
        ts = t3.triple_schedule(t3.parse_hex_key(key))
        cfg = t3.DispatchConfig(workers=workers)
        try:
            (t3.decrypt_batch if d else t3.encrypt_batch)(x, y, ts, cfg)
        finally:
            for r in regs:
                r.close()
        assert np.array_equal(y, want), (seed, case, n, key, d, kin, kout, inplace, off_in, off_out, workers)
        del keep_x, keep_y
