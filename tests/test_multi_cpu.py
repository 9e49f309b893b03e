"""Multi-GPU decomposition, exercised on CPU with world-size-2 gloo (no GPU
here): each rank takes its shard (t3des_cu_shard_range, the same function the
C ABI's ecb_multi and bench.py's ranks use), transforms it with the CPU
oracle as a stand-in for its device, and the ranks check that the shards
tile the stream exactly, that concatenating them equals the single-process
result, that the shard checksums add up (the invariant the GPU runs check
across 1/2/4/8 GPUs), and that the max-over-ranks timing reduction works."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1305_4376_b200.sharding import TILE_BLOCKS, shard_range
from tests.oracle_util import Oracle, checksum

KEY = "133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57"


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, nblocks: int, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        o = Oracle.load()
        s = o.schedule_hex(KEY)
        first, count = shard_range(nblocks, world, rank)
        x = o.splitmix(first, count, 0x3DE5C0DE)
        y = o.ecb(x, s, 0, threads=1)
        cs = torch.tensor([checksum(y, first) & ((1 << 63) - 1), checksum(y, first) >> 63], dtype=torch.int64)
        dist.all_reduce(cs, op=dist.ReduceOp.SUM)
        # bench.py's form: each rank's u64 checksum as a signed int64,
        # all_gather, sum mod 2^64 on the receiver
        import bench

        mine = torch.tensor([bench.u64_to_i64(checksum(y, first))], dtype=torch.int64)
        parts = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine)
        bench_sum = sum(int(p.item()) for p in parts) % 2**64
        bounds = torch.tensor([first, count], dtype=torch.int64)
        gathered = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(gathered, bounds)
        outs = [None] * world
        dist.all_gather_object(outs, y.tobytes())
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            q.put((cs.tolist(), [g.tolist() for g in gathered], b"".join(outs), float(t.item()), bench_sum))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("nblocks", [0, 1, 1023, 5 * TILE_BLOCKS + 17, 65536])
def test_two_rank_block_range_sharding(nblocks):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, nblocks, q)) for r in range(world)]
    for p in procs:
        p.start()
    cs, bounds, joined, tmax, bench_sum = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # shards tile [0, N) in order, boundaries on 1024-block tiles
    pos = 0
    for first, count in bounds:
        assert first == pos
        pos += count
    assert pos == nblocks
    assert all(f % TILE_BLOCKS == 0 for f, _ in bounds)
    o = Oracle.load()
    whole = o.ecb(o.splitmix(0, nblocks, 0x3DE5C0DE), o.schedule_hex(KEY), 0)
    assert joined == whole.tobytes()
    full = checksum(whole, 0)
    assert ((cs[1] << 63) + cs[0]) % 2**64 == full
    assert bench_sum == full
    assert tmax == 2.0


def test_shard_range_properties():
    for n in (0, 1, 1024, 10**6 + 3, 8_589_934_592):
        for world in (1, 2, 4, 8):
            spans = [shard_range(n, world, g) for g in range(world)]
            assert spans[0][0] == 0
            assert sum(c for _, c in spans) == n
            for (f0, c0), (f1, _) in zip(spans, spans[1:]):
                assert f0 + c0 == f1 and f1 % TILE_BLOCKS == 0
    # 64 GiB over 8 GPUs: exactly 8 GiB each (BASELINE configs[3])
    assert shard_range(8_589_934_592, 8, 3) == (3 * 1_073_741_824, 1_073_741_824)
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_bench_self_launches_n_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself under
    torch.distributed.run with 2 ranks (T3DES_BENCH_LAUNCH_PROBE: the ranks
    report and exit before touching a GPU); the two shards of the configs[3]
    64 GiB stream tile it exactly; a WORLD_SIZE that contradicts --gpus exits 2."""
    import json
    import subprocess
    import sys

    from tests.oracle_util import ROOT

    env = dict(os.environ, T3DES_BENCH_LAUNCH_PROBE="1")
    env.pop("WORLD_SIZE", None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"], capture_output=True,
                       text=True, env=env, timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    recs = sorted((json.loads(l) for l in p.stdout.splitlines() if l.startswith("{")), key=lambda r: r["rank"])
    assert [r["rank"] for r in recs] == [0, 1] and all(r["world"] == 2 for r in recs)
    n = (64 << 30) // 8
    (f0, c0), (f1, c1) = recs[0]["shard"], recs[1]["shard"]
    assert f0 == 0 and f1 == c0 and f1 + c1 == n
    bad = dict(env, WORLD_SIZE="3")
    assert subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"], env=bad,
                          capture_output=True, timeout=120).returncode == 2


def _md_shards(devs, home, n, flags=0):
    import ctypes

    from paper_1305_4376_b200 import _native as N

    k = len(devs)
    f, c = (ctypes.c_uint64 * k)(), (ctypes.c_uint64 * k)()
    assert N.lib().t3des_cu_multi_device_shards((ctypes.c_int * k)(*devs), k, home, n, flags, f, c) == 0
    return list(f), list(c)


@pytest.mark.parametrize("n", [0, 1, 1023, 5 * TILE_BLOCKS + 17, (64 << 30) // 8])
def test_multi_device_home_weighted_shards(n, monkeypatch):
    """t3des_cu_ecb_multi_device's split for data resident on `home`: the home
    shard (no NVLink copy) is weighted against the remote peer-copy bound —
    h = 396 / (396 + min(770, (G-1) * 396)): 0.5 at G = 2, ~0.34 from G = 3 —
    contiguous tile-aligned ranges covering [0, n); equal shards when the
    home GPU is absent, duplicated, or with STAGE_ALL."""
    monkeypatch.delenv("T3DES_MULTI_HOME_SHARE", raising=False)
    for devs, home, want_h in (([0, 1, 2, 3, 4, 5, 6, 7], 0, 396 / (396 + 770)), ([0, 1], 0, 0.5),
                               ([3, 1, 2], 1, 396 / (396 + 770))):
        f, c = _md_shards(devs, home, n)
        assert f[0] == 0 and sum(c) == n and all(f[g + 1] == f[g] + c[g] for g in range(len(devs) - 1))
        assert all(x % TILE_BLOCKS == 0 for x in f)
        hi = devs.index(home)
        if n >= 64 * TILE_BLOCKS * len(devs):
            assert abs(c[hi] / n - want_h) < 0.001
            rest = [c[g] for g in range(len(devs)) if g != hi]
            assert max(rest) - min(rest) <= 2 * TILE_BLOCKS
    for devs, home, flags in (([1, 2, 3], 0, 0), ([0, 0, 0], 0, 0), ([0, 1, 2], 0, 1)):
        f, c = _md_shards(devs, home, n, flags)
        assert [(a, b) for a, b in zip(f, c)] == [shard_range(n, len(devs), g) for g in range(len(devs))]
    monkeypatch.setenv("T3DES_MULTI_HOME_SHARE", "0.2")
    f, c = _md_shards([0, 0, 0], 0, n)
    assert sum(c) == n and (n < 64 * TILE_BLOCKS or abs(c[0] / n - 0.2) < 0.001)
