"""Block-range sharding across GPUs: ECB blocks are
independent (reference SPEC.md:221-223), so N blocks split into contiguous
ranges with no collective.  The arithmetic lives in the C ABI
(t3des_cu_shard_range) so t3des_cu_ecb_multi, bench.py's torchrun ranks and
the tests agree by construction."""
from __future__ import annotations

import ctypes

from . import _native as N

TILE_BLOCKS = 1024


def shard_range(nblocks: int, world: int, rank: int) -> tuple[int, int]:
    """(first_block, count) owned by `rank` of `world`."""
    first, count = ctypes.c_uint64(), ctypes.c_uint64()
    rc = N.lib().t3des_cu_shard_range(nblocks, world, rank, ctypes.byref(first), ctypes.byref(count))
    if rc:
        raise ValueError(N.strerror(rc))
    return first.value, count.value
