"""TEST INFRASTRUCTURE: ctypes access to the CPU checkers.

  oracle/liboracle.so          C restatement of the reference (always built)
  oracle/_ref/libt3des_ref.so  the reference itself (present when it was
                               compiled in the build container; travels with
                               the snapshot to the GPU box)
  tests/native bs_host         host build of the bitsliced core (CPU check
                               of the generated round code)

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg use this.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libt3des_ref.so")
BS_HOST_SO = os.path.join(ROOT, "tests", "native", "_build", "bs_host.so")

U64 = ctypes.c_uint64
_vp = ctypes.c_void_p
_sz = ctypes.c_size_t


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


class Oracle:
    def __init__(self, lib: ctypes.CDLL, ref: ctypes.CDLL | None):
        self.lib = lib
        self.ref = ref
        lib.oracle_ecb.argtypes = [_vp, _vp, _sz, ctypes.POINTER(U64), ctypes.c_int, ctypes.c_int, ctypes.c_int]
        lib.oracle_ecb.restype = ctypes.c_int
        lib.oracle_parse_hex_key.argtypes = [ctypes.c_char_p, _sz, ctypes.POINTER(U64)]
        lib.oracle_parse_hex_key.restype = ctypes.c_int
        lib.oracle_triple_schedule.argtypes = [U64, U64, U64, ctypes.POINTER(U64)]
        lib.oracle_key_schedule.argtypes = [U64, ctypes.POINTER(U64)]
        lib.oracle_make_payload.argtypes = [_vp, _sz, U64]
        lib.oracle_splitmix_payload.argtypes = [_vp, U64, _sz, U64]
        lib.oracle_splitmix_block.argtypes = [U64, U64]
        lib.oracle_splitmix_block.restype = U64
        lib.oracle_checksum.argtypes = [_vp, U64, _sz]
        lib.oracle_checksum.restype = U64
        lib.oracle_tdes_block.argtypes = [U64, ctypes.POINTER(U64), ctypes.c_int]
        lib.oracle_tdes_block.restype = U64
        lib.oracle_des_block.argtypes = [U64, U64, ctypes.c_int]
        lib.oracle_des_block.restype = U64
        lib.oracle_permute.argtypes = [U64, ctypes.c_int, ctypes.c_int]
        lib.oracle_permute.restype = U64
        lib.oracle_sbox.argtypes = [ctypes.c_int, ctypes.c_int]
        lib.oracle_sbox.restype = ctypes.c_int
        if ref is not None:
            ref.ref_ecb.argtypes = [_vp, _vp, _sz, ctypes.POINTER(U64), ctypes.c_int, ctypes.c_int,
                                    ctypes.c_uint, _sz, _sz]
            ref.ref_ecb.restype = ctypes.c_int
            ref.ref_schedule_hex.argtypes = [ctypes.c_char_p, ctypes.POINTER(U64), ctypes.POINTER(ctypes.c_int)]
            ref.ref_make_payload.argtypes = [_vp, U64, U64]
            ref.ref_resolve_workers.argtypes = [ctypes.c_uint]
            ref.ref_resolve_workers.restype = ctypes.c_uint

    @classmethod
    def load(cls) -> "Oracle":
        if not os.path.exists(ORACLE_SO):
            subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle")])
        lib = ctypes.CDLL(ORACLE_SO)
        ref = ctypes.CDLL(REF_SO) if os.path.exists(REF_SO) else None
        return cls(lib, ref)

    # -- keys --------------------------------------------------------------
    def schedule_hex(self, hexkey: str):
        k = (U64 * 3)()
        opt = self.lib.oracle_parse_hex_key(hexkey.encode(), len(hexkey), k)
        if opt < 0:
            raise ValueError(f"bad key ({opt})")
        s = (U64 * 48)()
        self.lib.oracle_triple_schedule(k[0], k[1], k[2], s)
        return s

    # -- batches -----------------------------------------------------------
    def ecb(self, data, sub48, decrypt: int, route: int = 1, threads: int = 0) -> np.ndarray:
        x = np.ascontiguousarray(np.frombuffer(bytes(data), dtype=np.uint8) if isinstance(data, (bytes, bytearray))
                                 else data, dtype=np.uint8).reshape(-1)
        y = np.empty_like(x)
        rc = self.lib.oracle_ecb(_ptr(x), _ptr(y), x.nbytes, sub48, int(decrypt), route, threads)
        assert rc == 0, rc
        return y

    def payload(self, nbytes: int, seed: int = 0x3DE5C0DE) -> np.ndarray:
        buf = np.empty(max(nbytes, 1), dtype=np.uint8)
        self.lib.oracle_make_payload(_ptr(buf), nbytes, seed)
        return buf[:nbytes]

    def splitmix(self, first_block: int, nblocks: int, seed: int) -> np.ndarray:
        buf = np.empty(max(8 * nblocks, 8), dtype=np.uint8)
        self.lib.oracle_splitmix_payload(_ptr(buf), first_block, nblocks, seed)
        return buf[: 8 * nblocks]

    def checksum(self, data: np.ndarray, first_block: int = 0) -> int:
        """oracle_checksum: the C restatement of t3_checksum_kernel."""
        assert data.nbytes % 8 == 0
        return int(self.lib.oracle_checksum(_ptr(data), first_block, data.nbytes // 8))

    def ref_ecb(self, data: np.ndarray, sub48, decrypt: int, backend: int = 1, workers: int = 0) -> np.ndarray:
        assert self.ref is not None
        y = np.empty_like(data)
        rc = self.ref.ref_ecb(_ptr(data), _ptr(y), data.nbytes, sub48, int(decrypt), backend, workers, 0, 0)
        assert rc == 0, rc
        return y


def sub48_from_hex_list(vals) -> "ctypes.Array":
    return (U64 * 48)(*[int(v, 16) for v in vals])


def checksum(data: np.ndarray, first_block: int = 0) -> int:
    """Host restatement of t3_checksum_kernel (kernels.cuh)."""
    w = np.frombuffer(data.tobytes(), dtype="<u8").astype(np.uint64)
    idx = np.arange(first_block, first_block + w.size, dtype=np.uint64)
    z = (w ^ idx) ^ np.uint64(0x3DE5C0DE)
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
        return int(np.sum(z, dtype=np.uint64))


def bs_host() -> ctypes.CDLL:
    """Build (if needed) and load the host build of the bitsliced core."""
    src = [os.path.join(ROOT, "tests", "native", "bs_host.cpp"),
           os.path.join(ROOT, "paper_1305_4376_b200", "csrc", "schedule.cpp")]
    deps = src + [os.path.join(ROOT, "paper_1305_4376_b200", "csrc", p) for p in
                  ("t3des_core.cuh", "schedule.hpp", "generated/bitslice_rounds.cuh", "generated/bitslice_tables.h")]
    if not os.path.exists(BS_HOST_SO) or any(os.path.getmtime(d) > os.path.getmtime(BS_HOST_SO) for d in deps):
        os.makedirs(os.path.dirname(BS_HOST_SO), exist_ok=True)
        subprocess.check_call(["/usr/bin/g++", "-std=c++17", "-O2", "-shared", "-fPIC",
                               "-I" + os.path.join(ROOT, "paper_1305_4376_b200", "csrc"), "-o", BS_HOST_SO] + src)
    lib = ctypes.CDLL(BS_HOST_SO)
    lib.bs_host_ecb.argtypes = [_vp, _vp, _sz, ctypes.POINTER(U64), ctypes.c_int]
    lib.bs_host_table.argtypes = [ctypes.POINTER(U64), ctypes.c_int, ctypes.POINTER(ctypes.c_uint32)]
    lib.bs_host_ecb_collapse.argtypes = [_vp, _vp, _sz, ctypes.POINTER(U64), ctypes.c_int]
    return lib
