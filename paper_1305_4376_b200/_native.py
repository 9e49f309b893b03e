"""ctypes binding of the C ABI (include/t3des_cu.h) in libt3des_b200.so.

The shared library is built in-tree by ``make -C paper_1305_4376_b200/csrc``
(or ``__graft_entry__.build()``).  If it is missing, importing the package
still works (key parsing is pure host code in the same library, so it is
missing too) but every call raises :class:`EngineUnavailable` — there is no
CPU fallback for the cipher.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libt3des_b200.so")

OK = 0
ERR_LENGTH = 1
ERR_OVERLAP = 2
ERR_KEY = 3
ERR_ARG = 4
ERR_NO_DEVICE = 5
ERR_CUDA = 6
ERR_NO_SCHEDULE = 7
ERR_PADDING = 8
ERR_IO = 9
ERR_JIT = 10

ENCRYPT = 0
DECRYPT = 1
VARIANT_BITSLICE = 0
VARIANT_SPTABLE = 1
VARIANT_BITSLICE_LDG = 2
VARIANT_BITSLICE_ALU = 3
VARIANT_BITSLICE_DFMA = 4
VARIANT_BITSLICE_SHRFMA = 5
VARIANT_AUTO = 6
VARIANT_KEYED = 7  # key-specialised, NVRTC-compiled at run time (opt-in)
AUTO_SMALL_BLOCKS = 131072
MULTI_STAGE_ALL = 1  # t3des_cu_ecb_multi_device flags
MULTI_COPY = 2
KEY_ODD_PARITY = 1  # t3des_cu_des_key_flags bits
KEY_WEAK = 2
KEY_SEMIWEAK = 4

class StreamReportC(ctypes.Structure):
    """t3des_cu_stream_report (include/t3des_cu.h)."""

    _fields_ = [("bytes_in", ctypes.c_uint64), ("bytes_out", ctypes.c_uint64), ("chunks", ctypes.c_uint64),
                ("compute_seconds", ctypes.c_double), ("io_seconds", ctypes.c_double),
                ("error_offset", ctypes.c_uint64)]


# Every symbol include/t3des_cu.h declares: name -> (restype, argtypes).
_u64p = ctypes.POINTER(ctypes.c_uint64)
_vp = ctypes.c_void_p
_sz = ctypes.c_size_t
_i = ctypes.c_int
SIGNATURES = {
    "t3des_cu_version": (_i, []),
    "t3des_cu_strerror": (ctypes.c_char_p, [_i]),
    "t3des_cu_parse_hex_key": (_i, [ctypes.c_char_p, _sz, _u64p, ctypes.POINTER(_i)]),
    "t3des_cu_triple_schedule": (_i, [_u64p, _u64p]),
    "t3des_cu_des_key_flags": (_i, [ctypes.c_uint64]),
    "t3des_cu_normalize_parity": (ctypes.c_uint64, [ctypes.c_uint64]),
    "t3des_cu_run_verification": (_i, [_i, ctypes.c_char_p, _sz]),
    "t3des_cu_device_count": (_i, [ctypes.POINTER(_i)]),
    "t3des_cu_create": (_i, [_i, ctypes.POINTER(_vp)]),
    "t3des_cu_destroy": (_i, [_vp]),
    "t3des_cu_set_schedule": (_i, [_vp, _u64p]),
    "t3des_cu_set_variant": (_i, [_vp, _i]),
    "t3des_cu_keyed_prepare": (_i, [_vp, _i, ctypes.POINTER(ctypes.c_double)]),
    "t3des_cu_keyed_compile": (_i, [_u64p, _i, _vp, _sz, ctypes.POINTER(_sz), ctypes.POINTER(ctypes.c_double)]),
    "t3des_cu_set_launch": (_i, [_vp, _sz, _i]),
    "t3des_cu_ecb_device": (_i, [_vp, _i, _vp, _vp, _sz, _vp]),
    "t3des_cu_ecb_host": (_i, [_vp, _i, _vp, _vp, _sz]),
    "t3des_cu_set_pipeline": (_i, [_vp, _sz, _i]),
    "t3des_cu_stream_fd": (_i, [_vp, _i, _i, _i, _sz, _i, ctypes.POINTER(StreamReportC)]),
    "t3des_cu_ecb_multi": (_i, [ctypes.POINTER(_i), _i, _u64p, _i, _vp, _vp, _sz]),
    "t3des_cu_ecb_workers": (_i, [ctypes.c_uint, _i, _u64p, _i, _vp, _vp, _sz]),
    "t3des_cu_ecb_multi_device": (_i, [ctypes.POINTER(_i), _i, _u64p, _i, _i, _vp, _vp, _sz, _i]),
    "t3des_cu_multi_device_shards": (_i, [ctypes.POINTER(_i), _i, _i, ctypes.c_uint64, _i, _u64p, _u64p]),
    "t3des_cu_shard_range": (_i, [ctypes.c_uint64, _i, _i, _u64p, _u64p]),
    "t3des_cu_host_alloc": (_i, [_sz, ctypes.POINTER(_vp)]),
    "t3des_cu_host_free": (_i, [_vp]),
    "t3des_cu_host_register": (_i, [_vp, _sz]),
    "t3des_cu_host_unregister": (_i, [_vp]),
    "t3des_cu_fill_splitmix": (_i, [_vp, _vp, ctypes.c_uint64, _sz, ctypes.c_uint64, _vp]),
    "t3des_cu_checksum": (_i, [_vp, _vp, ctypes.c_uint64, _sz, _u64p, _vp]),
    "t3des_cu_launch_count": (_i, [_vp, _u64p]),
}


class EngineUnavailable(RuntimeError):
    """The CUDA engine library is not built or cannot be loaded."""


_lib = None
_load_error: str | None = None


def lib() -> ctypes.CDLL:
    global _lib, _load_error
    if _lib is not None:
        return _lib
    if _load_error is not None:
        raise EngineUnavailable(_load_error)
    if not os.path.exists(LIB_PATH):
        _load_error = f"{LIB_PATH} not built (run __graft_entry__.build())"
        raise EngineUnavailable(_load_error)
    try:
        l = ctypes.CDLL(LIB_PATH)
    except OSError as e:  # pragma: no cover - environment dependent
        _load_error = f"cannot load {LIB_PATH}: {e}"
        raise EngineUnavailable(_load_error) from e
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(l, name)
        fn.restype = res
        fn.argtypes = args
    _lib = l
    return l


def strerror(code: int) -> str:
    return lib().t3des_cu_strerror(code).decode()
