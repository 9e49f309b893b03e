"""Python host API of the B200 3DES-ECB engine.

Mirrors the reference's hot-path API (/root/reference/proj/include/t3des)
so its tests read the same way:

    reference                              here
    parse_hex_key (tdes.hpp:32)            parse_hex_key(hex) -> TripleKey
    key_schedule (des.hpp:35)              key_schedule(DesKey|int) -> list[int]
    triple_schedule (tdes.hpp:42)          triple_schedule(TripleKey) -> TripleSchedule
    encrypt_batch/decrypt_batch            encrypt_batch(in, out, ts, cfg)
        (dispatch.hpp:64-69)
    Backend, DispatchConfig (:19-30)       Backend.CUDA (default), DispatchConfig
    plan_dispatch (:39-42)                 plan_dispatch(total_blocks, cfg)
    InputLengthError, KeyFormatError       same names (Python exceptions)

Everything goes through the C ABI (``_native``); there is no Python or CPU
cipher here.  Buffers may be bytes-like / numpy (host, end-to-end path with
host<->device copies) or CUDA torch tensors (device-resident path,
enqueued on the current torch stream).
"""
from __future__ import annotations

import ctypes
import enum
import threading
from dataclasses import dataclass, field

from . import _native as N


class KeyFormatError(ValueError):
    """Hex key of bad length or with a non-hex character (tdes.hpp:25-28)."""


class InputLengthError(ValueError):
    """Batch length not a multiple of 8, size mismatch, or partial overlap
    (dispatch.hpp:44-47)."""


class PaddingError(ValueError):
    """Malformed PKCS#7 padding (dispatch.hpp:49-52)."""


class IoError(OSError):
    """Stream read/write failure at byte_offset (dispatch.hpp:54-59)."""

    def __init__(self, msg: str, byte_offset: int):
        super().__init__(msg)
        self.byte_offset = byte_offset


class CudaError(RuntimeError):
    """Device or CUDA runtime failure; never silently falls back to a CPU."""

    def __init__(self, msg: str, code: int):
        super().__init__(msg)
        self.status = code


def _raise(rc: int, what: str = "") -> None:
    if rc == N.OK:
        return
    msg = N.strerror(rc) + (f" ({what})" if what else "")
    if rc in (N.ERR_LENGTH, N.ERR_OVERLAP):
        raise InputLengthError(msg)
    if rc == N.ERR_KEY:
        raise KeyFormatError(msg)
    if rc == N.ERR_PADDING:
        raise PaddingError(msg)
    if rc == N.ERR_ARG:
        raise ValueError(msg)
    raise CudaError(msg, rc)


class KeyingOption(enum.Enum):
    Option1 = 1  # three independent keys (48 hex chars)
    Option2 = 2  # k3 = k1 (32 hex chars)
    Option3 = 3  # k1 = k2 = k3 (16 hex chars)


@dataclass(frozen=True)
class DesKey:
    raw: int = 0


@dataclass(frozen=True)
class TripleKey:
    k1: DesKey
    k2: DesKey
    k3: DesKey
    option: KeyingOption = KeyingOption.Option1


@dataclass(frozen=True)
class TripleSchedule:
    """48 round keys, pass-major (16 for k1, then k2, then k3)."""

    pass1: tuple
    pass2: tuple
    pass3: tuple

    def sub48(self) -> "ctypes.Array[ctypes.c_uint64]":
        return (ctypes.c_uint64 * 48)(*self.pass1, *self.pass2, *self.pass3)


def parse_hex_key(hex_key: str) -> TripleKey:
    b = hex_key.encode() if isinstance(hex_key, str) else bytes(hex_key)
    keys = (ctypes.c_uint64 * 3)()
    opt = ctypes.c_int()
    rc = N.lib().t3des_cu_parse_hex_key(b, len(b), keys, ctypes.byref(opt))
    if rc == N.ERR_KEY:
        if len(b) not in (16, 32, 48):
            raise KeyFormatError(f"key must be 16, 32 or 48 hex characters, got {len(b)}")
        raise KeyFormatError("invalid hex character in key")
    _raise(rc)
    return TripleKey(DesKey(keys[0]), DesKey(keys[1]), DesKey(keys[2]), KeyingOption(opt.value))


def to_hex(key: TripleKey) -> str:
    if key.option is KeyingOption.Option1:
        return f"{key.k1.raw:016X}{key.k2.raw:016X}{key.k3.raw:016X}"
    if key.option is KeyingOption.Option2:
        return f"{key.k1.raw:016X}{key.k2.raw:016X}"
    return f"{key.k1.raw:016X}"


def _schedule3(k1: int, k2: int, k3: int) -> list[int]:
    keys = (ctypes.c_uint64 * 3)(k1, k2, k3)
    out = (ctypes.c_uint64 * 48)()
    _raise(N.lib().t3des_cu_triple_schedule(keys, out))
    return list(out)


def key_schedule(key) -> list[int]:
    raw = key.raw if isinstance(key, DesKey) else int(key)
    return _schedule3(raw, raw, raw)[:16]


def triple_schedule(key: TripleKey) -> TripleSchedule:
    s = _schedule3(key.k1.raw, key.k2.raw, key.k3.raw)
    return TripleSchedule(tuple(s[:16]), tuple(s[16:32]), tuple(s[32:]))


class ParityError(ValueError):
    """des.hpp:25-28 (raised by callers that enforce odd parity, e.g. the CLI's --check-parity)."""


def _raw(key) -> int:
    return key.raw if isinstance(key, DesKey) else int(key)


def has_odd_parity(key) -> bool:
    """des.hpp:42: every byte of the 64-bit key has odd parity."""
    return bool(N.lib().t3des_cu_des_key_flags(_raw(key)) & N.KEY_ODD_PARITY)


def normalize_parity(key) -> DesKey:
    """des.hpp:43: the LSB of each even-parity byte flipped."""
    return DesKey(int(N.lib().t3des_cu_normalize_parity(_raw(key))))


def is_weak_key(key) -> bool:
    """des.hpp:47: one of the 4 weak keys (parity bits masked)."""
    return bool(N.lib().t3des_cu_des_key_flags(_raw(key)) & N.KEY_WEAK)


def is_semiweak_key(key) -> bool:
    """des.hpp:48: one of the 12 semi-weak keys (parity bits masked)."""
    return bool(N.lib().t3des_cu_des_key_flags(_raw(key)) & N.KEY_SEMIWEAK)


def load_block(b: bytes) -> int:
    return int.from_bytes(bytes(b[:8]), "big")


def store_block(v: int) -> bytes:
    return int(v).to_bytes(8, "big")


class Backend(enum.Enum):
    ScalarReference = 0  # the reference's CPU oracle — not in this engine
    Threaded = 1         # the reference's OpenMP backend — not in this engine
    NoOpCopy = 2         # copy only (timing instrumentation)
    CUDA = 3             # B200 kernels


@dataclass
class DispatchConfig:
    chunk_blocks: int = 131072  # blocks per launch, applied only if gpu_chunked
    work_group: int = 256       # threads per CTA, applied only if gpu_chunked
    workers: int = 0            # CUDA: block-range shards, at most one per GPU, from `device` (0 = one)
    backend: Backend = Backend.CUDA
    device: int = 0
    variant: int = N.VARIANT_AUTO
    gpu_chunked: bool = False


@dataclass(frozen=True)
class ChunkSpan:
    offset: int
    length: int


def plan_dispatch(total_blocks: int, cfg: DispatchConfig) -> list[ChunkSpan]:
    step = cfg.chunk_blocks or max(total_blocks, 1)
    return [ChunkSpan(o, min(step, total_blocks - o)) for o in range(0, total_blocks, step)]


def resolve_workers(cfg: DispatchConfig) -> int:
    """dispatch.hpp:94 on Backend::CUDA: block-range shards per batch (0 -> 1)."""
    return cfg.workers or 1


class Engine:
    """One device context (t3des_cu_ctx).  Use from one thread at a time."""

    def __init__(self, device: int = 0):
        self._lib = N.lib()
        h = ctypes.c_void_p()
        _raise(self._lib.t3des_cu_create(int(device), ctypes.byref(h)), f"device {device}")
        self._h = h
        self.device = int(device)
        # last values installed through this wrapper: the batch API re-applies
        # schedule / variant / launch shape on every call, and skipping the
        # unchanged ones saves the ctypes round trips (TripleSchedule is frozen)
        self._ts = None
        self._variant = None
        self._launch = None

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.t3des_cu_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass

    def set_schedule(self, ts: TripleSchedule) -> None:
        if ts is self._ts:
            return
        self._ts = None
        _raise(self._lib.t3des_cu_set_schedule(self._h, ts.sub48()))
        self._ts = ts

    def set_sub48(self, sub48) -> None:
        """Install a raw pass-major 48-subkey array (ctypes c_uint64 * 48)."""
        self._ts = None
        _raise(self._lib.t3des_cu_set_schedule(self._h, sub48))

    def set_variant(self, variant: int) -> None:
        if variant == self._variant:
            return
        _raise(self._lib.t3des_cu_set_variant(self._h, int(variant)))
        self._variant = int(variant)

    def keyed_prepare(self, direction: int) -> float:
        """VARIANT_KEYED: compile (or find cached) and load the key-specialised
        kernel of the installed schedule for `direction`; returns the seconds
        spent (0.0 on a cache hit)."""
        secs = ctypes.c_double()
        _raise(self._lib.t3des_cu_keyed_prepare(self._h, int(direction), ctypes.byref(secs)))
        return secs.value

    def set_launch(self, chunk_blocks: int = 0, work_group: int = 0) -> None:
        shape = (int(chunk_blocks), int(work_group))
        if shape == self._launch:
            return
        _raise(self._lib.t3des_cu_set_launch(self._h, *shape))
        self._launch = shape

    def set_pipeline(self, chunk_bytes: int = 32 << 20, streams: int = 3) -> None:
        _raise(self._lib.t3des_cu_set_pipeline(self._h, int(chunk_bytes), int(streams)))

    def ecb_device(self, direction: int, din: int, dout: int, nbytes: int, stream: int = 0) -> None:
        _raise(self._lib.t3des_cu_ecb_device(self._h, int(direction), din, dout, int(nbytes), stream or None))

    def ecb_host(self, direction: int, src: int, dst: int, nbytes: int) -> None:
        _raise(self._lib.t3des_cu_ecb_host(self._h, int(direction), src, dst, int(nbytes)))

    def fill_splitmix(self, dptr: int, first_block: int, nblocks: int, seed: int, stream: int = 0) -> None:
        _raise(self._lib.t3des_cu_fill_splitmix(self._h, dptr, first_block, nblocks, seed, stream or None))

    def checksum(self, dptr: int, first_block: int, nblocks: int, stream: int = 0) -> int:
        """Checksum on `stream` (default: the legacy default stream)."""
        out = ctypes.c_uint64()
        _raise(self._lib.t3des_cu_checksum(self._h, dptr, first_block, nblocks, ctypes.byref(out), stream or None))
        return out.value

    def launch_count(self) -> int:
        out = ctypes.c_uint64()
        _raise(self._lib.t3des_cu_launch_count(self._h, ctypes.byref(out)))
        return out.value


_engines = threading.local()  # one context per device per thread (a context has one submitter at a time)


def engine(device: int = 0) -> Engine:
    """The calling thread's context for `device` (created on first use).
    Per thread, like the C++ mirror's context cache: the batch functions stay
    callable from several threads at once, as the reference's are."""
    cache = getattr(_engines, "by_device", None)
    if cache is None:
        cache = _engines.by_device = {}
    e = cache.get(device)
    if e is None:
        e = cache[device] = Engine(device)
    return e


def _is_cuda_tensor(x) -> bool:
    return getattr(x, "is_cuda", False) is True


def _host_view(x, writable: bool):
    """(address, nbytes, keepalive) of a host buffer."""
    import numpy as np

    if hasattr(x, "data_ptr") and hasattr(x, "element_size"):  # CPU torch tensor
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return x.data_ptr(), x.numel() * x.element_size(), x
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        if writable and not x.flags["WRITEABLE"]:
            raise ValueError("output array is read-only")
        return x.ctypes.data, x.nbytes, x
    mv = memoryview(x)
    if writable and mv.readonly:
        raise ValueError("output buffer is read-only")
    arr = np.frombuffer(mv, dtype=np.uint8) if mv.readonly else np.asarray(mv).view(np.uint8).reshape(-1)
    return arr.ctypes.data, arr.nbytes, (arr, mv)


def _run_batch(src, dst, ts: TripleSchedule, cfg: DispatchConfig, direction: int) -> None:
    if cfg.backend in (Backend.ScalarReference, Backend.Threaded):
        raise NotImplementedError(
            "the B200 engine provides Backend.CUDA (and NoOpCopy); CPU backends live in the reference"
        )
    if _is_cuda_tensor(src) or _is_cuda_tensor(dst):
        if not (_is_cuda_tensor(src) and _is_cuda_tensor(dst)):
            raise ValueError("in and out must both be CUDA tensors or both host buffers")
        import torch

        nin = src.numel() * src.element_size()
        nout = dst.numel() * dst.element_size()
        if nin != nout:
            raise InputLengthError("output buffer size mismatch")
        if not (src.is_contiguous() and dst.is_contiguous()):
            raise ValueError("tensors must be contiguous")
        if src.device != dst.device:
            raise ValueError(f"in and out must be on the same device ({src.device} vs {dst.device})")
        if cfg.backend is Backend.NoOpCopy:
            if src.data_ptr() != dst.data_ptr():
                dst.view(torch.uint8).copy_(src.view(torch.uint8).reshape(-1).view_as(dst.view(torch.uint8)))
            return
        e = engine(src.device.index or 0)
        e.set_schedule(ts)
        e.set_variant(cfg.variant)
        e.set_launch(cfg.chunk_blocks if cfg.gpu_chunked else 0, cfg.work_group if cfg.gpu_chunked else 0)
        stream = torch.cuda.current_stream(src.device).cuda_stream
        e.ecb_device(direction, src.data_ptr(), dst.data_ptr(), nin, stream)
        return
    pin, nin, keep_in = _host_view(src, False)
    pout, nout, keep_out = _host_view(dst, True)
    if nin % 8:
        raise InputLengthError(f"batch length {nin} is not a multiple of 8 bytes")
    if nin != nout:
        raise InputLengthError("output buffer size mismatch")
    if cfg.backend is Backend.NoOpCopy:
        if pin != pout and nin:
            ctypes.memmove(pout, pin, nin)
        return
    if nin == 0:
        return
    if cfg.workers and cfg.workers > 1:
        # min(workers, GPUs) shards on consecutive GPUs from cfg.device
        # (t3des_cu_ecb_workers)
        _raise(N.lib().t3des_cu_ecb_workers(cfg.workers, cfg.device, ts.sub48(), direction, pin, pout, nin))
        return
    e = engine(cfg.device)
    e.set_schedule(ts)
    e.set_variant(cfg.variant)
    e.set_launch(cfg.chunk_blocks if cfg.gpu_chunked else 0, cfg.work_group if cfg.gpu_chunked else 0)
    e.ecb_host(direction, pin, pout, nin)
    del keep_in, keep_out


class HostRegistration:
    """Opt-in page-locking of a host buffer passed to many batch calls
    (t3des_cu_host_register): the host path then DMAs straight from/to it
    instead of staging it through the engine's pinned ring.  Use as a context
    manager, or call close(); it must be closed before the buffer is freed."""

    def __init__(self, buf):
        p, n, keep = _host_view(buf, False)
        self._keep = keep
        self._p = None
        if n:
            _raise(N.lib().t3des_cu_host_register(p, n), "host register")
            self._p = p

    def close(self) -> None:
        if self._p is not None:
            _raise(N.lib().t3des_cu_host_unregister(self._p), "host unregister")
            self._p = None
            self._keep = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):  # pragma: no cover - best effort; holds the buffer alive until here
        try:
            self.close()
        except Exception:
            pass


def encrypt_batch(src, dst, ts: TripleSchedule, cfg: DispatchConfig | None = None) -> None:
    """ECB-encrypt `src` into `dst` (same length, multiple of 8 bytes;
    in place allowed, partial overlap rejected)."""
    _run_batch(src, dst, ts, cfg or DispatchConfig(), N.ENCRYPT)


def decrypt_batch(src, dst, ts: TripleSchedule, cfg: DispatchConfig | None = None) -> None:
    _run_batch(src, dst, ts, cfg or DispatchConfig(), N.DECRYPT)


# ---- streams (dispatch.hpp:32,71-91) ----------------------

def _one_block(block: int, ts: TripleSchedule, direction: int) -> int:
    buf = bytearray(store_block(block))
    _run_batch(buf, buf, ts, DispatchConfig(), direction)
    return load_block(buf)


def _single(ks) -> TripleSchedule:
    ks = tuple(ks)
    return TripleSchedule(ks, ks, ks)


def encrypt_block(block: int, ks) -> int:
    """des.hpp:37: single DES of one block under a 16-key schedule, as a
    one-block batch through the engine (EDE of (ks, ks, ks))."""
    return _one_block(block, _single(ks), N.ENCRYPT)


def decrypt_block(block: int, ks) -> int:
    """des.hpp:38 (see encrypt_block)."""
    return _one_block(block, _single(ks), N.DECRYPT)


def tdes_encrypt_block(block: int, ts: TripleSchedule) -> int:
    """tdes.hpp:46: one block through the engine (bulk work: encrypt_batch)."""
    return _one_block(block, ts, N.ENCRYPT)


def tdes_decrypt_block(block: int, ts: TripleSchedule) -> int:
    """tdes.hpp:47: one block through the engine (bulk work: decrypt_batch)."""
    return _one_block(block, ts, N.DECRYPT)


tdes_encrypt_block_fast = tdes_encrypt_block  # tdes.hpp:53: the same function
tdes_decrypt_block_fast = tdes_decrypt_block  # tdes.hpp:54


def run_verification(out=None, device: int = 0) -> bool:
    """verify.hpp:37: known answers and structural properties on the GPU
    (t3des_cu_run_verification); writes the report to `out` (default
    sys.stdout) and returns whether every group passed."""
    import sys

    buf = ctypes.create_string_buffer(4096)
    rc = N.lib().t3des_cu_run_verification(device, buf, len(buf))
    (out or sys.stdout).write(buf.value.decode())
    if rc not in (N.OK, N.ERR_ARG):
        _raise(rc)
    return rc == N.OK


class PaddingMode(enum.Enum):
    NONE = 0
    PKCS7 = 1


@dataclass(frozen=True)
class StreamReport:
    bytes_in: int
    bytes_out: int
    chunks: int
    compute_seconds: float
    io_seconds: float


def pkcs7_pad(data: bytes | bytearray) -> bytes:
    pad = 8 - len(data) % 8
    return bytes(data) + bytes([pad]) * pad


def pkcs7_unpad(data: bytes | bytearray) -> bytes:
    if not data or len(data) % 8:
        raise PaddingError("PKCS#7 data length must be a positive multiple of 8")
    pad = data[-1]
    if pad < 1 or pad > 8:
        raise PaddingError("bad PKCS#7 pad value")
    if any(b != pad for b in data[-pad:]):
        raise PaddingError("inconsistent PKCS#7 padding")
    return bytes(data[:-pad])


def _stream(source, sink, ts: TripleSchedule, cfg: DispatchConfig | None, pad: PaddingMode, direction: int):
    """Run t3des_cu_stream_fd.  `source`/`sink` are int file descriptors or
    file-like objects (bridged through OS pipes by two helper threads)."""
    import os
    import threading

    cfg = cfg or DispatchConfig()
    if cfg.backend is not Backend.CUDA:
        raise NotImplementedError("streams run on Backend.CUDA")
    if cfg.chunk_blocks <= 0:
        raise ValueError("chunk_blocks must be positive")
    e = engine(cfg.device)
    e.set_schedule(ts)
    e.set_variant(cfg.variant)
    e.set_launch(0, 0)
    threads, close_fds, errors = [], [], []
    if isinstance(source, int):
        in_fd = source
    else:
        r, w = os.pipe()
        in_fd = r
        close_fds.append(r)

        def feed():
            try:
                while True:
                    b = source.read(1 << 20)
                    if not b:
                        break
                    _write_all(w, b)
            except BrokenPipeError:
                pass
            except Exception as ex:  # surfaced after the engine returns
                errors.append(ex)
            finally:
                os.close(w)

        threads.append(threading.Thread(target=feed, daemon=True))
    if isinstance(sink, int):
        out_fd = sink
    else:
        r2, w2 = os.pipe()
        out_fd = w2

        def drain():
            try:
                while True:
                    b = os.read(r2, 1 << 20)
                    if not b:
                        break
                    sink.write(b)
            except Exception as ex:
                errors.append(ex)
            finally:
                os.close(r2)

        threads.append(threading.Thread(target=drain, daemon=True))
    for t in threads:
        t.start()
    rep = N.StreamReportC()
    try:
        rc = N.lib().t3des_cu_stream_fd(e._h, direction, in_fd, out_fd, cfg.chunk_blocks,
                                        1 if pad is PaddingMode.PKCS7 else 0, ctypes.byref(rep))
    finally:
        if not isinstance(sink, int):
            os.close(out_fd)
        for fd in close_fds:
            os.close(fd)
        for t in threads:
            t.join()
    if errors:
        raise IoError(str(errors[0]), rep.error_offset)
    if rc == N.ERR_IO:
        raise IoError(N.strerror(rc), rep.error_offset)
    _raise(rc)
    return StreamReport(rep.bytes_in, rep.bytes_out, rep.chunks, rep.compute_seconds, rep.io_seconds)


def _write_all(fd: int, b: bytes) -> None:
    import os

    mv = memoryview(b)
    while mv:
        n = os.write(fd, mv)
        mv = mv[n:]


def encrypt_stream(source, sink, ts: TripleSchedule, cfg: DispatchConfig | None = None,
                   pad: PaddingMode = PaddingMode.NONE) -> StreamReport:
    """Chunked ECB encryption of a stream (reference encrypt_stream)."""
    return _stream(source, sink, ts, cfg, pad, N.ENCRYPT)


def decrypt_stream(source, sink, ts: TripleSchedule, cfg: DispatchConfig | None = None,
                   pad: PaddingMode = PaddingMode.NONE) -> StreamReport:
    """Chunked ECB decryption of a stream (reference decrypt_stream)."""
    return _stream(source, sink, ts, cfg, pad, N.DECRYPT)
