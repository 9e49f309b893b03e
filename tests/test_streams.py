"""Stream path: chunked encrypt_stream/decrypt_stream with
PKCS#7 on the CUDA backend, mirroring the reference's stream tests
(proj/tests/test_dispatch.cpp:187-283) through the Python mirror (C-ABI
t3des_cu_stream_fd) and through the C++ mirror (istream/ostream)."""
import io
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1305_4376_b200 as t3
from paper_1305_4376_b200 import _native as N
from tests.oracle_util import ROOT

KEY = "0123456789ABCDEF23456789ABCDEF01456789ABCDEF0123"  # test_dispatch.cpp:13-14


def test_pkcs7_round_trip_all_lengths():
    rng = np.random.default_rng(46)
    for n in range(65):
        data = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        p = t3.pkcs7_pad(data)
        assert len(p) % 8 == 0 and len(p) > len(data)
        assert t3.pkcs7_unpad(p) == data


def test_pkcs7_unpad_rejects_malformed():
    for bad in (bytes(8), bytes([9]) * 8, bytes([1, 2, 3, 4, 5, 6, 3, 2]), b""):
        with pytest.raises(t3.PaddingError):
            t3.pkcs7_unpad(bad)


CPP_PKCS7 = r'''
#include <cstdio>
#include <vector>
#include "t3des_b200/t3des.hpp"
using namespace t3des;
int main() {
    for (std::size_t n = 0; n <= 64; ++n) {
        std::vector<std::uint8_t> d(n), o;
        for (std::size_t i = 0; i < n; ++i) d[i] = static_cast<std::uint8_t>(i * 37 + 1);
        o = d;
        pkcs7_pad(d);
        if (d.size() % 8 || d.size() <= n) return 2;
        pkcs7_unpad(d);
        if (d != o) return 3;
    }
    std::vector<std::vector<std::uint8_t>> bads = {std::vector<std::uint8_t>(8, 0), std::vector<std::uint8_t>(8, 9),
                                                   {1, 2, 3, 4, 5, 6, 3, 2}, {}};
    for (auto& b : bads) {
        try { pkcs7_unpad(b); return 4; } catch (const PaddingError&) {}
    }
    std::puts("ok");
    return 0;
}
'''


def _build_cpp(tmp_path, src: str, name: str):
    f = tmp_path / f"{name}.cpp"
    f.write_text(src)
    exe = tmp_path / name
    subprocess.check_call(["/usr/bin/g++", "-std=c++20", "-I" + os.path.join(ROOT, "include"), str(f), N.LIB_PATH,
                           "-Wl,-rpath," + os.path.dirname(N.LIB_PATH), "-o", str(exe)])
    return exe


def test_cpp_pkcs7(engine_lib, tmp_path):
    exe = _build_cpp(tmp_path, CPP_PKCS7, "pk")
    assert subprocess.run([str(exe)], capture_output=True, text=True).stdout.strip() == "ok"


# ---- GPU ------------------------------------------------------------------

@pytest.fixture(scope="module")
def ts():
    return t3.triple_schedule(t3.parse_hex_key(KEY))


@pytest.mark.gpu
def test_empty_stream_no_padding(ts):
    out = io.BytesIO()
    r = t3.encrypt_stream(io.BytesIO(b""), out, ts, t3.DispatchConfig(), t3.PaddingMode.NONE)
    assert (r.bytes_in, r.bytes_out, r.chunks) == (0, 0, 0)
    assert out.getvalue() == b""


@pytest.mark.gpu
def test_stream_round_trip_pkcs7_across_chunks(ts, oracle):
    cfg = t3.DispatchConfig(chunk_blocks=16)
    s = oracle.schedule_hex(KEY)
    rng = np.random.default_rng(47)
    for n in (0, 1, 7, 8, 127, 128, 129, 1000, 16 * 8 * 3):
        payload = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        mid = io.BytesIO()
        t3.encrypt_stream(io.BytesIO(payload), mid, ts, cfg, t3.PaddingMode.PKCS7)
        ct = mid.getvalue()
        assert len(ct) % 8 == 0 and len(ct) > n
        assert ct == oracle.ecb(np.frombuffer(t3.pkcs7_pad(payload), np.uint8), s, 0).tobytes()
        out = io.BytesIO()
        t3.decrypt_stream(io.BytesIO(ct), out, ts, cfg, t3.PaddingMode.PKCS7)
        assert out.getvalue() == payload, n


@pytest.mark.gpu
def test_stream_none_padding_requires_multiple_of_8(ts):
    with pytest.raises(t3.InputLengthError):
        t3.encrypt_stream(io.BytesIO(b"x" * 9), io.BytesIO(), ts)
    with pytest.raises(t3.InputLengthError):
        t3.decrypt_stream(io.BytesIO(b"123456789"), io.BytesIO(), ts)


@pytest.mark.gpu
def test_stream_report_counts(ts):
    payload = b"a" * (1 << 20)  # 131072 blocks = one default chunk
    out = io.BytesIO()
    r = t3.encrypt_stream(io.BytesIO(payload), out, ts)
    assert (r.bytes_in, r.bytes_out, r.chunks) == (len(payload), len(payload), 1)
    assert len(out.getvalue()) == len(payload)


@pytest.mark.gpu
def test_stream_decrypt_round_trip_no_padding_and_fds(ts, oracle, tmp_path):
    x = np.random.default_rng(48).integers(0, 256, 4096, dtype=np.uint8).tobytes()
    cfg = t3.DispatchConfig(chunk_blocks=64)
    enc = io.BytesIO()
    t3.encrypt_stream(io.BytesIO(x), enc, ts, cfg)
    assert enc.getvalue() == oracle.ecb(np.frombuffer(x, np.uint8), oracle.schedule_hex(KEY), 0).tobytes()
    dec = io.BytesIO()
    t3.decrypt_stream(io.BytesIO(enc.getvalue()), dec, ts, cfg)
    assert dec.getvalue() == x
    # raw file descriptors, many chunks, the output equals the batch path
    big = np.random.default_rng(49).integers(0, 256, 8 * 100_003, dtype=np.uint8)
    src, dst = tmp_path / "in.bin", tmp_path / "out.bin"
    big.tofile(src)
    with open(src, "rb") as fi, open(dst, "wb") as fo:
        r = t3.encrypt_stream(fi.fileno(), fo.fileno(), ts, t3.DispatchConfig(chunk_blocks=4096))
    assert r.chunks == -(-100_003 // 4096) and r.bytes_out == big.nbytes
    assert dst.read_bytes() == oracle.ecb(big, oracle.schedule_hex(KEY), 0).tobytes()


@pytest.mark.gpu
def test_stream_padding_errors(ts):
    with pytest.raises(t3.PaddingError):
        t3.decrypt_stream(io.BytesIO(b""), io.BytesIO(), ts, pad=t3.PaddingMode.PKCS7)
    ct = io.BytesIO()
    t3.encrypt_stream(io.BytesIO(bytes(16)), ct, ts)  # no padding inside
    with pytest.raises(t3.PaddingError):
        t3.decrypt_stream(io.BytesIO(ct.getvalue()), io.BytesIO(), ts, pad=t3.PaddingMode.PKCS7)


CPP_STREAMS = r'''
#include <cstdio>
#include <sstream>
#include <string>
#include "t3des_b200/t3des.hpp"
using namespace t3des;
int main() {
    const auto ts = triple_schedule(parse_hex_key("0123456789ABCDEF23456789ABCDEF01456789ABCDEF0123"));
    DispatchConfig cfg;
    cfg.chunk_blocks = 16;
    for (std::size_t len : {0ul, 1ul, 7ul, 8ul, 127ul, 128ul, 129ul, 1000ul}) {
        std::string payload(len, '\0');
        for (std::size_t i = 0; i < len; ++i) payload[i] = static_cast<char>(i * 131 + 7);
        std::istringstream in(payload);
        std::ostringstream mid;
        encrypt_stream(in, mid, ts, cfg, PaddingMode::Pkcs7);
        if (mid.str().size() % 8 || mid.str().size() <= len) return 2;
        std::istringstream back(mid.str());
        std::ostringstream out;
        decrypt_stream(back, out, ts, cfg, PaddingMode::Pkcs7);
        if (out.str() != payload) return 3;
    }
    {
        std::istringstream in(std::string(9, 'x'));
        std::ostringstream out;
        try { encrypt_stream(in, out, ts, DispatchConfig{}, PaddingMode::None); return 4; }
        catch (const InputLengthError&) {}
    }
    {
        const std::string payload(1 << 20, 'a');
        std::istringstream in(payload);
        std::ostringstream out;
        const StreamReport r = encrypt_stream(in, out, ts, DispatchConfig{}, PaddingMode::None);
        if (r.bytes_in != payload.size() || r.bytes_out != payload.size() || r.chunks != 1) return 5;
        std::fwrite(out.str().data(), 1, out.str().size(), stdout);
    }
    return 0;
}
'''


@pytest.mark.gpu
def test_cpp_streams_on_device(engine_lib, oracle, tmp_path):
    exe = _build_cpp(tmp_path, CPP_STREAMS, "st")
    p = subprocess.run([str(exe)], capture_output=True)
    assert p.returncode == 0, p.stderr
    want = oracle.ecb(np.frombuffer(b"a" * (1 << 20), np.uint8), oracle.schedule_hex(KEY), 0).tobytes()
    assert p.stdout == want


@pytest.mark.gpu
def test_stream_on_a_non_current_device(ts, oracle):
    """encrypt_stream on device D while the caller's current device is 0: the
    stream path opens a device scope.  Needs two GPUs."""
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs a second GPU")
    torch.cuda.set_device(0)
    payload = np.random.default_rng(49).integers(0, 256, 5000, dtype=np.uint8).tobytes()
    mid = io.BytesIO()
    t3.encrypt_stream(io.BytesIO(payload), mid, ts, t3.DispatchConfig(device=1, chunk_blocks=100), t3.PaddingMode.PKCS7)
    assert mid.getvalue() == oracle.ecb(np.frombuffer(t3.pkcs7_pad(payload), np.uint8), oracle.schedule_hex(KEY), 0).tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("io_mib", [None, "1"])
def test_regular_file_streams_keep_reference_chunk_semantics(ts, oracle, tmp_path, monkeypatch, io_mib):
    """The fd entry on regular files (parallel pread/pwrite, I/O pieces of many
    reference chunks): same bytes, the reference's chunk count, and on a
    padding error exactly the chunks the reference writes before throwing
    (every chunk but the last)."""
    if io_mib:
        monkeypatch.setenv("T3DES_STREAM_IO_MIB", io_mib)
    s = oracle.schedule_hex(KEY)
    cb = 64  # 512-byte reference chunks
    rng = np.random.default_rng(51)
    for n in (0, 8, 4096, 3 << 20, (3 << 20) + 5):
        payload = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        src, mid, out = tmp_path / "in", tmp_path / "mid", tmp_path / "out"
        src.write_bytes(payload)
        with open(src, "rb") as fi, open(mid, "wb") as fo:
            r = t3.encrypt_stream(fi.fileno(), fo.fileno(), ts, t3.DispatchConfig(chunk_blocks=cb), t3.PaddingMode.PKCS7)
            assert fi.tell() == n and fo.tell() == len(t3.pkcs7_pad(payload))  # offsets as sequential I/O leaves them
        padded = t3.pkcs7_pad(payload)
        assert mid.read_bytes() == oracle.ecb(np.frombuffer(padded, np.uint8), s, 0).tobytes()
        assert r.chunks == max(1, -(-n // (8 * cb))) and r.bytes_in == n and r.bytes_out == len(padded)
        with open(mid, "rb") as fi, open(out, "wb") as fo:
            t3.decrypt_stream(fi.fileno(), fo.fileno(), ts, t3.DispatchConfig(chunk_blocks=cb), t3.PaddingMode.PKCS7)
        assert out.read_bytes() == payload
    # bad padding: a multi-chunk ciphertext whose plaintext ends without padding
    body = rng.integers(0, 256, 8 * cb * 37 + 8 * 5, dtype=np.uint8)
    body[-1] = 0  # pad byte 0 is invalid
    ct = oracle.ecb(body, s, 0).tobytes()
    src.write_bytes(ct)
    with open(src, "rb") as fi, open(out, "wb") as fo:
        with pytest.raises(t3.PaddingError):
            t3.decrypt_stream(fi.fileno(), fo.fileno(), ts, t3.DispatchConfig(chunk_blocks=cb), t3.PaddingMode.PKCS7)
    written = out.read_bytes()
    assert written == body[: 8 * cb * 37].tobytes()  # the 37 full chunks before the last (5-block) one


@pytest.mark.gpu
def test_decrypt_length_error_output_matches_reference(ts, oracle, tmp_path):
    """A ciphertext whose length is not a multiple of 8, PKCS#7 decrypt: the
    reference (dispatch.cpp:111-206) holds each decrypted chunk back until
    the next is read, so when the short last chunk throws InputLengthError
    it has written every chunk but the last two."""
    s = oracle.schedule_hex(KEY)
    cb = 16
    body = np.random.default_rng(52).integers(0, 256, 8 * cb * 9, dtype=np.uint8)
    ct = oracle.ecb(body, s, 0).tobytes() + b"\x01\x02\x03"  # 9 full chunks + 3 stray bytes
    src, out = tmp_path / "ct", tmp_path / "pt"
    src.write_bytes(ct)
    with open(src, "rb") as fi, open(out, "wb") as fo:
        with pytest.raises(t3.InputLengthError):
            t3.decrypt_stream(fi.fileno(), fo.fileno(), ts, t3.DispatchConfig(chunk_blocks=cb), t3.PaddingMode.PKCS7)
    assert out.read_bytes() == body[: 8 * cb * 8].tobytes()
    with open(src, "rb") as fi, open(out, "wb") as fo:  # without padding: every full chunk
        with pytest.raises(t3.InputLengthError):
            t3.decrypt_stream(fi.fileno(), fo.fileno(), ts, t3.DispatchConfig(chunk_blocks=cb), t3.PaddingMode.NONE)
    assert out.read_bytes() == body.tobytes()


def _golden_stream_cases():
    import json

    with open(os.path.join(ROOT, "tests", "golden", "stream_cases.json")) as f:
        return json.load(f)


@pytest.mark.gpu
@pytest.mark.parametrize("via", ["regular_fd", "pipe"])
def test_streams_match_reference_outputs_and_errors(tmp_path, via):
    """Every case of tests/golden/stream_cases.json — what the reference's own
    encrypt_stream/decrypt_stream writes and throws (make_stream_golden.py) —
    through the engine's fd path on regular files (parallel I/O, large I/O
    pieces) and through pipes (chunk-by-chunk): same bytes written, same
    exception type, and on success the reference's StreamReport counters."""
    import hashlib

    gold = _golden_stream_cases()
    ts = t3.triple_schedule(t3.parse_hex_key(gold["key"]))
    errs = {"InputLengthError": t3.InputLengthError, "PaddingError": t3.PaddingError}
    for name, c in gold["cases"].items():
        data = bytes.fromhex(c["input_hex"])
        cfg = t3.DispatchConfig(chunk_blocks=c["chunk_blocks"])
        pad = t3.PaddingMode.PKCS7 if c["pkcs7"] else t3.PaddingMode.NONE
        fn = t3.encrypt_stream if c["direction"] == "e" else t3.decrypt_stream
        out = tmp_path / f"{name}.out"
        err, rep = "none", None
        try:
            if via == "regular_fd":
                src = tmp_path / f"{name}.in"
                src.write_bytes(data)
                with open(src, "rb") as fi, open(out, "wb") as fo:
                    rep = fn(fi.fileno(), fo.fileno(), ts, cfg, pad)
            else:
                with open(out, "wb") as fo:
                    rep = fn(io.BytesIO(data), fo, ts, cfg, pad)
        except (t3.InputLengthError, t3.PaddingError) as exc:
            err = next(k for k, v in errs.items() if isinstance(exc, v))
        got = out.read_bytes()
        assert err == c["error"], name
        assert len(got) == c["written_len"] and hashlib.sha256(got).hexdigest() == c["written_sha256"], name
        if err == "none":
            assert (rep.bytes_in, rep.bytes_out, rep.chunks) == (c["bytes_in"], c["bytes_out"], c["chunks"]), name


STREAM_FAULT_CHILD = r'''
import io, sys
sys.path.insert(0, sys.argv[1])
import numpy as np
import paper_1305_4376_b200 as t3
from tests.oracle_util import Oracle
o = Oracle.load()
key = "0123456789ABCDEF23456789ABCDEF01456789ABCDEF0123"
ts = t3.triple_schedule(t3.parse_hex_key(key))
cb = 16
body = np.random.default_rng(53).integers(0, 256, 8 * cb * 10, dtype=np.uint8)
out = io.BytesIO()
try:
    t3.encrypt_stream(io.BytesIO(body.tobytes()), out, ts, t3.DispatchConfig(chunk_blocks=cb), t3.PaddingMode.NONE)
    raise SystemExit("no error")
except t3.CudaError:
    pass
want = o.ecb(body[: 8 * cb * 3], o.schedule_hex(key), 0).tobytes()
assert out.getvalue() == want, (len(out.getvalue()), len(want))
print("ok")
'''


@pytest.mark.gpu
def test_stream_gpu_failure_writes_the_chunks_before_it():
    """A GPU failure at chunk 3 of a stream (fault injection,
    T3DES_FAULT_AT_STAGE) surfaces as CudaError after the three earlier
    chunks have been written, like the reference's stream errors."""
    env = dict(os.environ, T3DES_FAULT_AT_STAGE="3")
    p = subprocess.run([sys.executable, "-c", STREAM_FAULT_CHILD, ROOT], capture_output=True, text=True, env=env,
                       timeout=300)
    assert p.returncode == 0 and p.stdout.strip().endswith("ok"), p.stdout + p.stderr
