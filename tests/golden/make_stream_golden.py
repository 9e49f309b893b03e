#!/usr/bin/env python3
"""Generate tests/golden/stream_cases.json: what the UNMODIFIED reference's
encrypt_stream/decrypt_stream (proj/src/dispatch.cpp:111-206, Backend::
Threaded) writes — and which exception it throws — for stream inputs that
exercise the chunk / padding / error edges: bytes written (length + SHA-256),
the exception type, and the StreamReport counters.

Run in the build container (needs /root/reference and oracle/_ref built by
`make -C oracle`); the JSON is committed and the GPU tests
(tests/test_streams.py) compare the engine's fd stream path against it.
Inputs are deterministic: splitmix payload blocks (oracle), ciphertexts made
with the reference's own encrypt_batch.
"""
from __future__ import annotations

import hashlib
import json
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
REF_INC = "/root/reference/proj/include"
KEY = "0123456789ABCDEF23456789ABCDEF01456789ABCDEF0123"

DRIVER = r'''
#include <cstdio>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include "t3des/dispatch.hpp"
#include "t3des/tdes.hpp"
using namespace t3des;
// argv: key dir(e|d) pad(p|n) chunk_blocks in out
int main(int argc, char** argv) {
    const TripleSchedule ts = triple_schedule(parse_hex_key(argv[1]));
    DispatchConfig cfg;
    cfg.backend = Backend::Threaded;
    cfg.chunk_blocks = std::stoul(argv[4]);
    std::ifstream in(argv[5], std::ios::binary);
    std::ofstream out(argv[6], std::ios::binary);
    const PaddingMode pad = argv[3][0] == 'p' ? PaddingMode::Pkcs7 : PaddingMode::None;
    const char* err = "none";
    StreamReport r{};
    try {
        r = argv[2][0] == 'e' ? encrypt_stream(in, out, ts, cfg, pad) : decrypt_stream(in, out, ts, cfg, pad);
    } catch (const InputLengthError&) { err = "InputLengthError"; }
    catch (const PaddingError&) { err = "PaddingError"; }
    catch (const IoError&) { err = "IoError"; }
    out.flush();
    std::printf("%s %llu %llu %llu\n", err, (unsigned long long)r.bytes_in, (unsigned long long)r.bytes_out,
                (unsigned long long)r.chunks);
    return 0;
}
'''


def cases(o):
    """(name, direction, pkcs7, chunk_blocks, input bytes)"""
    import numpy as np

    s = o.schedule_hex(KEY)
    cb = 16
    body = o.splitmix(0, cb * 9, 0x5EED)
    ct = o.ref_ecb(body, s, 0).tobytes()
    bad_pad = body.copy()
    bad_pad[-1] = 0
    ct_bad_pad = o.ref_ecb(bad_pad, s, 0).tobytes()
    padded = body.tobytes() + bytes([8] * 8)
    ct_padded = o.ref_ecb(np.frombuffer(padded, np.uint8), s, 0).tobytes()
    return [
        ("encrypt_pkcs7_exact_chunks", "e", True, cb, body.tobytes()),
        ("encrypt_pkcs7_ragged", "e", True, cb, body.tobytes()[:1000]),
        ("encrypt_pkcs7_empty", "e", True, cb, b""),
        ("encrypt_none_length_error", "e", False, cb, body.tobytes() + b"\x01\x02\x03"),
        ("decrypt_pkcs7_ok", "d", True, cb, ct_padded),
        ("decrypt_pkcs7_bad_padding", "d", True, cb, ct_bad_pad),
        ("decrypt_pkcs7_length_error", "d", True, cb, ct + b"\x01\x02\x03"),
        ("decrypt_none_length_error", "d", False, cb, ct + b"\x01\x02\x03"),
        ("decrypt_pkcs7_empty", "d", True, cb, b""),
    ]


def main() -> None:
    from tests.oracle_util import REF_SO, Oracle

    o = Oracle.load()
    if o.ref is None or not os.path.isdir(REF_INC):
        sys.exit("needs /root/reference and oracle/_ref")
    with tempfile.TemporaryDirectory() as td:
        src = os.path.join(td, "drv.cpp")
        exe = os.path.join(td, "drv")
        with open(src, "w") as f:
            f.write(DRIVER)
        subprocess.check_call(["/usr/bin/g++", "-std=c++20", "-O1", "-I" + REF_INC, src, REF_SO, "-fopenmp",
                               "-Wl,-rpath," + os.path.dirname(REF_SO), "-o", exe])
        rec = {"key": KEY, "generator": "tests/golden/make_stream_golden.py (reference encrypt_stream/decrypt_stream, "
                                        "Backend::Threaded, oracle/_ref)", "cases": {}}
        for name, d, pkcs7, cb, data in cases(o):
            fin, fout = os.path.join(td, "in"), os.path.join(td, "out")
            with open(fin, "wb") as f:
                f.write(data)
            line = subprocess.check_output([exe, KEY, d, "p" if pkcs7 else "n", str(cb), fin, fout], text=True).split()
            with open(fout, "rb") as f:
                got = f.read()
            rec["cases"][name] = {"direction": d, "pkcs7": pkcs7, "chunk_blocks": cb, "input_hex": data.hex(),
                                  "error": line[0], "bytes_in": int(line[1]), "bytes_out": int(line[2]),
                                  "chunks": int(line[3]), "written_len": len(got),
                                  "written_sha256": hashlib.sha256(got).hexdigest()}
    with open(os.path.join(ROOT, "tests", "golden", "stream_cases.json"), "w") as f:
        json.dump(rec, f, indent=1)
        f.write("\n")
    for k, v in rec["cases"].items():
        print(k, v["error"], v["written_len"], v["chunks"])


if __name__ == "__main__":
    main()
