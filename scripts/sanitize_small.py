#!/usr/bin/env python3
"""Small driver for compute-sanitizer: every kernel variant on sizes that hit
full tiles, the tail kernel, unaligned (8-byte) buffers, in place, the TMA
prefetch loop (several tiles per warp), and the stream path."""
import io
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_4376_b200 as t3  # noqa: E402
from paper_1305_4376_b200 import _native as N  # noqa: E402

ts = t3.triple_schedule(t3.parse_hex_key("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57"))
e = t3.Engine(0)
e.set_schedule(ts)
s = torch.cuda.current_stream().cuda_stream
variants = [N.VARIANT_AUTO, N.VARIANT_BITSLICE, N.VARIANT_BITSLICE_ALU, N.VARIANT_BITSLICE_LDG, N.VARIANT_SPTABLE]
for v in variants:
    e.set_variant(v)
    for n in (1, 33, 1024, 1025, 8 * 1024 * 40 + 17, 300_000):
        for pad in (0, 8):
            buf = torch.randint(0, 255, (8 * n + pad + 64,), dtype=torch.uint8, device="cuda")
            src = buf[pad:pad + 8 * n]
            out = torch.full((8 * n + 128,), 0xA5, dtype=torch.uint8, device="cuda")
            dst = out[64 + pad:64 + pad + 8 * n]
            guard = out.clone()
            e.ecb_device(0, src.data_ptr(), dst.data_ptr(), 8 * n, s)
            e.ecb_device(1, dst.data_ptr(), dst.data_ptr(), 8 * n, s)
            torch.cuda.synchronize()
            assert torch.equal(dst, src), (v, n, pad)
            assert torch.equal(out[:64 + pad], guard[:64 + pad]) and torch.equal(out[64 + pad + 8 * n:],
                                                                                guard[64 + pad + 8 * n:]), (v, n, pad)
x = bytes(range(256)) * 4000
out = io.BytesIO()
t3.encrypt_stream(io.BytesIO(x), out, ts, t3.DispatchConfig(chunk_blocks=1000), t3.PaddingMode.PKCS7)
back = io.BytesIO()
t3.decrypt_stream(io.BytesIO(out.getvalue()), back, ts, t3.DispatchConfig(chunk_blocks=1000), t3.PaddingMode.PKCS7)
assert back.getvalue() == x
print("sanitize driver ok")
