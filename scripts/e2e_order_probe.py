#!/usr/bin/env python3
"""e2e_kernel_effect_probe showed that a 1-thread spin kernel (no memory
traffic) between H2D and D2H costs the pipeline as much as the real kernel:
the loss is the dependency delay, i.e. a copy that is blocked on its kernel
holds back later copies queued behind it.  Test the two remedies:
  order L   enqueue H2D L stages ahead of the kernel/D2H of earlier stages
            (split queues: H2D stream, kernel stream, D2H stream; ring R)
  the same under CUDA_DEVICE_MAX_CONNECTIONS=32 (run this script twice).
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_4376_b200 as t3  # noqa: E402

GiB = 1 << 30
nbytes = GiB
C = int(os.environ.get("PROBE_CHUNK_MIB", "32")) << 20
h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
h.random_(0, 255)
KEY = "133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57"
e = t3.Engine(0)
e.set_schedule(t3.triple_schedule(t3.parse_hex_key(KEY)))
e.set_variant(t3.VARIANT_BITSLICE)
RMAX = 8
ring = [torch.empty(C, dtype=torch.uint8, device="cuda") for _ in range(RMAX)]
s_in, s_k, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
per_stage = [torch.cuda.Stream() for _ in range(RMAX)]
SLEEP = int(1.965e9 * 100e-6)


def kern(kind, b, s):
    if kind == "sleep":
        with torch.cuda.stream(s):
            torch.cuda._sleep(SLEEP)
    elif kind == "bitslice":
        e.ecb_device(0, b.data_ptr(), b.data_ptr(), b.numel(), s.cuda_stream)


def split(kind, L, R):
    nst = (nbytes + C - 1) // C
    ev_in = [torch.cuda.Event() for _ in range(R)]
    ev_k = [torch.cuda.Event() for _ in range(R)]
    ev_out = [torch.cuda.Event() for _ in range(R)]
    used = [False] * R
    for k in range(nst + L):
        if k < nst:
            off = k * C
            n = min(C, nbytes - off)
            j = k % R
            if used[j]:
                s_in.wait_event(ev_out[j])
            with torch.cuda.stream(s_in):
                ring[j][:n].copy_(h[off:off + n], non_blocking=True)
                ev_in[j].record(s_in)
            used[j] = True
        q = k - L
        if q >= 0:
            off = q * C
            n = min(C, nbytes - off)
            j = q % R
            b = ring[j][:n]
            s_k.wait_event(ev_in[j])
            kern(kind, b, s_k)
            ev_k[j].record(s_k)
            s_out.wait_event(ev_k[j])
            with torch.cuda.stream(s_out):
                h[off:off + n].copy_(b, non_blocking=True)
                ev_out[j].record(s_out)


def per_stream(kind, L, S):
    """the engine's pattern (stage k on stream k % S: H2D, kernel, D2H), with
    the H2D of stage k enqueued L stages ahead of its kernel + D2H"""
    nst = (nbytes + C - 1) // C
    for k in range(nst + L):
        if k < nst:
            off = k * C
            n = min(C, nbytes - off)
            s = per_stage[k % S]
            with torch.cuda.stream(s):
                ring[k % S][:n].copy_(h[off:off + n], non_blocking=True)
        q = k - L
        if q >= 0:
            off = q * C
            n = min(C, nbytes - off)
            s = per_stage[q % S]
            b = ring[q % S][:n]
            kern(kind, b, s)
            with torch.cuda.stream(s):
                h[off:off + n].copy_(b, non_blocking=True)


def timed(fn):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return round(nbytes / best / 1e9, 2)


def main():
    tag = f"conn={os.environ.get('CUDA_DEVICE_MAX_CONNECTIONS', 'default')}"
    for rep in range(2):
        for kind in ("none", "sleep", "bitslice"):
            row = {"kind": kind, "tag": tag}
            for L in (0, 1, 2):
                row[f"split_L{L}_R6"] = timed(lambda: split(kind, L, 6))
            for L, S in ((0, 3), (1, 3), (1, 4), (2, 4)):
                row[f"perstream_L{L}_S{S}"] = timed(lambda: per_stream(kind, L, S))
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
