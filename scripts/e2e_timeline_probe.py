#!/usr/bin/env python3
"""Why does the pinned e2e pipeline run at 45 GB/s when the same stage
pattern without the kernel runs at 48.4 (scripts/e2e_ceiling_probe.py)?

Stage pattern of t3des_cu_ecb_host (3 streams, 32 MiB stages, 1 GiB in place)
rebuilt with torch streams, with a CUDA event after every H2D, kernel and D2H,
for several "kernels" in the middle: none, a torch elementwise pass, the
engine's bitsliced kernel (ecb_device on the stage's stream), the SP-table
kernel.  Prints per-variant rate and the timeline of the first/last stages.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_4376_b200 as t3  # noqa: E402

GiB = 1 << 30
nbytes = int(os.environ.get("PROBE_BYTES", GiB))
C = int(os.environ.get("PROBE_CHUNK_MIB", "32")) << 20
S = int(os.environ.get("PROBE_STREAMS", "3"))
h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
h.random_(0, 255)
streams = [torch.cuda.Stream() for _ in range(S)]
bufs = [torch.empty(C, dtype=torch.uint8, device="cuda") for _ in range(S)]
e = t3.Engine(0)
e.set_schedule(t3.triple_schedule(t3.parse_hex_key("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57")))


def make(kind):
    def kern(b, s):
        if kind == "none":
            return
        if kind == "torch":
            b.bitwise_not_()
        elif kind in ("bitslice", "sptable"):
            e.set_variant(t3.VARIANT_BITSLICE if kind == "bitslice" else t3.VARIANT_SPTABLE)
            e.ecb_device(0, b.data_ptr(), b.data_ptr(), b.numel(), s.cuda_stream)

    def run(evs=None):
        for k, off in enumerate(range(0, nbytes, C)):
            n = min(C, nbytes - off)
            s = streams[k % S]
            b = bufs[k % S][:n]
            with torch.cuda.stream(s):
                b.copy_(h[off:off + n], non_blocking=True)
                if evs is not None:
                    evs[k][0].record(s)
                kern(b, s)
                if evs is not None:
                    evs[k][1].record(s)
                h[off:off + n].copy_(b, non_blocking=True)
                if evs is not None:
                    evs[k][2].record(s)
    return run


def split_run(R, kind="bitslice"):
    """H2D stream, kernel stream, D2H stream chained by events over a ring
    of R buffers (buffer j reused only after its D2H)."""
    s_in, s_k, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    ring = [torch.empty(C, dtype=torch.uint8, device="cuda") for _ in range(R)]

    def run():
        ev_in = [torch.cuda.Event() for _ in range(R)]
        ev_k = [torch.cuda.Event() for _ in range(R)]
        ev_out = [torch.cuda.Event() for _ in range(R)]
        used = [False] * R
        for k, off in enumerate(range(0, nbytes, C)):
            n = min(C, nbytes - off)
            j = k % R
            b = ring[j][:n]
            if used[j]:
                s_in.wait_event(ev_out[j])
            with torch.cuda.stream(s_in):
                b.copy_(h[off:off + n], non_blocking=True)
                ev_in[j].record(s_in)
            s_k.wait_event(ev_in[j])
            if kind != "none":
                e.set_variant(t3.VARIANT_BITSLICE)
                e.ecb_device(0, b.data_ptr(), b.data_ptr(), n, s_k.cuda_stream)
            ev_k[j].record(s_k)
            s_out.wait_event(ev_k[j])
            with torch.cuda.stream(s_out):
                h[off:off + n].copy_(b, non_blocking=True)
                ev_out[j].record(s_out)
            used[j] = True
    return run


def main():
    nst = (nbytes + C - 1) // C
    out = {}
    for R in (3, 4, 6):
        for kind in ("none", "bitslice"):
            run = split_run(R, kind)
            run()
            torch.cuda.synchronize()
            best = 1e9
            for _ in range(4):
                t0 = time.perf_counter()
                run()
                torch.cuda.synchronize()
                best = min(best, time.perf_counter() - t0)
            print(f"split R={R} {kind}", json.dumps({"GBps": round(nbytes / best / 1e9, 2)}), flush=True)
    for kind in ("none", "torch", "bitslice", "sptable"):
        run = make(kind)
        run()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(4):
            t0 = time.perf_counter()
            run()
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(nst)]
        start = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        start.record(streams[0])
        for s in streams[1:]:
            s.wait_event(start)
        run(evs)
        torch.cuda.synchronize()
        tl = [[round(start.elapsed_time(ev), 3) for ev in row] for row in evs]
        out[kind] = {"GBps": round(nbytes / best / 1e9, 2), "total_ms": tl[-1][2],
                     "first_stages_ms[h2d_end,kern_end,d2h_end]": tl[:5], "last_stages": tl[-3:],
                     "kernel_ms_mean": round(sum(r[1] - r[0] for r in tl) / nst, 4),
                     "h2d_gaps_ms": [round(tl[k][0] - tl[k - 1][0], 3) for k in range(1, 8)],
                     "d2h_gaps_ms": [round(tl[k][2] - tl[k - 1][2], 3) for k in range(1, 8)]}
        print(kind, json.dumps(out[kind]), flush=True)
    e.set_pipeline(C, S)
    e.set_variant(t3.VARIANT_AUTO)
    e.ecb_host(0, h.data_ptr(), h.data_ptr(), nbytes)
    best = 1e9
    for _ in range(4):
        t0 = time.perf_counter()
        e.ecb_host(0, h.data_ptr(), h.data_ptr(), nbytes)
        best = min(best, time.perf_counter() - t0)
    print("engine", json.dumps({"GBps": round(nbytes / best / 1e9, 2)}), flush=True)


if __name__ == "__main__":
    main()
