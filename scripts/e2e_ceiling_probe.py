#!/usr/bin/env python3
"""Where does the pinned end-to-end path lose against the PCIe ceiling?

For 1 GiB of pinned host memory (in place, as bench.py's e2e), compare:
  copies_only   the engine's stage pattern without the kernel: stage k =
                H2D -> D2H on stream k % S, chunk C (torch copies);
  split_queues  copies on a dedicated H2D stream and a dedicated D2H stream,
                chained by events through a ring of R device buffers;
  engine        t3des_cu_ecb_host with t3des_cu_set_pipeline(C, S);
  bidir         independent H2D and D2H streams of C-sized copies (the
                bench's ceiling, at this chunk size).
All timed with host wall clock around a synchronize (what e2e measures) and
with CUDA events.  Prints one JSON object per configuration.
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
h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
h.random_(0, 255)
hb = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
MAXS = 8


def timed(fn, reps=4):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return round(nbytes / best / 1e9, 2)


def copies_only(C, S, bufs, streams):
    def run():
        for k, off in enumerate(range(0, nbytes, C)):
            n = min(C, nbytes - off)
            s = streams[k % S]
            b = bufs[k % S][:n]
            with torch.cuda.stream(s):
                b.copy_(h[off:off + n], non_blocking=True)
                h[off:off + n].copy_(b, non_blocking=True)
    return run


def split_queues(C, R, bufs, s_in, s_out):
    def run():
        ev_in = [torch.cuda.Event() for _ in range(R)]
        ev_out = [torch.cuda.Event() for _ in range(R)]
        used = [False] * R
        for k, off in enumerate(range(0, nbytes, C)):
            n = min(C, nbytes - off)
            j = k % R
            b = bufs[j][:n]
            if used[j]:
                s_in.wait_event(ev_out[j])
            with torch.cuda.stream(s_in):
                b.copy_(h[off:off + n], non_blocking=True)
                ev_in[j].record(s_in)
            s_out.wait_event(ev_in[j])
            with torch.cuda.stream(s_out):
                h[off:off + n].copy_(b, non_blocking=True)
                ev_out[j].record(s_out)
            used[j] = True
    return run


def bidir(C, d_a, d_b, s1, s2):
    def run():
        for off in range(0, nbytes, C):
            n = min(C, nbytes - off)
            with torch.cuda.stream(s1):
                d_a[:n].copy_(h[off:off + n], non_blocking=True)
            with torch.cuda.stream(s2):
                hb[off:off + n].copy_(d_b[:n], non_blocking=True)
    return run


def main():
    streams = [torch.cuda.Stream() for _ in range(MAXS)]
    e = t3.Engine(0)
    e.set_schedule(t3.triple_schedule(t3.parse_hex_key("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57")))
    e_def = t3.Engine(0)
    e_def.set_schedule(t3.triple_schedule(t3.parse_hex_key("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57")))
    print(json.dumps({"engine_default": timed(lambda: e_def.ecb_host(0, h.data_ptr(), h.data_ptr(), nbytes))}), flush=True)
    d_a = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for C_mib in (8, 16, 32, 64, 128):
        C = C_mib << 20
        bufs = [torch.empty(C, dtype=torch.uint8, device="cuda") for _ in range(MAXS)]
        row = {"chunk_mib": C_mib, "bidir": timed(bidir(C, d_a, d_b, streams[0], streams[1]))}
        for S in (2, 3, 4, 6):
            row[f"copies_only_s{S}"] = timed(copies_only(C, S, bufs, streams))
            row[f"split_queues_r{S}"] = timed(split_queues(C, S, bufs, streams[6], streams[7]))
            e.set_pipeline(C, S)
            row[f"engine_s{S}"] = timed(lambda: e.ecb_host(0, h.data_ptr(), h.data_ptr(), nbytes))
        print(json.dumps(row), flush=True)
        del bufs
    e.close()


if __name__ == "__main__":
    main()
