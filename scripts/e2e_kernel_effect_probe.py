#!/usr/bin/env python3
"""Which property of the kernel between H2D and D2H costs the pipelined e2e
path ~7%?  (e2e_timeline_probe: 48.1 GB/s without a kernel, 44.5 with the
bitsliced kernel, in the split-queue pattern as well as the engine's; a
kernel on *other* buffers slows concurrent copies by only ~3%,
copy_interference_probe.)  Split-queue pipeline (H2D stream, kernel stream,
D2H stream, ring of R = 4 buffers of 32 MiB), 1 GiB pinned in place, with:
  none        no kernel
  sleep       torch.cuda._sleep (1 thread spinning ~kernel time): dependency delay only
  bitslice    the engine's kernel in place
  bs_oop      the engine's kernel out of place (D2H from a separate out ring)
  bs_grid1    in place, grid capped at 1 CTA/SM-equivalent (T3DES_BS_CTAS_PER_SM=1)
  torch       elementwise not in place (HBM-bound, short)
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
R = 4
h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
h.random_(0, 255)
KEY = "133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57"
e = t3.Engine(0)
e.set_schedule(t3.triple_schedule(t3.parse_hex_key(KEY)))
e.set_variant(t3.VARIANT_BITSLICE)
os.environ["T3DES_BS_CTAS_PER_SM"] = "1"
e1 = t3.Engine(0)  # created with the grid cap
e1.set_schedule(t3.triple_schedule(t3.parse_hex_key(KEY)))
e1.set_variant(t3.VARIANT_BITSLICE)
del os.environ["T3DES_BS_CTAS_PER_SM"]
ring = [torch.empty(C, dtype=torch.uint8, device="cuda") for _ in range(R)]
oring = [torch.empty(C, dtype=torch.uint8, device="cuda") for _ in range(R)]
s_in, s_k, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
SLEEP_CYCLES = int(1.965e9 * 100e-6)  # ~100 us, the in-pipeline kernel time


def run(kind):
    ev_in = [torch.cuda.Event() for _ in range(R)]
    ev_k = [torch.cuda.Event() for _ in range(R)]
    ev_out = [torch.cuda.Event() for _ in range(R)]
    used = [False] * R
    for k, off in enumerate(range(0, nbytes, C)):
        n = min(C, nbytes - off)
        j = k % R
        b = ring[j][:n]
        o = oring[j][:n] if kind == "bs_oop" else b
        if used[j]:
            s_in.wait_event(ev_out[j])
        with torch.cuda.stream(s_in):
            b.copy_(h[off:off + n], non_blocking=True)
            ev_in[j].record(s_in)
        s_k.wait_event(ev_in[j])
        with torch.cuda.stream(s_k):
            if kind == "sleep":
                torch.cuda._sleep(SLEEP_CYCLES)
            elif kind in ("bitslice", "bs_oop"):
                e.ecb_device(0, b.data_ptr(), o.data_ptr(), n, s_k.cuda_stream)
            elif kind == "bs_grid1":
                e1.ecb_device(0, b.data_ptr(), b.data_ptr(), n, s_k.cuda_stream)
            elif kind == "torch":
                b.bitwise_not_()
            ev_k[j].record(s_k)
        s_out.wait_event(ev_k[j])
        with torch.cuda.stream(s_out):
            h[off:off + n].copy_(o, non_blocking=True)
            ev_out[j].record(s_out)
        used[j] = True


def main():
    for kind in ["none", "sleep", "bitslice", "bs_oop", "bs_grid1", "torch"] * 3:
        run(kind)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            t0 = time.perf_counter()
            run(kind)
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        # kernel alone on one 32 MiB buffer
        ka = None
        if kind not in ("none",):
            a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s_k):
                a.record(s_k)
                for _ in range(10):
                    if kind == "sleep":
                        torch.cuda._sleep(SLEEP_CYCLES)
                    elif kind in ("bitslice", "bs_oop"):
                        e.ecb_device(0, ring[0].data_ptr(), oring[0].data_ptr(), C, s_k.cuda_stream)
                    elif kind == "bs_grid1":
                        e1.ecb_device(0, ring[0].data_ptr(), ring[0].data_ptr(), C, s_k.cuda_stream)
                    elif kind == "torch":
                        ring[0].bitwise_not_()
                b_.record(s_k)
            torch.cuda.synchronize()
            ka = round(a.elapsed_time(b_) / 10 * 1e3, 1)
        print(kind, json.dumps({"GBps": round(nbytes / best / 1e9, 2), "kernel_alone_us": ka}), flush=True)


if __name__ == "__main__":
    main()
