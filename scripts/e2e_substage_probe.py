#!/usr/bin/env python3
"""Two last questions on the pinned e2e pipeline (scripts/e2e_order_probe.py:
any ~100 us dependency between a stage's H2D and its D2H costs ~7%, whatever
the enqueue order or connection count):
  1. does the SM clock sag while the pipeline runs (NVML, 1 ms sampling)?
  2. does splitting each 32 MiB stage's kernel + D2H into P sub-stages (kernel
     on 32/P MiB, then its D2H, same stream) shorten the D2H engine's wait?
"""
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1305_4376_b200 as t3  # noqa: E402

GiB = 1 << 30
nbytes = GiB
C = 32 << 20
S = 3
h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
h.random_(0, 255)
e = t3.Engine(0)
e.set_schedule(t3.triple_schedule(t3.parse_hex_key("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57")))
e.set_variant(t3.VARIANT_BITSLICE)
streams = [torch.cuda.Stream() for _ in range(S)]
bufs = [torch.empty(C, dtype=torch.uint8, device="cuda") for _ in range(S)]


def run(P, kernel=True):
    sub = C // P
    for k, off in enumerate(range(0, nbytes, C)):
        n = min(C, nbytes - off)
        s = streams[k % S]
        b = bufs[k % S]
        with torch.cuda.stream(s):
            b[:n].copy_(h[off:off + n], non_blocking=True)
            for p in range(0, n, sub):
                m = min(sub, n - p)
                if kernel:
                    e.ecb_device(0, b.data_ptr() + p, b.data_ptr() + p, m, s.cuda_stream)
                h[off + p:off + p + m].copy_(b[p:p + m], non_blocking=True)


class Clk:
    def __init__(self):
        import pynvml

        pynvml.nvmlInit()
        self.p = pynvml
        self.h = pynvml.nvmlDeviceGetHandleByIndex(int(os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0] or 0))
        self.s = []
        self.stop = False

    def loop(self):
        while not self.stop:
            self.s.append(self.p.nvmlDeviceGetClockInfo(self.h, self.p.NVML_CLOCK_SM))
            time.sleep(0.001)


def main():
    for P in (1, 2, 4, 8):
        for kernel in (False, True):
            f = lambda: run(P, kernel)  # noqa: E731
            f()
            torch.cuda.synchronize()
            clk = Clk()
            th = threading.Thread(target=clk.loop)
            th.start()
            best = 1e9
            for _ in range(10):
                t0 = time.perf_counter()
                f()
                torch.cuda.synchronize()
                best = min(best, time.perf_counter() - t0)
            clk.stop = True
            th.join()
            sm = sorted(clk.s)
            print(json.dumps({"P": P, "kernel": kernel, "GBps": round(nbytes / best / 1e9, 2),
                              "sm_mhz_min_med_max": [sm[0], sm[len(sm) // 2], sm[-1]]}), flush=True)
    e.set_pipeline(C, S)
    e.set_variant(t3.VARIANT_AUTO)
    best = 1e9
    for _ in range(6):
        t0 = time.perf_counter()
        e.ecb_host(0, h.data_ptr(), h.data_ptr(), nbytes)
        best = min(best, time.perf_counter() - t0)
    print(json.dumps({"engine": round(nbytes / best / 1e9, 2)}), flush=True)


if __name__ == "__main__":
    main()
