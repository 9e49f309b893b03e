#!/usr/bin/env python3
"""Sustained device-resident encrypt: 4 GiB in place, back to back for
~60 s; every 5 s prints GB/s over the last window (CUDA events) with the
SM clock, power draw, temperature and throttle reasons from NVML."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml  # noqa: E402
import torch  # noqa: E402

import paper_1305_4376_b200 as t3  # noqa: E402

secs = float(os.environ.get("T3_SUSTAIN_S", "60"))
n = (4 << 30) // 8
e = t3.Engine(0)
e.set_schedule(t3.triple_schedule(t3.parse_hex_key("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57")))
buf = torch.empty(8 * n, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
e.fill_splitmix(buf.data_ptr(), 0, n, 0x3DE5C0DE, s)
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
t_end = time.time() + secs
while time.time() < t_end:
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    k = 0
    t0 = time.time()
    while time.time() - t0 < 5.0:
        for _ in range(4):
            e.ecb_device(0, buf.data_ptr(), buf.data_ptr(), 8 * n, s)
        k += 4
        torch.cuda.synchronize()
    b.record()
    torch.cuda.synchronize()
    gbs = k * 8 * n / (a.elapsed_time(b) / 1e3) / 1e9
    clk = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
    pw = pynvml.nvmlDeviceGetPowerUsage(h) / 1000
    tmp = pynvml.nvmlDeviceGetTemperature(h, pynvml.NVML_TEMPERATURE_GPU)
    rs = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
    print(f"{k * 4} GiB in window: {gbs:6.1f} GB/s | SM {clk} MHz | {pw:5.0f} W | {tmp} C | throttle 0x{rs:x}", flush=True)
