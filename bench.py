#!/usr/bin/env python3
"""Benchmark of the B200 3DES-ECB engine (BASELINE.json metric:
"3DES-ECB encrypt GB/s (1 and 8 B200) and % of LOP3-issue roofline").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one pass of the hot path over one batch, ECB-encrypt under the
bench key of the reference harness (bench.cpp:15-16):
  N = 1  BASELINE configs[1]: 1 GiB (134,217,728 blocks) device-resident;
  N > 1  BASELINE configs[3]: 64 GiB (8,589,934,592 blocks) split into N
         contiguous block ranges (t3des_cu_shard_range), one rank per GPU,
         each rank generating its own range of the one global payload on its
         device (strong scaling; no data-path collective — the only
         collectives are the timing barrier, the max over ranks and the
         gather of the per-shard checksums, whose sum must equal the
         reference's checksum of the whole 64 GiB ciphertext,
         tests/golden/c3_checksum.json).
`--gpus N` without torchrun re-launches itself under torch.distributed.run
with N ranks; a run whose WORLD_SIZE differs from --gpus exits non-zero.

value  = whole-job GB/s (decimal) from CUDA events on the launch stream,
         inputs resident in HBM (>= 1 GiB per rank per step > 126 MB L2, so no
         flush);
e2e    = the same metric through the C ABI's host-buffer entry
         (t3des_cu_ecb_host: pinned H2D -> kernel -> D2H inside the timing),
         next to its ceiling (pinned copy rates measured with CUDA events) and
         the pageable-span path a reference caller's std::vector takes;
roofline = the LOP3-issue roofline of SURVEY.md §8d: W_alg = 402 lane-ops
         per block; peak = SMs x 64 lane-ops/clk x sm_max_mhz.
cpu_baseline = the reference's own OpenMP CPU path (oracle/_ref, Backend::
         Threaded) on the full 1 GiB, all host threads and 1 thread, rank 0 at
         N=1.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BENCH_KEY = "133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57"
METRIC = "3DES-ECB encrypt GB/s (1 and 8 B200) and % of LOP3-issue roofline"
W_ALG = 402.0  # LOP3 lane-ops per block (fixed yardstick)
ALU_LANES_PER_CLK_PER_SM = 64
SEED = 0x3DE5C0DE


def env_int(name: str, default: int) -> int:
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def measured_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region via NVML
    (every ~2 ms in a thread; nvidia-smi's 100 ms floor would see a 30 ms
    region only once)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, device: int):
        self.device = device
        self.samples: list[tuple[float, float, int]] = []
        self._stop = threading.Event()
        self._t = None
        self._nvml = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = None
            try:  # CUDA and NVML orderings can differ: match by UUID
                import torch

                uuid = str(torch.cuda.get_device_properties(self.device).uuid)
                h = pynvml.nvmlDeviceGetHandleByUUID(("GPU-" + uuid) if not uuid.startswith("GPU-") else uuid)
            except Exception:
                vis = os.environ.get("CUDA_VISIBLE_DEVICES")
                idx = int(vis.split(",")[self.device]) if vis else self.device
                h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self._nvml = (pynvml, h)
            self._ready = threading.Event()
            self._t = threading.Thread(target=self._loop, daemon=True)
            self._t.start()
            # the sampler's first NVML queries can take longer than a short
            # timed region (one fresh box gave 0 samples over 54 ms): start
            # timing only once it is sampling
            self._ready.wait(timeout=5.0)
            self.samples.clear()
        except Exception:
            self._nvml = None
        return self

    def _loop(self):
        pynvml, h = self._nvml
        try:
            mx = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
        except Exception:
            mx = float("nan")
        while not self._stop.is_set():
            try:
                sm = float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                rs = int(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h))
                self.samples.append((sm, mx, rs))
            except Exception:
                pass
            self._ready.set()
            time.sleep(0.002)

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=2)
        if self._nvml and not self.samples:  # still none: one read as the region ends
            pynvml, h = self._nvml
            try:
                self.samples.append((float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)),
                                     float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)),
                                     int(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h))))
            except Exception:
                pass

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "source": "unavailable"}
        sm = sorted(x[0] for x in self.samples)
        reasons = sorted({n for _, _, r in self.samples for n, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(x[1] for x in self.samples), "sm_min_mhz": sm[0],
                "reasons": reasons, "samples": len(sm), "source": "nvml"}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def golden_c3() -> dict | None:
    """Reference checksums of the configs[3] payload/ciphertext
    (tests/golden/c3_checksum.json, made by tests/golden/make_c3_checksum.py
    with the reference's own encrypt_batch)."""
    try:
        with open(os.path.join(ROOT, "tests", "golden", "c3_checksum.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


class CpuRef:
    """The reference's own CPU implementation of the path: oracle/_ref
    (encrypt_batch, Backend::Threaded, OpenMP) when it was compiled, else the
    C restatement (oracle/liboracle.so, fused route, OpenMP) — test/baseline
    infrastructure, only ever timed here, never the product."""

    def __init__(self):
        from tests.oracle_util import Oracle

        self.o = Oracle.load()
        self.s = self.o.schedule_hex(BENCH_KEY)
        self.kind = "reference" if self.o.ref is not None else "port"

    @staticmethod
    def all_threads() -> int:
        # explicit, not the reference's workers = 0: that resolves through
        # omp_get_max_threads(), which torchrun pins to 1 (OMP_NUM_THREADS=1)
        try:
            return len(os.sched_getaffinity(0))
        except AttributeError:  # pragma: no cover
            return os.cpu_count() or 1

    def threads(self, workers: int) -> int:
        return workers or self.all_threads()

    def payload(self, nbytes: int):
        # the first nbytes of the bench's global payload (block i =
        # splitmix64(seed ^ i), big-endian) — the same bytes our arm encrypts
        return self.o.splitmix(0, nbytes // 8, SEED)

    def encrypt(self, buf, out, workers: int) -> float:
        workers = self.threads(workers)
        t0 = time.perf_counter()
        if self.o.ref is not None:
            rc = self.o.ref.ref_ecb(buf.ctypes.data, out.ctypes.data, buf.nbytes, self.s, 0, 1, workers, 0, 0)
        else:
            rc = self.o.lib.oracle_ecb(buf.ctypes.data, out.ctypes.data, buf.nbytes, self.s, 0, 1, workers)
        dt = time.perf_counter() - t0
        assert rc == 0, rc
        return dt

    def what(self) -> str:
        return ("reference encrypt_batch, Backend::Threaded (oracle/_ref, -O3 -DNDEBUG -fopenmp), "
                "chunk_blocks 131072, work_group 256" if self.kind == "reference" else
                "C restatement of the reference (oracle/liboracle.so, fused SP route, OpenMP)")


def cpu_reference_arm(full_bytes: int = 1 << 30, one_thread_bytes: int = 64 << 20) -> dict:
    """SURVEY §8d CPU rows: the full 1 GiB configs[1] payload on all host
    threads (1 warm-up + min of 3, as the reference harness, bench.cpp:97-109),
    and workers = 1 on a bounded sample (1 warm-up + min of 2)."""
    import numpy as np

    r = CpuRef()
    buf = r.payload(full_bytes)
    out = np.empty_like(buf)
    r.encrypt(buf, out, 0)  # warm-up (threads, page faults of `out`)
    best = min(r.encrypt(buf, out, 0) for _ in range(3))
    cores = r.threads(0)
    small, sout = buf[:one_thread_bytes], out[:one_thread_bytes]
    r.encrypt(small[: 8 << 20], sout[: 8 << 20], 1)
    best1 = min(r.encrypt(small, sout, 1) for _ in range(2))
    return {
        "value": round(full_bytes / best / 1e9, 4), "unit": "GB/s", "cores": cores, "kind": r.kind,
        "sample": f"encrypt of the full {full_bytes >> 20} MiB configs[1] payload (the bench's splitmix stream, "
                  f"bench key), {r.what()}, workers={cores} (all host threads), 1 warm-up + min of 3",
        "cpu_model": cpu_model(), "host_threads": os.cpu_count(),
        "workers_1": {"value": round(one_thread_bytes / best1 / 1e9, 4), "unit": "GB/s", "cores": 1,
                      "sample": f"first {one_thread_bytes >> 20} MiB of the same payload, workers=1, "
                                "1 warm-up (8 MiB) + min of 2"},
    }


def run_reference_impl(args, rank: int, world: int) -> None:
    """--impl reference: the reference's CPU path on this box's host cores,
    rank 0 only (other ranks exit without work).  Each step encrypts the
    first 1 GiB of the workload's payload with all host threads (at N = 1 that
    is the whole configs[1] batch; at N > 1 a 1 GiB sample of the 64 GiB
    configs[3] stream — 64 GiB would take ~3 min per step on 16 threads)."""
    if rank != 0:
        return
    import numpy as np

    r = CpuRef()
    nbytes = 1 << 30
    buf = r.payload(nbytes)
    out = np.empty_like(buf)
    for _ in range(args.warmup):
        r.encrypt(buf, out, 0)
    times = [r.encrypt(buf, out, 0) for _ in range(args.steps)]
    gbs = args.steps * nbytes / sum(times) / 1e9
    cores = r.threads(0)
    sample = (f"{'whole' if world == 1 else 'sample of the'} workload: encrypt of {nbytes >> 20} MiB (the first GiB "
              f"of the bench's splitmix stream, bench key) per step, {r.what()}, workers={cores} (all host threads); "
              f"value = {args.steps} steps x {nbytes >> 20} MiB / their total time (best step "
              f"{nbytes / min(times) / 1e9:.4f} GB/s); cpu: {cpu_model()}")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gbs, 4), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * sum(times) / args.steps, 3),
        "higher_is_better": True, "scaling": "weak" if world == 1 else "strong",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": workload_config(args, world),
        "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": cores, "kind": r.kind, "sample": sample},
        "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def executed_alu_ops_per_block() -> float:
    """ALU-pipe lane-ops per block of the shipped bitsliced kernel: 48 rounds x
    (S-box LOP3 total + 32 Feistel/key LOP3) / 32 blocks per slice, plus four
    32x32 slice transposes (64 PRMT + 96 LOP3 + 48 SHF each) / 32 blocks.  The
    16 E-duplicate corrections and the whitening run on the FMA pipe."""
    import re

    with open(os.path.join(ROOT, "paper_1305_4376_b200", "csrc", "generated", "bitslice_rounds.cuh")) as f:
        total = int(re.search(r"T3_SBOX_LOP3_TOTAL (\d+)", f.read()).group(1))
    return round(48 * (total + 32) / 32 + 4 * (64 + 96 + 48) / 32, 2)



def pcie_ceiling(torch, nbytes: int = 256 << 20, iters: int = 8) -> dict:
    """Pinned host <-> device copy rates, the ceiling of the e2e number:
    H2D alone, D2H alone, and both directions at once on two streams (each
    `iters` x nbytes), timed with CUDA events on the copy streams."""
    h_in = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d_a = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def run(h2d: bool, d2h: bool) -> float:
        torch.cuda.synchronize()
        start, e1, e2 = ev(), ev(), ev()
        start.record(s1)
        s2.wait_event(start)
        for _ in range(iters):
            if h2d:
                with torch.cuda.stream(s1):
                    d_a.copy_(h_in, non_blocking=True)
            if d2h:
                with torch.cuda.stream(s2):
                    h_out.copy_(d_b, non_blocking=True)
        e1.record(s1)
        e2.record(s2)
        torch.cuda.synchronize()
        ms = max(start.elapsed_time(e1) if h2d else 0.0, start.elapsed_time(e2) if d2h else 0.0)
        return iters * nbytes / (ms * 1e-3) / 1e9

    run(True, True)  # warm-up
    out = {"h2d_gbs": round(run(True, False), 2), "d2h_gbs": round(run(False, True), 2),
           "bidir_gbs_each_way": round(run(True, True), 2),
           "how": f"{iters} x {nbytes >> 20} MiB pinned copies per direction, CUDA events on the copy streams"}
    del h_in, h_out, d_a, d_b
    return out


def self_launch(args) -> int | None:
    """--gpus N > 1 outside torchrun: re-run this script under
    torch.distributed.run with N ranks (one per GPU) on 127.0.0.1."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    import socket
    import subprocess

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def bind_to_gpu_cpus(device: int) -> dict:
    """Pin this rank's threads to the CPUs NVML reports as local to its GPU
    (the GPU's NUMA node), so its pinned staging, copy threads and PCIe
    traffic stay on one socket.  Returns what was done."""
    try:
        import pynvml
        import torch

        pynvml.nvmlInit()
        uuid = str(torch.cuda.get_device_properties(device).uuid)
        h = pynvml.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = {64 * w + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1}
        cpus &= os.sched_getaffinity(0)
        if not cpus or cpus == os.sched_getaffinity(0):
            return {"bound": False, "cpus": len(os.sched_getaffinity(0)), "why": "GPU is local to every allowed CPU"}
        os.sched_setaffinity(0, cpus)
        return {"bound": True, "cpus": len(cpus)}
    except Exception as exc:  # NVML absent or no affinity info
        return {"bound": False, "why": type(exc).__name__}


def u64_to_i64(x: int) -> int:
    return x - (1 << 64) if x >= (1 << 63) else x


def nist_kat_ok(t3) -> bool:
    pt = bytes.fromhex("54686520717566636B2062726F776E20666F78206A756D70")
    ct = bytearray(len(pt))
    t3.encrypt_batch(pt, ct, t3.triple_schedule(t3.parse_hex_key("0123456789ABCDEF23456789ABCDEF01456789ABCDEF0123")))
    return ct.hex().upper() == "A826FD8CE53B855FCCE21C8112256FE668D5C05DD9B6B900"


def cross_check(e, N, torch, src, dst, nblocks, stream, variant) -> bool:
    """Bitsliced output vs the SP-table kernel (an independent implementation)
    on every 4096th block, and the decrypt round trip, on the bench payload."""
    idx = torch.arange(0, nblocks, max(1, nblocks // 4096), device="cuda")
    sample_in = src.view(torch.int64)[idx].contiguous()
    e.set_variant(variant)
    e.ecb_device(0, src.data_ptr(), dst.data_ptr(), 8 * nblocks, stream)
    torch.cuda.synchronize()
    got = dst.view(torch.int64)[idx].contiguous()
    ref = torch.empty_like(sample_in)
    e.set_variant(N.VARIANT_SPTABLE)
    e.ecb_device(0, sample_in.data_ptr(), ref.data_ptr(), 8 * ref.numel(), stream)
    e.set_variant(variant)
    torch.cuda.synchronize()
    cs_in = e.checksum(src.data_ptr(), 0, nblocks, stream)
    e.ecb_device(1, dst.data_ptr(), dst.data_ptr(), 8 * nblocks, stream)
    ok = bool(torch.equal(got, ref)) and e.checksum(dst.data_ptr(), 0, nblocks, stream) == cs_in
    return ok



def extra_configs(e, t3, N, torch, np) -> dict:
    """The other BASELINE.json configs, each checked before it is timed:
    [0] 1 MiB encrypt+decrypt, 3 distinct keys, NIST KAT;
    [2] 4 GiB decrypt, device-resident and end to end;
    [4] edge cases (option 3 = single DES, option 2, odd tails) — parity only."""
    out = {}
    stream = torch.cuda.current_stream().cuda_stream
    # configs[0]
    kat_key = "0123456789ABCDEF23456789ABCDEF01456789ABCDEF0123"
    pt = bytes.fromhex("54686520717566636B2062726F776E20666F78206A756D70")
    ct = bytearray(len(pt))
    t3.encrypt_batch(pt, ct, t3.triple_schedule(t3.parse_hex_key(kat_key)))
    kat_ok = ct.hex().upper() == "A826FD8CE53B855FCCE21C8112256FE668D5C05DD9B6B900"
    nb1 = (1 << 20) // 8
    d = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    e.fill_splitmix(d.data_ptr(), 0, nb1, SEED, stream)
    y = torch.empty_like(d)
    z = torch.empty_like(d)
    e.set_variant(N.VARIANT_BITSLICE)
    e.ecb_device(0, d.data_ptr(), z.data_ptr(), 1 << 20, stream)
    e.set_variant(N.VARIANT_AUTO)  # the product default: <= 1 MiB runs the low-latency SP-table kernel
    e.ecb_device(0, d.data_ptr(), y.data_ptr(), 1 << 20, stream)
    torch.cuda.synchronize()
    ok = bool(torch.equal(y, z))  # both kernels agree
    e.ecb_device(1, y.data_ptr(), z.data_ptr(), 1 << 20, stream)
    torch.cuda.synchronize()
    ok = ok and bool(torch.equal(z, d))  # and decrypt inverts encrypt
    x = d
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        e.ecb_device(0, d.data_ptr(), y.data_ptr(), x.nbytes, stream)
    ev0.record()
    for _ in range(50):
        e.ecb_device(0, d.data_ptr(), y.data_ptr(), x.nbytes, stream)
        e.ecb_device(1, y.data_ptr(), z.data_ptr(), x.nbytes, stream)
    ev1.record()
    torch.cuda.synchronize()
    us = ev0.elapsed_time(ev1) * 1e3 / 50
    # the same 50 pairs captured once in a CUDA graph and replayed (the C ABI
    # is stream-ordered and capture-safe): launch overhead amortised
    gs = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=gs):
        for _ in range(50):
            e.ecb_device(0, d.data_ptr(), y.data_ptr(), x.nbytes, gs.cuda_stream)
            e.ecb_device(1, y.data_ptr(), z.data_ptr(), x.nbytes, gs.cuda_stream)
    with torch.cuda.stream(gs):  # replay() launches on the current stream
        g.replay()
        torch.cuda.synchronize()
        ev0.record(gs)
        g.replay()
        ev1.record(gs)
    torch.cuda.synchronize()
    us_graph = ev0.elapsed_time(ev1) * 1e3 / 50
    ok = ok and bool(torch.equal(z, d))
    del g
    out["c0_1MiB_enc_dec"] = {"us_per_enc_plus_dec": round(us, 2), "GBps_enc_plus_dec": round(2 * x.nbytes / us / 1e3, 2),
                              "graph_us_per_enc_plus_dec": round(us_graph, 2),
                              "kernels_agree_and_round_trip": ok, "nist_sp800_67_kat": kat_ok,
                              "note": "latency bound (1 MiB = 128 warp tiles); variant AUTO runs the SP-table "
                                      "kernel at this size"}
    del d, y, z
    e.set_variant(N.VARIANT_BITSLICE)
    # configs[2]: 4 GiB decrypt
    n4 = (4 << 30) // 8
    buf = torch.empty(8 * n4, dtype=torch.uint8, device="cuda")
    e.fill_splitmix(buf.data_ptr(), 0, n4, SEED, stream)
    e.ecb_device(0, buf.data_ptr(), buf.data_ptr(), 8 * n4, stream)  # ciphertext of the payload
    dec = torch.empty_like(buf)
    e.ecb_device(1, buf.data_ptr(), dec.data_ptr(), 8 * n4, stream)
    torch.cuda.synchronize()
    rt_ok = e.checksum(dec.data_ptr(), 0, n4, stream) == _splitmix_checksum(e, torch, n4)
    ev0.record()
    for _ in range(5):
        e.ecb_device(1, buf.data_ptr(), dec.data_ptr(), 8 * n4, stream)
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / 5
    del dec
    host = torch.empty(8 * n4, dtype=torch.uint8).pin_memory()
    host.copy_(buf.cpu())
    del buf
    torch.cuda.empty_cache()
    out_h = torch.empty_like(host).pin_memory()
    e.ecb_host(1, host.data_ptr(), out_h.data_ptr(), 8 * n4)
    t0 = time.perf_counter()
    for _ in range(2):
        e.ecb_host(1, host.data_ptr(), out_h.data_ptr(), 8 * n4)
    e2e = 2 * 8 * n4 / (time.perf_counter() - t0) / 1e9
    del out_h
    out["c2_4GiB_decrypt"] = {"device_GBps": round(8 * n4 / ms / 1e6, 2), "e2e_GBps": round(e2e, 2),
                              "round_trip_checksum_ok": bool(rt_ok),
                              "note": "device: 5 decrypts of the 4 GiB ciphertext, CUDA events; "
                                      "e2e: t3des_cu_ecb_host pinned in -> pinned out incl. H2D/D2H"}
    del host
    # configs[4] edge case: K1 = K2 = K3 (option 3) is single DES; the engine
    # detects the collapsed EDE and runs 16 rounds instead of 48
    e3 = t3.Engine(e.device)
    e3.set_schedule(t3.triple_schedule(t3.parse_hex_key("0123456789ABCDEF")))
    n1 = (1 << 30) // 8
    b1 = torch.empty(8 * n1, dtype=torch.uint8, device="cuda")
    b2 = torch.empty_like(b1)
    e3.fill_splitmix(b1.data_ptr(), 0, n1, SEED, stream)
    kat = bytearray(8)
    t3.encrypt_batch(bytes.fromhex("4E6F772069732074"), kat, t3.triple_schedule(t3.parse_hex_key("0123456789ABCDEF")))
    for _ in range(3):
        e3.ecb_device(0, b1.data_ptr(), b2.data_ptr(), 8 * n1, stream)
    torch.cuda.synchronize()
    ev0.record()
    for _ in range(5):
        e3.ecb_device(0, b1.data_ptr(), b2.data_ptr(), 8 * n1, stream)
    ev1.record()
    torch.cuda.synchronize()
    ms3 = ev0.elapsed_time(ev1) / 5
    e3.ecb_device(1, b2.data_ptr(), b2.data_ptr(), 8 * n1, stream)
    torch.cuda.synchronize()
    out["c4_option3_1GiB_encrypt"] = {"device_GBps": round(8 * n1 / ms3 / 1e6, 2),
                                      "kat_3FA40E8A984D4815": kat.hex().upper() == "3FA40E8A984D4815",
                                      "round_trip_ok": bool(torch.equal(b1, b2)),
                                      "note": "K1 = K2 = K3: EDE collapses to single DES, 16 rounds"}
    del b2
    e3.close()
    # the key-specialised variant (NVRTC at run time, opt-in):
    # compile + load time, then the configs[1] payload through it, checked
    # against the shipped kernel's output
    e.set_variant(N.VARIANT_KEYED)
    try:
        # (the variants leg may already have compiled the encrypt module: the
        # decrypt module's first prepare is the compile + load time)
        t_first = e.keyed_prepare(1)
        t_hit = e.keyed_prepare(1)
        e.fill_splitmix(b1.data_ptr(), 0, n1, SEED, stream)
        kb = torch.empty_like(b1)
        e.ecb_device(0, b1.data_ptr(), kb.data_ptr(), 8 * n1, stream)
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(5):
            e.ecb_device(0, b1.data_ptr(), kb.data_ptr(), 8 * n1, stream)
        ev1.record()
        torch.cuda.synchronize()
        msk = ev0.elapsed_time(ev1) / 5
        e.set_variant(N.VARIANT_BITSLICE)  # the table-driven kernel (AUTO would now run the prepared module)
        ref = torch.empty_like(b1)
        e.ecb_device(0, b1.data_ptr(), ref.data_ptr(), 8 * n1, stream)
        torch.cuda.synchronize()
        out["f4_keyed_1GiB_encrypt"] = {
            "device_GBps": round(8 * n1 / msk / 1e6, 2), "jit_compile_load_s_first_use": round(t_first, 3),
            "cache_hit_s": round(t_hit, 6), "equal_to_shipped_kernel": bool(torch.equal(kb, ref)),
            "note": "T3DES_CU_VARIANT_KEYED: round keys folded into LOP3 immediates, NVRTC-compiled for this key; "
                    "opt-in: AUTO never compiles it, and runs it for large launches once t3des_cu_keyed_prepare "
                    "has built it (about the same ALU work per block as the table-driven kernel, DESIGN §3.7)"}
        del kb, ref
    except Exception as exc:  # NVRTC missing on the box: report, never a fallback
        out["f4_keyed_1GiB_encrypt"] = {"unavailable": f"{type(exc).__name__}: {exc}"}
    e.set_variant(N.VARIANT_BITSLICE)
    del b1
    torch.cuda.empty_cache()
    # configs[3]: the 64 GiB stream on one device — one launch, and the 8
    # block ranges 8 GPUs would own run back to back — checked against the
    # reference's checksum of the whole 64 GiB ciphertext
    from paper_1305_4376_b200.sharding import shard_range

    n64 = (64 << 30) // 8
    free, _ = torch.cuda.mem_get_info()
    gold = golden_c3()
    if free >= 8 * n64 + (4 << 30):
        big = torch.empty(8 * n64, dtype=torch.uint8, device="cuda")
        e.fill_splitmix(big.data_ptr(), 0, n64, SEED, stream)
        e.ecb_device(0, big.data_ptr(), big.data_ptr(), 8 * n64, stream)  # warm-up pair
        e.ecb_device(1, big.data_ptr(), big.data_ptr(), 8 * n64, stream)
        sums, times, plain_ok = {}, {}, True
        for g in (1, 8):  # each g: encrypt the payload in place as g shard ranges, checksum, decrypt back
            torch.cuda.synchronize()
            ev0.record()
            for r in range(g):
                first, count = shard_range(n64, g, r)
                e.ecb_device(0, big.data_ptr() + 8 * first, big.data_ptr() + 8 * first, 8 * count, stream)
            ev1.record()
            torch.cuda.synchronize()
            times[g] = ev0.elapsed_time(ev1)
            sums[g] = e.checksum(big.data_ptr(), 0, n64, stream)
            e.ecb_device(1, big.data_ptr(), big.data_ptr(), 8 * n64, stream)
            if gold:
                plain_ok = plain_ok and e.checksum(big.data_ptr(), 0, n64, stream) == int(gold["plaintext_checksum"], 16)
        want = int(gold["ciphertext_checksum"], 16) if gold else None
        out["c3_64GiB_block_range_shards"] = {
            "device_GBps_1_launch": round(8 * n64 / times[1] / 1e6, 2),
            "device_GBps_8_shards_back_to_back": round(8 * n64 / times[8] / 1e6, 2),
            "ciphertext_checksum": f"{sums[1]:016x}",
            "checksum_equal_1_vs_8_shards": sums[1] == sums[8],
            "checksum_equal_to_reference": (sums[1] == want and sums[8] == want and plain_ok) if gold else None,
            "note": "in-place encrypt of 64 GiB on one B200; the 8 shard ranges are the ones 8 GPUs own; "
                    "reference checksum from tests/golden/c3_checksum.json (reference encrypt_batch)"}
        del big
        torch.cuda.empty_cache()
    return out


def workload_config(args, world: int) -> dict:
    if world == 1:
        wl = (f"BASELINE configs[1]: 3DES-ECB encrypt {args.gib} GiB device-resident on 1 B200 "
              f"(configs[3], 64 GiB in block ranges, is the N>1 workload and a configs_measured leg here)")
        n = (args.gib << 30) // 8
    else:
        wl = (f"BASELINE configs[3]: 3DES-ECB encrypt {args.c3_gib} GiB device-resident, split into {world} "
              f"contiguous block ranges (t3des_cu_shard_range), one per GPU")
        n = (args.c3_gib << 30) // 8
    return {
        "workload": wl, "key": BENCH_KEY, "keying_option": 1,
        "global_blocks": n, "blocks_per_gpu": n // world,
        "variant": args.variant, "payload": "block i = splitmix64(0x3DE5C0DE ^ i), big-endian, generated on device",
        "l2_policy": "inputs larger than L2 (>= 1 GiB per rank per step vs 126 MB L2), no flush",
        "parallelism": f"block-range shards x{world}, no data-path collective",
    }


def _splitmix_checksum(e, torch, n) -> int:
    tmp = torch.empty(8 * n, dtype=torch.uint8, device="cuda")
    e.fill_splitmix(tmp.data_ptr(), 0, n, SEED, torch.cuda.current_stream().cuda_stream)
    v = e.checksum(tmp.data_ptr(), 0, n, torch.cuda.current_stream().cuda_stream)
    del tmp
    return v


def e2e_multi(torch, N, ts, host, one: int, world: int, ndev: int, k3: int) -> dict:
    """One process driving all N GPUs through t3des_cu_ecb_multi (the
    workers axis of DispatchConfig) on a pinned buffer of N x `one` bytes."""
    devs = [r % max(ndev, 1) for r in range(world)]
    mh = torch.empty(world * one, dtype=torch.uint8).pin_memory()
    for r in range(world):
        mh[r * one:(r + 1) * one].copy_(host)
    cdevs = (ctypes.c_int * world)(*devs)
    sub = ts.sub48()
    f = N.lib().t3des_cu_ecb_multi
    rc = f(cdevs, world, sub, 0, mh.data_ptr(), mh.data_ptr(), mh.numel())
    t0 = time.perf_counter()
    for _ in range(k3):
        rc = rc or f(cdevs, world, sub, 0, mh.data_ptr(), mh.data_ptr(), mh.numel())
    dtm = (time.perf_counter() - t0) / k3
    return {"value": round(world * one / dtm / 1e9, 3) if rc == 0 else None, "unit": "GB/s",
            "devices": devs, "bytes": world * one, "status": N.strerror(rc),
            "path": "t3des_cu_ecb_multi from one process (one host thread + context per "
                    "device, pinned buffer), the GPU reading of DispatchConfig.workers"}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--variant", choices=["bitslice", "bitslice_alu", "bitslice_dfma", "bitslice_shrfma", "bitslice_ldg", "sptable",
                                          "keyed"], default="bitslice")
    ap.add_argument("--gib", type=int, default=1, help="GiB per step at N = 1 (configs[1])")
    ap.add_argument("--c3-gib", type=int, default=64, help="global GiB per step at N > 1 (configs[3])")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-variants", action="store_true")
    ap.add_argument("--no-extra-configs", action="store_true")
    ap.add_argument("--traffic-bytes", type=float, default=None,
                    help="dram bytes per launch from an ncu --set full capture (else read profiles/)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rc = self_launch(args)
    if rc is not None:
        sys.exit(rc)
    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if os.environ.get("T3DES_BENCH_LAUNCH_PROBE"):  # tests: the launcher only, no work
        from paper_1305_4376_b200.sharding import shard_range

        n = ((args.gib if world == 1 else args.c3_gib) << 30) // 8
        print(json.dumps({"rank": rank, "world": world, "local_rank": local, "shard": shard_range(n, world, rank)}),
              flush=True)
        return
    if args.impl == "reference":
        run_reference_impl(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    import paper_1305_4376_b200 as t3
    from paper_1305_4376_b200 import _native as N

    # one rank per GPU; T3DES_BENCH_DIST_BACKEND=gloo lets the multi-rank
    # logic run with several ranks on one GPU (ranks never wait on each
    # other's kernels; NCCL refuses two ranks on one device)
    backend = os.environ.get("T3DES_BENCH_DIST_BACKEND", "nccl")
    ndev = torch.cuda.device_count()
    if backend == "nccl" and world > ndev:
        print(f"bench.py: {world} ranks need {world} GPUs, {ndev} visible "
              f"(T3DES_BENCH_DIST_BACKEND=gloo shares one GPU between ranks)", file=sys.stderr)
        sys.exit(2)
    device = local % max(ndev, 1)
    torch.cuda.set_device(device)
    numa = bind_to_gpu_cpus(device) if world > 1 else {"bound": False, "why": "N = 1"}
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", device))
        else:
            dist.init_process_group(backend)

    # host-side barrier (gloo): ranks that wait on it leave their GPUs idle,
    # unlike an NCCL barrier, whose kernel spins on the GPU — which would
    # time-slice with rank 0 driving every GPU in the e2e.multi leg
    hostgroup = dist.new_group(backend="gloo") if world > 1 else None

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def host_barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier(group=hostgroup)

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def gather_ints(x: int) -> list[int]:
        if world == 1:
            return [x]
        dev_ = "cuda" if backend == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.int64, device=dev_)
        parts = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        return [int(p.item()) for p in parts]

    e = t3.Engine(device)
    ts = t3.triple_schedule(t3.parse_hex_key(BENCH_KEY))
    e.set_schedule(ts)
    VARIANTS = {"bitslice": N.VARIANT_BITSLICE, "bitslice_alu": N.VARIANT_BITSLICE_ALU,
                "bitslice_dfma": N.VARIANT_BITSLICE_DFMA, "bitslice_shrfma": N.VARIANT_BITSLICE_SHRFMA,
                "bitslice_ldg": N.VARIANT_BITSLICE_LDG, "sptable": N.VARIANT_SPTABLE, "keyed": N.VARIANT_KEYED}
    e.set_variant(VARIANTS[args.variant])
    from paper_1305_4376_b200.sharding import shard_range

    n_global = ((args.gib if world == 1 else args.c3_gib) << 30) // 8
    first_block, nblocks = shard_range(n_global, world, rank)
    nbytes = 8 * nblocks
    stream = torch.cuda.Stream()
    sp = stream.cuda_stream
    src = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    dst = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    with torch.cuda.stream(stream):
        e.fill_splitmix(src.data_ptr(), first_block, nblocks, SEED, sp)
    torch.cuda.synchronize()

    # correctness gate before timing, without the CPU oracle (that is test
    # infrastructure; tests/ compare the kernels against it bit for bit):
    # the NIST SP 800-67 vector through the engine, the bitsliced output vs
    # the independent SP-table kernel on a sample, and decrypt(encrypt(x)) == x
    import numpy as np

    parity_ok = nist_kat_ok(t3) and cross_check(e, N, torch, src, dst, nblocks, sp, VARIANTS[args.variant])

    for _ in range(args.warmup):
        e.ecb_device(0, src.data_ptr(), dst.data_ptr(), nbytes, sp)
    barrier()
    l0 = e.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(device) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            e.ecb_device(0, src.data_ptr(), dst.data_ptr(), nbytes, sp)
        ev1.record(stream)
        barrier()
    launches = sum(gather_ints(e.launch_count() - l0))
    ms_total = ev0.elapsed_time(ev1)
    ms_step = max_over_ranks(ms_total / args.steps)
    gbs = 8 * n_global / (ms_step * 1e-3) / 1e9
    clocks = clk.summary()

    # the output of the timed steps against the reference's checksums: the
    # per-shard checksums add up to the reference checksum of the whole
    # stream (tests/golden/c3_checksum.json; its 1 GiB pieces cover configs[1])
    gold = golden_c3()
    shard_sums = gather_ints(u64_to_i64(e.checksum(dst.data_ptr(), first_block, nblocks, sp)))
    total_sum = sum(shard_sums) % 2**64
    want = None
    if gold and world > 1 and args.c3_gib == 64:
        want = int(gold["ciphertext_checksum"], 16)
    elif gold and world == 1 and args.gib == 1:
        want = int(gold["piece_ciphertext_checksums"][0], 16)
    output_check = {"checksum": f"{total_sum:016x}", "reference_checksum": f"{want:016x}" if want is not None else None,
                    "checksum_equal_to_reference": (total_sum == want) if want is not None else None}
    if world > 1:
        output_check["checksum_equal_to_N1"] = output_check["checksum_equal_to_reference"]
        output_check["how"] = ("sum of the ranks' shard checksums == the single-run checksum of the 64 GiB "
                               "ciphertext (reference encrypt_batch, tests/golden/c3_checksum.json; the N=1 "
                               "configs[3] leg reproduces it on one GPU)")

    peaks = measured_peaks()
    sms = torch.cuda.get_device_properties(device).multi_processor_count
    fmax = float(peaks.get("sm_max_mhz", 1965.0))
    peak_tlops = sms * ALU_LANES_PER_CLK_PER_SM * fmax * 1e6 / 1e12
    per_gpu_bps = nblocks / (ms_step * 1e-3)
    alu_ops = executed_alu_ops_per_block()
    achieved = per_gpu_bps * W_ALG / 1e12
    traffic = args.traffic_bytes
    if traffic is None:
        try:
            with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
                traffic = json.load(f).get(args.variant)
        except Exception:
            traffic = None
    hbm_peak = float(peaks.get("hbm_gbs", 6553.3))
    roofline = {
        "bound": "alu", "achieved": round(achieved, 4), "peak": round(peak_tlops, 4), "unit": "Tlop3/s",
        "frac": round(achieved / peak_tlops, 4), "traffic": traffic,
        "kernel_ms": round(ms_step, 4),
        "per": "one GPU (rank 0's shard at N > 1; the slowest rank sets ms_per_step)",
        "peak_source": f"{sms} SMs x {ALU_LANES_PER_CLK_PER_SM} ALU lanes/clk (LOP3 issue rate measured by "
                       f"tools/microbench/pipe_rates.cu, profiles/r1/pipe_rates_b200.txt) x sm_max_mhz {fmax:.0f} "
                       f"({'MEASURED_PEAKS.json' if 'sm_max_mhz' in peaks else 'fallback'})",
        "frac_at_run_clock": (round(achieved / (sms * 64 * clocks["sm_mhz"] * 1e6 / 1e12), 4)
                              if clocks.get("sm_mhz") else None),
        "w_alg_lane_ops_per_block": W_ALG,
        # what the shipped kernel actually issues to the ALU pipe per block
        # (static count: S-box LOP3 + Feistel LOP3 per round, plus the slice
        # transposes; tests/test_sass.py pins it to the binary), and the
        # utilisation that implies
        "executed_alu_lane_ops_per_block": alu_ops,
        "alu_pipe_frac": round(per_gpu_bps * alu_ops / (peak_tlops * 1e12), 4),
        "hbm": {"achieved_gbs": round(per_gpu_bps * 16 / 1e9, 2), "peak_gbs": hbm_peak,
                "frac": round(per_gpu_bps * 16 / 1e9 / hbm_peak, 4), "bytes_per_block": 16},
    }

    line = {
        "metric": METRIC, "value": round(gbs, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
        "scaling": "weak" if world == 1 else "strong",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": workload_config(args, world),
        "roofline": roofline, "clocks": clocks, "gpu_launches": int(launches),
        "self_check": {"ok": parity_ok, "how": "NIST SP 800-67 KAT via the engine; bitsliced == SP-table kernel "
                       "on a 1/4096 sample; decrypt(encrypt(x)) == x checksum"},
        "output_check": output_check,
    }
    if world > 1:
        line["numa"] = numa
        line["dist_backend"] = backend

    # the other variants (north star: bitsliced vs SP-table, ncu picks)
    if not args.no_variants and world == 1:
        line["variants"] = {args.variant: round(gbs, 3)}
        for other, code in VARIANTS.items():
            if other == args.variant:
                continue
            e.set_variant(code)
            for _ in range(2):
                e.ecb_device(0, src.data_ptr(), dst.data_ptr(), nbytes, sp)
            barrier()
            k2 = max(3, args.steps // 4)
            ev0.record(stream)
            for _ in range(k2):
                e.ecb_device(0, src.data_ptr(), dst.data_ptr(), nbytes, sp)
            ev1.record(stream)
            barrier()
            ms2 = max_over_ranks(ev0.elapsed_time(ev1) / k2)
            line["variants"][other] = round(world * nbytes / (ms2 * 1e-3) / 1e9, 3)
        e.set_variant(VARIANTS[args.variant])

    # N > 1: the weak-scaling figure next to it — 1 GiB per rank (the first
    # GiB of each rank's range), checked against the reference's per-GiB
    # checksums
    one = min(nbytes, 1 << 30)
    if world > 1:
        for _ in range(2):
            e.ecb_device(0, src.data_ptr(), dst.data_ptr(), one, sp)
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            e.ecb_device(0, src.data_ptr(), dst.data_ptr(), one, sp)
        ev1.record(stream)
        barrier()
        msw = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
        cs = e.checksum(dst.data_ptr(), first_block, one // 8, sp)
        ok = None
        if gold and args.c3_gib == 64 and one == 1 << 30 and first_block % (1 << 27) == 0:
            ok = cs == int(gold["piece_ciphertext_checksums"][first_block >> 27], 16)
        oks = gather_ints(-1 if ok is None else int(ok))
        line["weak_1GiB_per_gpu"] = {
            "value": round(world * one / (msw * 1e-3) / 1e9, 3), "unit": "GB/s", "ms_per_step": round(msw, 4),
            "steps": args.steps, "checksums_equal_to_reference": None if -1 in oks else all(oks),
            "how": "each rank encrypts the first GiB of its own block range; max over ranks"}

    del dst
    torch.cuda.empty_cache()

    # end to end through the C ABI host entry (pinned H2D + kernel + D2H);
    # 1 GiB per rank (host RAM bounds it at N > 1; weak)
    if not args.no_e2e:
        host = torch.empty(one, dtype=torch.uint8).pin_memory()
        host.copy_(src[:one].cpu())
        del src
        torch.cuda.empty_cache()
        e.ecb_host(0, host.data_ptr(), host.data_ptr(), one)  # warm (allocates staging)
        k3 = max(5, min(args.steps, 8))
        barrier()
        t0 = time.perf_counter()
        for _ in range(k3):
            e.ecb_host(0, host.data_ptr(), host.data_ptr(), one)
        dt = max_over_ranks((time.perf_counter() - t0) / k3)
        line["e2e"] = {"value": round(world * one / dt / 1e9, 3), "unit": "GB/s",
                       "h2d_bytes_per_step": world * one, "d2h_bytes_per_step": world * one,
                       "path": f"t3des_cu_ecb_host, pinned host buffer, {one >> 20} MiB per rank, in place, "
                               "default pipeline (3 streams, 32 MiB stages with an 8 MiB ramp)",
                       "steps": k3, "timing": "host wall clock around the synchronous C-ABI call, max over ranks"}
        # the ceiling: pinned copy rates measured with CUDA events
        ceil = pcie_ceiling(torch)
        line["e2e"]["pcie"] = ceil
        line["e2e"]["frac_of_bidir_ceiling"] = round((one / dt / 1e9) / ceil["bidir_gbs_each_way"], 3)
        # the same call from pageable memory (what a reference caller's
        # std::vector is): staged through the engine's pinned ring by host
        # copy threads
        page = host.numpy().copy()
        e.ecb_host(0, page.ctypes.data, page.ctypes.data, one)
        barrier()
        t0 = time.perf_counter()
        for _ in range(k3):
            e.ecb_host(0, page.ctypes.data, page.ctypes.data, one)
        dtp = max_over_ranks((time.perf_counter() - t0) / k3)
        line["e2e"]["pageable"] = {"value": round(world * one / dtp / 1e9, 3), "unit": "GB/s",
                                   "path": "t3des_cu_ecb_host, pageable host buffer (numpy), in place"}
        # the same pageable buffer after the opt-in t3des_cu_host_register
        # (a caller that reuses its buffer): the pinned DMA path, no staging
        try:
            t0 = time.perf_counter()
            reg = t3.HostRegistration(page)
            reg_ms = (time.perf_counter() - t0) * 1e3
            e.ecb_host(0, page.ctypes.data, page.ctypes.data, one)
            ok_reg = True
        except Exception as exc:  # an extra leg: never lose the line over it
            ok_reg, reg_err = False, f"{type(exc).__name__}: {exc}"[:300]
        barrier()
        t0 = time.perf_counter()
        for _ in range(k3 if ok_reg else 0):
            e.ecb_host(0, page.ctypes.data, page.ctypes.data, one)
        dtr = max_over_ranks((time.perf_counter() - t0) / k3)
        if ok_reg:
            reg.close()
            line["e2e"]["pageable_registered"] = {
                "value": round(world * one / dtr / 1e9, 3), "unit": "GB/s", "register_ms": round(reg_ms, 1),
                "path": "the pageable buffer registered once with t3des_cu_host_register (opt-in, outside the timing)"}
        else:
            line["e2e"]["pageable_registered"] = {"value": None, "error": reg_err}
        del page
        # one process driving all N GPUs through t3des_cu_ecb_multi (the
        # workers axis of DispatchConfig): rank 0, the other ranks idle on a
        # host-side barrier
        host_barrier()
        if rank == 0:
            try:
                line["e2e"]["multi"] = e2e_multi(torch, N, ts, host, one, world, ndev, k3)
            except Exception as exc:  # an extra leg: never lose the line over it
                line["e2e"]["multi"] = {"value": None, "error": f"{type(exc).__name__}: {exc}"[:300]}
        host_barrier()
        del host
    else:
        line["e2e"] = None
        del src

    if not args.no_extra_configs and world == 1:
        try:
            line["configs_measured"] = extra_configs(e, t3, N, torch, np)
        except Exception as exc:
            line["configs_measured"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
            torch.cuda.empty_cache()

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_reference_arm()

    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        host_barrier()
        dist.destroy_process_group()
    e.close()


if __name__ == "__main__":
    main()
