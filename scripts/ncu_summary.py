#!/usr/bin/env python3
"""Summarise ncu captures into profiles/ (committed evidence).

  python scripts/ncu_summary.py <report.ncu-rep> <out.md> [--launches launches.csv]
      [--traffic-key bitslice]

Writes a markdown summary (the metrics the roofline and DESIGN.md cite) and
updates profiles/traffic.json with dram read+write bytes per launch, which
bench.py reports as roofline.traffic.
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

METRICS = [
    ("gpu__time_duration.sum", "kernel duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe % of peak (active)"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed", "ALU pipe % of peak (elapsed)"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe % of peak"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe % of peak"),
    ("sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active", "uniform pipe % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("smsp__inst_executed.sum", "warp instructions executed"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__warps_eligible.avg.per_cycle_active", "eligible warps / scheduler"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_static", "static smem / block"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem load bank conflicts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smem store bank conflicts"),
    ("smsp__sass_inst_executed_op_shared_ld.sum", "shared loads (warp)"),
    ("smsp__inst_executed_op_tma_ld.sum", "TMA loads"),
]
STALLS = ["math_pipe_throttle", "wait", "short_scoreboard", "long_scoreboard", "not_selected", "selected",
          "no_instructions", "mio_throttle", "lg_throttle", "barrier", "dispatch_stall", "branch_resolving"]


def raw(report: str) -> list[dict]:
    out = subprocess.check_output(["ncu", "-i", report, "--page", "raw", "--csv"], text=True,
                                  stderr=subprocess.DEVNULL)
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [{"_units": dict(zip(hdr, units)), **dict(zip(hdr, r))} for r in rows[2:]]


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("out")
    ap.add_argument("--launches")
    ap.add_argument("--traffic-key")
    a = ap.parse_args()
    lines = [f"# ncu summary: `{os.path.basename(a.report)}`", ""]
    for k in raw(a.report):
        units = k["_units"]
        lines.append(f"## {k.get('Kernel Name', '?')}")
        lines.append("")
        lines.append("| metric | value | unit | ncu name |")
        lines.append("|---|---|---|---|")
        for m, label in METRICS:
            if m in k:
                lines.append(f"| {label} | {k[m]} | {units.get(m, '')} | `{m}` |")
        st = []
        for s in STALLS:
            key = f"smsp__pcsamp_warps_issue_stalled_{s}"
            if key in k and k[key] not in ("", "0"):
                st.append((s, float(k[key])))
        if st:
            tot = sum(v for _, v in st)
            lines.append("")
            lines.append("Stall reasons (pc sampling, share of samples): " +
                         ", ".join(f"{s} {100 * v / tot:.1f}%" for s, v in sorted(st, key=lambda x: -x[1])))
        lines.append("")
        if a.traffic_key and "dram__bytes_read.sum" in k:
            mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd = float(k["dram__bytes_read.sum"]) * mul.get(units["dram__bytes_read.sum"], 1)
            wr = float(k["dram__bytes_write.sum"]) * mul.get(units["dram__bytes_write.sum"], 1)
            tpath = os.path.join(ROOT, "profiles", "traffic.json")
            t = json.load(open(tpath)) if os.path.exists(tpath) else {}
            t[a.traffic_key] = rd + wr
            json.dump(t, open(tpath, "w"), indent=1)
    if a.launches:
        rows = list(csv.reader(open(a.launches)))
        hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        hdr = rows[hdr_i]
        ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
        per = {}
        for r in rows[hdr_i + 1:]:
            if len(r) <= vi:
                continue
            name = r[ki].split("(")[0]
            per.setdefault(name, []).append(float(r[vi].replace(",", "")))
        tot = sum(sum(v) for v in per.values())
        lines.append("## launch list (gpu__time_duration.sum, cold-cache, serialised)")
        lines.append("")
        lines.append("| kernel | launches | total | share |")
        lines.append("|---|---|---|---|")
        for n, v in sorted(per.items(), key=lambda x: -sum(x[1])):
            lines.append(f"| `{n}` | {len(v)} | {sum(v):.0f} | {100 * sum(v) / tot:.1f}% |")
        lines.append("")
    with open(a.out, "w") as f:
        f.write("\n".join(lines))
    print("\n".join(lines))


if __name__ == "__main__":
    sys.exit(main())
