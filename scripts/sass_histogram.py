#!/usr/bin/env python3
"""SASS opcode histograms of the shipped kernels, read from the built
library with cuobjdump (no GPU needed).

  python scripts/sass_histogram.py [--so paper_1305_4376_b200/libt3des_b200.so] [--out profiles/r2/sass_histogram.txt]

For the bitsliced kernel it also locates the round loop (the backward branch
of the 2-round body) and counts the ALU work of its straight-line body, which
is what bench.py's `executed_alu_lane_ops_per_block` is derived from;
tests/test_sass.py pins those counts to the generated S-box circuits.
"""
from __future__ import annotations

import argparse
import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "paper_1305_4376_b200", "libt3des_b200.so")
CUOBJDUMP = "/usr/local/cuda/bin/cuobjdump"
SHIPPED = {
    "bitsliced (shipped, OPT 5, 48 rounds)": "_Z16t3_bs_tma_kernelILi5ELi48EEvPKhPhm9T3BsTable",
    "bitsliced, collapsed EDE (16 rounds)": "_Z16t3_bs_tma_kernelILi5ELi16EEvPKhPhm9T3BsTable",
    "SP-table (shipped mask 490)": "_Z12t3_sp_kernelILi490EEvPK5uint2PS0_mPKjiS5_7T3SpMul12T3SpKeyParami",
}
_INS = re.compile(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;")


def sass_functions(so: str = SO) -> dict[str, list[tuple[int, str, str]]]:
    """mangled name -> [(address, opcode, full text)]"""
    txt = subprocess.run([CUOBJDUMP, "-sass", so], check=True, capture_output=True, text=True).stdout
    funcs: dict[str, list] = {}
    cur = None
    for line in txt.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = funcs.setdefault(m.group(1), [])
            continue
        m = _INS.match(line)
        if m and cur is not None:
            body = m.group(2)
            op = re.sub(r"^@!?U?P\w+\s+", "", body).split()[0].split(".")[0]
            cur.append((int(m.group(1), 16), op, body))
    return funcs


def histogram(ins) -> collections.Counter:
    return collections.Counter(op for _, op, _ in ins)


def round_loop(ins) -> dict:
    """The round loop: the innermost loop (a backward branch whose range holds
    no other backward branch) with the most LOP3.  Its straight-line head
    block (loop start up to the first branch) is the 2-round body every
    iteration executes; the pass-boundary re-whitening rounds follow it as
    conditional blocks."""
    back = []
    for a, op, body in ins:
        m = re.search(r"BRA(?:\.\w+)*\s+(?:!?U?P\w+,\s*)?0x([0-9a-f]+)", body)
        if op == "BRA" and m and int(m.group(1), 16) < a:
            back.append((int(m.group(1), 16), a))
    inner = [(lo, hi) for lo, hi in back if not any(lo <= a < hi for l2, a in back if (l2, a) != (lo, hi))]
    if not inner:
        return {}
    lop3 = lambda r: sum(1 for a, op, _ in ins if r[0] <= a <= r[1] and op == "LOP3")  # noqa: E731
    lo, hi = max(inner, key=lop3)
    loop = [x for x in ins if lo <= x[0] <= hi]
    head_end = next(a for a, op, _ in loop if op == "BRA")
    head = [x for x in loop if x[0] < head_end]
    return {"start": lo, "end": hi, "loop": histogram(loop), "body": histogram(head),
            "outside": histogram([x for x in ins if not lo <= x[0] <= hi])}


def report(so: str = SO) -> str:
    funcs = sass_functions(so)
    out = [f"# cuobjdump -sass {os.path.relpath(so, ROOT)} — opcode histograms of the shipped kernels", ""]
    for label, name in SHIPPED.items():
        ins = funcs.get(name)
        if ins is None:
            out.append(f"## {label}: {name} not found")
            continue
        h = histogram(ins)
        out.append(f"## {label}\n{name}\n{len(ins)} instructions")
        out.append("  " + "  ".join(f"{op} {n}" for op, n in h.most_common()))
        if "bs_tma" in name:
            rl = round_loop(ins)
            b, o = rl["body"], rl["outside"]
            out.append(f"round loop 0x{rl['start']:x}-0x{rl['end']:x}; 2-round body: LOP3 {b['LOP3']} IMAD {b['IMAD']} "
                       f"LDC {b['LDC']} LDCU {b['LDCU']} SHF {b['SHF']} PRMT {b['PRMT']}")
            out.append(f"outside the loop (tile load/transposes/store): LOP3 {o['LOP3']} PRMT {o['PRMT']} SHF {o['SHF']} "
                       f"IMAD {o['IMAD']}")
        out.append("")
    return "\n".join(out)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--so", default=SO)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    r = report(a.so)
    if a.out:
        os.makedirs(os.path.dirname(a.out), exist_ok=True)
        with open(a.out, "w") as f:
            f.write(r + "\n")
    print(r)


if __name__ == "__main__":
    main()
