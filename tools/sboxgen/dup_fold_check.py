#!/usr/bin/env python3
"""Can the 16 E-duplicate key corrections fold into the S-box circuits?

The table-driven round XORs the 16 duplicated E slots with their correction
words D (IMAD x*S + D on the FMA pipe, plus 16 constant loads per round).  A
correction folds for free into a gate that has a spare operand (a LUT that
ignores one input, or a repeated input): g(a ^ d, b) is one LOP3 of (a, b, d).
It folds for a duplicated R bit if every consumer of one of its two E slots
has a spare operand.  Prints, per duplicated R bit, the consumers of both
slots in the shipped circuits (paper_1305_4376_b200/csrc/sbox_circuits).
"""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..",
                                "paper_1305_4376_b200", "csrc"))
import gen_bitslice as G  # noqa: E402


def depends(lut: int, pos: int) -> bool:
    sh = (4, 2, 1)[pos]
    return any(((lut >> m) & 1) != ((lut >> (m ^ sh)) & 1) for m in range(8))


def slot_users(circ, j):
    box, kvar = j // 6, 5 - (j % 6)
    gates, outs = circ[box]
    users = blocked = 0
    for _g, a, b, c, lut in gates:
        ins = (a, b, c)
        if kvar in ins:
            users += 1
            blocked += not (any(not depends(lut, p) for p in range(3)) or len(set(ins)) < 3)
    for o in outs.values():
        if (o[0] == "f" and kvar in o[1:3]) or o[0] == kvar:  # Feistel lop3 (L, a, b): no spare slot
            users += 1
            blocked += 1
    return users, blocked


def main() -> None:
    circ = [G.load_circuit(b) for b in range(8)]
    slots = defaultdict(list)
    for j, q in enumerate(G.E):
        slots[q - 1].append(j)
    foldable = 0
    for q, js in sorted(slots.items()):
        if len(js) != 2:
            continue
        info = [(j, *slot_users(circ, j)) for j in js]
        ok = any(b == 0 for _, _, b in info)
        foldable += ok
        print(f"R[{q:2d}] " + "  ".join(f"slot {j:2d} (S{j // 6 + 1} x{5 - j % 6}): {u} users, {b} without a spare"
                                        for j, u, b in info) + f"  foldable={ok}")
    print(f"foldable duplicated bits: {foldable} of 16")


if __name__ == "__main__":
    main()
