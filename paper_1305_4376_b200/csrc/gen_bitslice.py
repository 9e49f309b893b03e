#!/usr/bin/env python3
"""Generate the bitsliced 3DES round code and its host-side tables.

Inputs
  csrc/sbox_circuits/box{0..7}.txt   LOP3 circuits found by tools/sboxgen
  the FIPS 46-3 permutation tables (data; reference proj/src/des.cpp:8-41)

Outputs
  csrc/generated/bitslice_rounds.cuh  t3_round(): one Feistel round on 32+32
                                      slice words (all 8 S-boxes as lop3
                                      circuits, E and P as register renaming)
                                      plus the IP/FP slice gathers.
  csrc/generated/bitslice_tables.h    maps the host needs to build the
                                      per-round constant table (E primary /
                                      secondary slots).

Bit conventions (reference des.hpp:8-15, des.cpp:77-96):
  * FIPS bit 1 is the MSB; bytes are big-endian on the wire.
  * S-box i reads E slots 6i..6i+5; slot 6i is bit 5 of `six`.  Circuit
    variable k is bit k of `six`, i.e. slot 6i+5-k.
  * S-box i output value bit o (o=3 is the MSB) lands at FIPS position
    4i+4-o of the 32-bit S output, then P maps it (f bit p = S bit P[p-1]).

Slice layout: a thread owns 32 blocks; after the 32x32 transposes
lo[k] bit m = bit k of the little-endian word holding bytes 0..3 of the
thread's block m (hi[k]: bytes 4..7).  Bit k of such a word is FIPS bit
8*(k>>3) + 8 - (k&7) (+32 for hi).

Whitening: every R-role slice word is stored XORed with the
key bit of its *primary* E slot for the round that next reads it, so the
key XOR of the 32 primary slots folds into the Feistel XOR
(L' = L ^ f ^ C, one 3-input lop3) and only the 16 duplicated E slots
need an explicit XOR (with D).  The host computes C and D per round.
"""
from __future__ import annotations

import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))

IP = [58, 50, 42, 34, 26, 18, 10, 2, 60, 52, 44, 36, 28, 20, 12, 4,
      62, 54, 46, 38, 30, 22, 14, 6, 64, 56, 48, 40, 32, 24, 16, 8,
      57, 49, 41, 33, 25, 17, 9, 1, 59, 51, 43, 35, 27, 19, 11, 3,
      61, 53, 45, 37, 29, 21, 13, 5, 63, 55, 47, 39, 31, 23, 15, 7]
FP = [40, 8, 48, 16, 56, 24, 64, 32, 39, 7, 47, 15, 55, 23, 63, 31,
      38, 6, 46, 14, 54, 22, 62, 30, 37, 5, 45, 13, 53, 21, 61, 29,
      36, 4, 44, 12, 52, 20, 60, 28, 35, 3, 43, 11, 51, 19, 59, 27,
      34, 2, 42, 10, 50, 18, 58, 26, 33, 1, 41, 9, 49, 17, 57, 25]
E = [32, 1, 2, 3, 4, 5, 4, 5, 6, 7, 8, 9, 8, 9, 10, 11,
     12, 13, 12, 13, 14, 15, 16, 17, 16, 17, 18, 19, 20, 21, 20, 21,
     22, 23, 24, 25, 24, 25, 26, 27, 28, 29, 28, 29, 30, 31, 32, 1]
P = [16, 7, 20, 21, 29, 12, 28, 17, 1, 15, 23, 26, 5, 18, 31, 10,
     2, 8, 24, 14, 32, 27, 3, 9, 19, 13, 30, 6, 22, 11, 4, 25]
SBOX = [
    [14, 4, 13, 1, 2, 15, 11, 8, 3, 10, 6, 12, 5, 9, 0, 7, 0, 15, 7, 4, 14, 2, 13, 1, 10, 6, 12, 11, 9, 5, 3, 8,
     4, 1, 14, 8, 13, 6, 2, 11, 15, 12, 9, 7, 3, 10, 5, 0, 15, 12, 8, 2, 4, 9, 1, 7, 5, 11, 3, 14, 10, 0, 6, 13],
    [15, 1, 8, 14, 6, 11, 3, 4, 9, 7, 2, 13, 12, 0, 5, 10, 3, 13, 4, 7, 15, 2, 8, 14, 12, 0, 1, 10, 6, 9, 11, 5,
     0, 14, 7, 11, 10, 4, 13, 1, 5, 8, 12, 6, 9, 3, 2, 15, 13, 8, 10, 1, 3, 15, 4, 2, 11, 6, 7, 12, 0, 5, 14, 9],
    [10, 0, 9, 14, 6, 3, 15, 5, 1, 13, 12, 7, 11, 4, 2, 8, 13, 7, 0, 9, 3, 4, 6, 10, 2, 8, 5, 14, 12, 11, 15, 1,
     13, 6, 4, 9, 8, 15, 3, 0, 11, 1, 2, 12, 5, 10, 14, 7, 1, 10, 13, 0, 6, 9, 8, 7, 4, 15, 14, 3, 11, 5, 2, 12],
    [7, 13, 14, 3, 0, 6, 9, 10, 1, 2, 8, 5, 11, 12, 4, 15, 13, 8, 11, 5, 6, 15, 0, 3, 4, 7, 2, 12, 1, 10, 14, 9,
     10, 6, 9, 0, 12, 11, 7, 13, 15, 1, 3, 14, 5, 2, 8, 4, 3, 15, 0, 6, 10, 1, 13, 8, 9, 4, 5, 11, 12, 7, 2, 14],
    [2, 12, 4, 1, 7, 10, 11, 6, 8, 5, 3, 15, 13, 0, 14, 9, 14, 11, 2, 12, 4, 7, 13, 1, 5, 0, 15, 10, 3, 9, 8, 6,
     4, 2, 1, 11, 10, 13, 7, 8, 15, 9, 12, 5, 6, 3, 0, 14, 11, 8, 12, 7, 1, 14, 2, 13, 6, 15, 0, 9, 10, 4, 5, 3],
    [12, 1, 10, 15, 9, 2, 6, 8, 0, 13, 3, 4, 14, 7, 5, 11, 10, 15, 4, 2, 7, 12, 9, 5, 6, 1, 13, 14, 0, 11, 3, 8,
     9, 14, 15, 5, 2, 8, 12, 3, 7, 0, 4, 10, 1, 13, 11, 6, 4, 3, 2, 12, 9, 5, 15, 10, 11, 14, 1, 7, 6, 0, 8, 13],
    [4, 11, 2, 14, 15, 0, 8, 13, 3, 12, 9, 7, 5, 10, 6, 1, 13, 0, 11, 7, 4, 9, 1, 10, 14, 3, 5, 12, 2, 15, 8, 6,
     1, 4, 11, 13, 12, 3, 7, 14, 10, 15, 6, 8, 0, 5, 9, 2, 6, 11, 13, 8, 1, 4, 10, 7, 9, 5, 0, 15, 14, 2, 3, 12],
    [13, 2, 8, 4, 6, 15, 11, 1, 10, 9, 3, 14, 5, 0, 12, 7, 1, 15, 13, 8, 10, 3, 7, 4, 12, 5, 6, 11, 0, 14, 9, 2,
     7, 11, 4, 1, 9, 12, 14, 2, 0, 6, 10, 13, 15, 3, 5, 8, 2, 1, 14, 7, 4, 10, 8, 13, 15, 12, 9, 0, 3, 5, 6, 11],
]


def sbox_value(box: int, six: int) -> int:
    row = ((six >> 4) & 2) | (six & 1)
    col = (six >> 1) & 0xF
    return SBOX[box][row * 16 + col]


def load_circuit(box: int, path: str | None = None):
    path = path or os.path.join(HERE, "sbox_circuits", f"box{box}.txt")
    gates, outs = [], {}
    with open(path) as f:
        for line in f:
            t = line.split()
            if not t:
                continue
            if t[0] == "g":
                gates.append((int(t[1]), int(t[2]), int(t[3]), int(t[4]), int(t[5], 16)))
            elif t[0] == "o":
                outs[int(t[1])] = (int(t[2]), int(t[3]))
            elif t[0] == "f":  # output = h(a, b), h bit (2A + B): Feistel top
                o, a, b, h = int(t[1]), int(t[2]), int(t[3]), int(t[4], 16)
                if h in (0xA, 0x5):  # h = b or ~b: a plain output
                    outs[o] = (b, int(h == 0x5))
                elif h in (0xC, 0x3):  # h = a or ~a
                    outs[o] = (a, int(h == 0x3))
                else:
                    outs[o] = ("f", a, b, h)
    return gates, outs


def out_value(val: dict, o) -> int:
    if o[0] == "f":
        _, a, b, h = o
        return (h >> (2 * val[a] + val[b])) & 1
    g, inv = o
    return val[g] ^ inv


def feistel_lut(h: int) -> int:
    """LOP3 immediate of L ^ h(a, b) over (L, a, b)."""
    lut = 0
    for m in range(8):
        L, a, b = (m >> 2) & 1, (m >> 1) & 1, m & 1
        lut |= (L ^ ((h >> (2 * a + b)) & 1)) << m
    return lut


def lut_apply(lut: int, a: int, b: int, c: int) -> int:
    return (lut >> ((a << 2) | (b << 1) | c)) & 1


def verify_circuit(box: int, gates, outs) -> None:
    """Exhaustive check: 64 inputs x 4 outputs against the FIPS table."""
    for six in range(64):
        val = {k: (six >> k) & 1 for k in range(6)}
        for g, a, b, c, lut in gates:
            val[g] = lut_apply(lut, val[a], val[b], val[c])
        s = sbox_value(box, six)
        for o in range(4):
            if out_value(val, outs[o]) != ((s >> o) & 1):
                raise SystemExit(f"circuit for S{box + 1} wrong at six={six} bit {o}")


def slice_of_fips_in(f: int) -> str:
    """Slice array element holding FIPS input bit f (1..64)."""
    half = "lo" if f <= 32 else "hi"
    g = (f - 1) % 32
    k = 8 * (g >> 3) + 7 - (g & 7)
    return f"{half}[{k}]"


def e_slot_maps():
    first = {}
    prim_slot = [0] * 32  # R bit q (0-based) -> primary slot
    secondary = []  # list of slots that are secondary, in D order
    for j, q in enumerate(E):
        if q - 1 not in first:
            first[q - 1] = j
            prim_slot[q - 1] = j
        else:
            secondary.append(j)
    assert len(secondary) == 16
    return prim_slot, secondary


# E-duplicate corrections that may go to the FMA pipe (bit d = D word d);
# the default is all 16 (measured best).
DFMA_MASK = int(os.environ.get("T3_GEN_DFMA_MASK", "0xFFFF"), 0)


def gen_round(circuits) -> list[str]:
    prim_slot, secondary = e_slot_maps()
    d_index = {j: i for i, j in enumerate(secondary)}
    # f bit p (0-based) <- S output FIPS position P[p]
    pos_to_p = {P[p]: p for p in range(32)}
    out = []
    out.append("// One Feistel round on slice words: L ^= f(R, K) with the key folded")
    out.append("// into the whitening constants (see gen_bitslice.py docstring).")
    out.append("//   k[0..31]  : C, XORed into L bit p together with f bit p")
    out.append("//   k[32..47] : D, XORed into the 16 duplicated E slots")
    out.append("//   k[48..63] : S = D | 1, for the FMA-pipe form x ^ D = x * S + D")
    out.append("template <int OPT, class KP>")
    out.append("T3_FI void t3_round(uint32_t (&L)[32], const uint32_t (&R)[32], const T3Fk fk, const KP k) {")
    # per-S-box statement lists; T3_GEN_ORDER (experiments) interleaves them:
    # "box" (default: one S-box after the other), "rr" (gate i of every box in
    # turn), "pairs" (round-robin within S-box pairs)
    order = os.environ.get("T3_GEN_ORDER", "box")
    pre = "" if order == "box" else "s{box}"
    streams = []
    for box in range(8):
        gates, outs = circuits[box]
        st = []
        names = {}
        pf = pre.format(box=box)
        for kvar in range(6):
            j = 6 * box + 5 - kvar
            q = E[j] - 1
            if j in d_index:
                nm = f"{pf}x{kvar}"
                if (DFMA_MASK >> d_index[j]) & 1:
                    st.append(f"const uint32_t {nm} = t3_dfix<OPT>(R[{q}], k[{32 + d_index[j]}], k[{48 + d_index[j]}]);")
                else:  # kept on the ALU pipe (T3_GEN_DFMA_MASK experiments)
                    st.append(f"const uint32_t {nm} = R[{q}] ^ k[{32 + d_index[j]}];")
                names[kvar] = nm
            else:
                names[kvar] = f"R[{q}]"
        for g, a, b, c, lut in gates:
            st.append(f"const uint32_t {pf}g{g} = lop3<0x{lut:02x}>({names[a]}, {names[b]}, {names[c]});")
            names[g] = f"{pf}g{g}"
        for o in range(4):
            pos = 4 * box + 4 - o  # FIPS position in the 32-bit S output
            p = pos_to_p[pos]
            if outs[o][0] == "f":
                # Feistel top: the output's last step h(a, b) merges into the
                # Feistel lop3; C moves to the FMA pipe (t3_cfix, 2 IMAD).
                _, a, b, h = outs[o]
                st.append(f"L[{p}] = t3_cfix(lop3<0x{feistel_lut(h):02x}>(L[{p}], {names[a]}, {names[b]}), k[{p}], fk);")
                continue
            g, inv = outs[o]
            lut = 0x69 if inv else 0x96  # a^b^c (or its complement)
            st.append(f"L[{p}] = lop3<0x{lut:02x}>(L[{p}], {names[g]}, k[{p}]);")
        streams.append((box, len(gates), st))
    if order == "box":
        for box, ng, st in streams:
            out.append(f"  {{  // S{box + 1}: {ng} lop3")
            out += ["    " + x for x in st]
            out.append("  }")
    else:
        groups = [streams] if order == "rr" else [streams[i:i + 2] for i in range(0, 8, 2)]
        out.append(f"  {{  // S-boxes interleaved ({order})")
        for grp in groups:
            for i in range(max(len(st) for _, _, st in grp)):
                for _, _, st in grp:
                    if i < len(st):
                        out.append("    " + st[i])
        out.append("  }")
    out.append("}")
    return out


def l_role(t: int) -> int:
    """0 if half A plays L in round t, else 1 (schedule.cpp build_bitslice_table)."""
    p, loc = divmod(t, 16)
    a = loc % 2
    return 1 - a if p == 1 else a


def gen_keyed_rounds(circuits) -> list[str]:
    """The key-specialised round as a template on the 48-bit
    round key K: the same circuits as gen_round, with each key bit folded into
    the lop3 immediates of the gates reading that S-box input (a key bit of 1
    complements the input: t3k_gate), so a round is the 186 S-box gates plus
    the 32 Feistel lop3 and nothing else — no key table, no whitening, no
    FMA-pipe corrections.  The immediates are constant expressions of K, so a
    compiler (NVRTC at run time, csrc/keyed.cpp) instantiating
    t3_keyed_round<K> for concrete keys emits plain LOP3s."""
    pos_to_p = {P[p]: p for p in range(32)}
    out = [
        "// key bit j (0-based FIPS subkey bit j+1, machine bit 47-j) of a round key; j < 0: none",
        "T3K_CE unsigned t3k_bit(uint64_t K, int j) { return j < 0 ? 0u : unsigned((K >> (47 - j)) & 1u); }",
        "// LUT of f(a ^ fa, b ^ fb, c ^ fc); fl bit 2/1/0 = fa/fb/fc",
        "T3K_CE unsigned t3k_flip(unsigned lut, unsigned fl) {",
        "    unsigned r = 0;",
        "    for (unsigned m = 0; m < 8; ++m) r |= ((lut >> (m ^ fl)) & 1u) << m;",
        "    return r;",
        "}",
        "T3K_CE unsigned t3k_gate(uint64_t K, unsigned lut, int ja, int jb, int jc) {",
        "    return t3k_flip(lut, (t3k_bit(K, ja) << 2) | (t3k_bit(K, jb) << 1) | t3k_bit(K, jc));",
        "}",
        "// Feistel top: L ^ h(a ^ ka, b ^ kb) as one lop3 over (L, a, b)",
        "T3K_CE unsigned t3k_ftop(uint64_t K, unsigned h, int ja, int jb) {",
        "    const unsigned fa = t3k_bit(K, ja), fb = t3k_bit(K, jb);",
        "    unsigned lut = 0;",
        "    for (unsigned m = 0; m < 8; ++m) {",
        "        const unsigned q = ((((m >> 1) & 1u) ^ fa) << 1) | ((m & 1u) ^ fb);",
        "        lut |= (((m >> 2) & 1u) ^ ((h >> q) & 1u)) << m;",
        "    }",
        "    return lut;",
        "}",
        "// 0 if half A plays L in round t, else 1 (passes 0 and 2 start with A, pass 1",
        "// with B: the pass swaps are role renaming, as in build_bitslice_table)",
        f"constexpr int T3K_ROLE[48] = {{{', '.join(str(l_role(t)) for t in range(48))}}};",
        "// L ^ (g ^ inv ^ kg): an output read from a gate (jg < 0) or an input",
        "T3K_CE unsigned t3k_direct(uint64_t K, unsigned inv, int jg) { return 0x3cu ^ ((inv ^ t3k_bit(K, jg)) ? 0xffu : 0u); }",
        "",
        "// One round L ^= f(R, K) with K folded into the immediates.",
        "template <uint64_t K>",
        "T3_FI void t3_keyed_round(uint32_t (&L)[32], const uint32_t (&R)[32]) {",
    ]
    for box in range(8):
        gates, outs = circuits[box]
        names, kj = {}, {}
        for kvar in range(6):
            j = 6 * box + 5 - kvar
            names[kvar] = f"R[{E[j] - 1}]"
            kj[kvar] = j
        out.append(f"    // S{box + 1}")
        for g, a, b, c, lut in gates:
            out.append(f"    const uint32_t s{box}g{g} = lop3<t3k_gate(K, 0x{lut:02x}, {kj.get(a, -1)}, {kj.get(b, -1)}, "
                       f"{kj.get(c, -1)})>({names[a]}, {names[b]}, {names[c]});")
            names[g] = f"s{box}g{g}"
        for o in range(4):
            p = pos_to_p[4 * box + 4 - o]
            if outs[o][0] == "f":
                _, a, b, h = outs[o]
                out.append(f"    L[{p}] = lop3<t3k_ftop(K, 0x{h:x}, {kj.get(a, -1)}, {kj.get(b, -1)})>(L[{p}], {names[a]}, {names[b]});")
            else:
                g, inv = outs[o]
                out.append(f"    L[{p}] = lop3<t3k_direct(K, {inv}, {kj.get(g, -1)})>(L[{p}], {names[g]}, 0u);")
    out.append("}")
    return out


def gen_gathers() -> list[str]:
    out = []
    # After IP: L_i = input bit IP[i-1], R_i = input bit IP[31+i]
    a = ", ".join(slice_of_fips_in(IP[i]) for i in range(32))
    b = ", ".join(slice_of_fips_in(IP[32 + i]) for i in range(32))
    out.append("// IP as renaming: half A = L0 (IP output bits 1..32), half B = R0.")
    out.append(f"#define T3_GATHER_A(lo, hi) {{ {a} }}")
    out.append(f"#define T3_GATHER_B(lo, hi) {{ {b} }}")
    # Output: preoutput = B || A (after the final pass swap); out FIPS bit f
    # = pre bit FP[f-1]; out lo slice k holds out FIPS bit 8*(k>>3)+8-(k&7).
    def pre(gbit):
        return f"B[{gbit - 1}]" if gbit <= 32 else f"A[{gbit - 33}]"

    lo, hi = [], []
    for k in range(32):
        f_lo = 8 * (k >> 3) + 8 - (k & 7)
        lo.append(pre(FP[f_lo - 1]))
        hi.append(pre(FP[32 + f_lo - 1]))
    out.append("// FP as renaming: output slice words from the final halves.")
    out.append(f"#define T3_SCATTER_LO(A, B) {{ {', '.join(lo)} }}")
    out.append(f"#define T3_SCATTER_HI(A, B) {{ {', '.join(hi)} }}")
    return out


def main() -> None:
    circuits = []
    total = 0
    ftops = 0
    # T3_GEN_FEISTEL_ALL=1 (testing): every output in Feistel-top form
    # h(a, b) = b, so the FMA-pipe C path runs for all 32 outputs.
    force = os.environ.get("T3_GEN_FEISTEL_ALL") == "1"
    for box in range(8):
        gates, outs = load_circuit(box)
        if force:
            for o in range(4):
                if outs[o][0] != "f":
                    g, inv = outs[o]
                    outs[o] = ("f", 0, g, 0x5 if inv else 0xA)
        ftops += sum(1 for o in range(4) if outs[o][0] == "f")
        verify_circuit(box, gates, outs)
        circuits.append((gates, outs))
        total += len(gates)
    prim_slot, secondary = e_slot_maps()
    gen_dir = os.path.join(HERE, "generated")
    os.makedirs(gen_dir, exist_ok=True)
    hdr = [
        "// GENERATED by csrc/gen_bitslice.py from csrc/sbox_circuits/*.txt — do not edit.",
        f"// S-box circuits: {total} lop3 in total ({total / 8:.2f} per S-box), each",
        "// verified exhaustively (64 inputs x 4 outputs) against the FIPS tables.",
        "#pragma once",
        f"#define T3_SBOX_LOP3_TOTAL {total}",
        f"// outputs whose last gate is merged into the Feistel lop3 (C on the FMA pipe)",
        f"#define T3_FEISTEL_TOPS {ftops}",
        "",
    ]
    body = hdr + gen_gathers() + [""] + gen_round(circuits) + [""]
    with open(os.path.join(gen_dir, "bitslice_rounds.cuh"), "w") as f:
        f.write("\n".join(body))
    tab = [
        "// GENERATED by csrc/gen_bitslice.py — do not edit.",
        "#pragma once",
        "// E expansion (FIPS, 1-based R bit per slot) and the whitening maps.",
        f"static const unsigned char T3_E[48] = {{{', '.join(map(str, E))}}};",
        "// primary E slot of R bit q (0-based)",
        f"static const unsigned char T3_PRIM_SLOT[32] = {{{', '.join(map(str, prim_slot))}}};",
        "// secondary (duplicated) E slots in D-constant order",
        f"static const unsigned char T3_SECONDARY_SLOT[16] = {{{', '.join(map(str, secondary))}}};",
        "",
    ]
    with open(os.path.join(gen_dir, "bitslice_tables.h"), "w") as f:
        f.write("\n".join(tab))
    # The keyed kernel has no whitening word C, so an output in Feistel-top
    # form h(a, b) merges into the Feistel lop3 for free: circuits searched
    # with free tops (tools/sboxgen SBOXGEN_FEISTEL=1 SBOXGEN_TOP_COST=0) that
    # are smaller by that measure live in sbox_circuits_keyed/ and replace the
    # shipped ones for the keyed rounds only.
    kcirc, ktotal = [], 0
    for box in range(8):
        path = os.path.join(HERE, "sbox_circuits_keyed", f"box{box}.txt")
        if os.path.exists(path) and os.environ.get("T3_GEN_KEYED_BASE") != "1":  # (A/B: shipped circuits)
            gates, outs = load_circuit(box, path)
            verify_circuit(box, gates, outs)
        else:
            gates, outs = circuits[box]
        kcirc.append((gates, outs))
        ktotal += len(gates)
    keyed = [
        "// GENERATED by csrc/gen_bitslice.py from csrc/sbox_circuits/*.txt and",
        "// csrc/sbox_circuits_keyed/*.txt — do not edit.",
        f"// {ktotal} S-box gates per round (Feistel tops merged into the 32 Feistel lop3).",
        "// Key-specialised rounds (SURVEY §8f-4): included by keyed_kernel.cuh, which",
        "// NVRTC compiles at run time for one key sequence (csrc/keyed.cpp).",
        "#pragma once",
        "#ifdef __CUDACC__",
        "#define T3K_CE __host__ __device__ constexpr",
        "#else",
        "#define T3K_CE constexpr",
        "#endif",
        "",
    ] + gen_keyed_rounds(kcirc) + [""]
    with open(os.path.join(gen_dir, "keyed_rounds.cuh"), "w") as f:
        f.write("\n".join(keyed))
    print(f"generated: {total} lop3 over 8 S-boxes", file=sys.stderr)


if __name__ == "__main__":
    main()
