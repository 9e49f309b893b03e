#!/usr/bin/env python3
"""Exact (SMT) resynthesis of S-box LUT3 circuits — an offline companion of
sboxgen.c for the bitsliced kernel's S-box circuits.

For a gate g of a circuit, its maximum fanout-free cone (MFFC: the gates that
die with g) is replaced by a smaller one if z3 finds a network of |MFFC| - 1
LUT3 gates computing tt[g] (or its complement: every consumer is a lop3 or
the Feistel lop3, which absorb an inversion) from any signals outside g's
cone and transitive fanout.  Signals are 64-bit truth tables over the six
S-box inputs, so the whole 64-point function is one bit-vector constraint.

Usage: exact_resyn.py <box> <circuit.txt> <out.txt> [timeout_s] [max_cone]
Writes <out.txt> whenever the circuit shrinks; the S-box tables are those of
gen_bitslice.py (FIPS 46-3; reference proj/src/des.cpp:43-75).
"""
from __future__ import annotations

import os
import sys
import time

import z3

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "paper_1305_4376_b200", "csrc"))
import gen_bitslice as G  # noqa: E402

M64 = (1 << 64) - 1


def lut_tt(lut, a, b, c):
    r = 0
    for m in range(8):
        if (lut >> m) & 1:
            r |= (a if m & 4 else ~a & M64) & (b if m & 2 else ~b & M64) & (c if m & 1 else ~c & M64)
    return r


class Circ:
    def __init__(self, gates, outs):
        self.gates = list(gates)  # (id, a, b, c, lut), ids 6.. in topological order
        self.outs = dict(outs)    # o -> (gate, inv)

    def tts(self):
        tt = {k: sum(1 << x for x in range(64) if (x >> k) & 1) for k in range(6)}
        for g, a, b, c, lut in self.gates:
            tt[g] = lut_tt(lut, tt[a], tt[b], tt[c])
        return tt

    def fanout(self):
        fo = {g: 0 for g, *_ in self.gates}
        for k in range(6):
            fo[k] = 0
        for g, a, b, c, _ in self.gates:
            for x in (a, b, c):
                fo[x] += 1
        for g, _ in self.outs.values():
            fo[g] += 1
        return fo

    def mffc(self, h):
        fo = self.fanout()
        cone = {h}
        uses = {}
        for g, a, b, c, _ in self.gates:
            for x in (a, b, c):
                uses.setdefault(x, []).append(g)
        outs = {g for g, _ in self.outs.values()}
        changed = True
        while changed:
            changed = False
            for g, a, b, c, _ in self.gates:
                if g not in cone:
                    continue
                for x in (a, b, c):
                    if x < 6 or x in cone or x in outs:
                        continue
                    if all(u in cone for u in uses.get(x, [])) and fo[x] == len(uses.get(x, [])):
                        cone.add(x)
                        changed = True
        return cone

    def tfo(self, h):
        t = {h}
        for g, a, b, c, _ in self.gates:
            if a in t or b in t or c in t:
                t.add(g)
        return t


def synth(cands, target, k, timeout_s):
    """Network of k LUT3 gates over the candidate truth tables computing
    target or ~target; returns [(sel_a, sel_b, sel_c, lut)] (selector indices
    into cands + earlier new gates) or None.

    Plain CNF (the usual exact-synthesis encoding): per new gate j, one-hot
    selectors s[j][p][i] for its 3 inputs, the input values v[j][p][t] and the
    output values x[j][t] at the 64 evaluation points, the 8 LUT bits f[j][m];
    candidate values are constants, so selecting candidate i for input p just
    fixes v[j][p][t] to c_i(t)."""
    n = len(cands)
    for inv in (0, M64):
        tgt = target ^ inv
        s = z3.SolverFor("QF_FD")
        s.set("timeout", int(timeout_s * 1000))
        B = z3.Bool
        x = [[B(f"x{j}_{t}") for t in range(64)] for j in range(k)]
        f = [[B(f"f{j}_{m}") for m in range(8)] for j in range(k)]
        sel = []
        for j in range(k):
            avail = n + j
            sj = []
            for p in range(3):
                bits = [B(f"s{j}_{p}_{i}") for i in range(avail)]
                s.add(z3.PbEq([(b_, 1) for b_ in bits], 1))
                v = [B(f"v{j}_{p}_{t}") for t in range(64)]
                for i in range(avail):
                    for t in range(64):
                        if i < n:
                            lit = v[t] if (cands[i] >> t) & 1 else z3.Not(v[t])
                            s.add(z3.Or(z3.Not(bits[i]), lit))
                        else:
                            xi = x[i - n][t]
                            s.add(z3.Or(z3.Not(bits[i]), v[t] == xi))
                sj.append((bits, v))
            # input order a < b < c: input p+1 may only pick i if input p picked i' < i
            for p in range(2):
                lo, hi = sj[p][0], sj[p + 1][0]
                for i in range(avail):
                    s.add(z3.Or(z3.Not(hi[i]), *[lo[i2] for i2 in range(i)]) if i > 0 else z3.Not(hi[0]))
            for t in range(64):
                va, vb, vc = sj[0][1][t], sj[1][1][t], sj[2][1][t]
                for m in range(8):
                    conds = [va if m & 4 else z3.Not(va), vb if m & 2 else z3.Not(vb), vc if m & 1 else z3.Not(vc)]
                    s.add(z3.Implies(z3.And(*conds), x[j][t] == f[j][m]))
            sel.append(sj)
        for t in range(64):
            s.add(x[k - 1][t] if (tgt >> t) & 1 else z3.Not(x[k - 1][t]))
        for j in range(k - 1):  # every new gate but the top feeds a later one
            s.add(z3.Or(*[sel[j2][p][0][n + j] for j2 in range(j + 1, k) for p in range(3)]))
        if s.check() != z3.sat:
            continue
        mdl = s.model()
        res = []
        for j in range(k):
            pick = [next(i for i, b_ in enumerate(sel[j][p][0]) if z3.is_true(mdl.eval(b_))) for p in range(3)]
            lv = sum(1 << m for m in range(8) if z3.is_true(mdl.eval(f[j][m])))
            res.append((pick[0], pick[1], pick[2], lv))
        return res
    return None


def splice(box, circ, h, cone, cand_ids, newg):
    """Replace h's cone by the new gates (placed after every candidate and
    before h's transitive fanout), redirect h's users to the new top, and
    restore each kept gate's function with LUT input flips where the top
    came out inverted.  Returns the renumbered circuit or None."""
    tt_old = circ.tts()
    tfo = circ.tfo(h) - {h}
    keep = [gt for gt in circ.gates if gt[0] not in cone]
    pre = [gt for gt in keep if gt[0] not in tfo]
    post = [gt for gt in keep if gt[0] in tfo]
    ids = list(cand_ids)
    added = []
    nxt = 10_000
    for (a, b, c, lut) in newg:
        added.append((nxt, ids[a], ids[b], ids[c], lut))
        ids.append(nxt)
        nxt += 1
    top = ids[-1]
    tt = {k: tt_old[k] for k in range(6)}
    gates = []
    for g, a, b, c, lut in pre + added + post:
        a, b, c = (top if x == h else x for x in (a, b, c))
        val = lut_tt(lut, tt[a], tt[b], tt[c])
        if g in tt_old and val != tt_old[g]:
            for flips in range(8):
                l2 = sum(((lut >> (m ^ flips)) & 1) << m for m in range(8))
                if lut_tt(l2, tt[a], tt[b], tt[c]) == tt_old[g]:
                    lut, val = l2, tt_old[g]
                    break
            else:
                return None
        tt[g] = val
        gates.append((g, a, b, c, lut))
    outs = {}
    for o in range(4):
        target = sum(((G.sbox_value(box, x) >> o) & 1) << x for x in range(64))
        g = circ.outs[o][0]
        g = top if g == h else g
        if tt[g] == target:
            outs[o] = (g, 0)
        elif tt[g] == ~target & M64:
            outs[o] = (g, 1)
        else:
            return None
    ren = {k: k for k in range(6)}
    out_gates = []
    for i, (g, a, b, c, lut) in enumerate(gates):
        ren[g] = 6 + i
        out_gates.append((6 + i, ren[a], ren[b], ren[c], lut))
    return Circ(out_gates, {o: (ren[g], inv) for o, (g, inv) in outs.items()})


def verify(box, circ):
    G.verify_circuit(box, circ.gates, circ.outs)


def dump(path, box, circ):
    with open(path, "w") as f:
        f.write(f"box {box} gates {len(circ.gates)}\n")
        for g, a, b, c, lut in circ.gates:
            f.write(f"g {g} {a} {b} {c} 0x{lut:02x}\n")
        for o in range(4):
            g, inv = circ.outs[o]
            f.write(f"o {o} {g} {inv}\n")


def sweep(circ):
    """Drop gates without fanout and renumber."""
    while True:
        fo = circ.fanout()
        dead = [g for g, *_ in circ.gates if fo[g] == 0]
        if not dead:
            break
        circ = Circ([gt for gt in circ.gates if gt[0] not in dead], circ.outs)
    ren = {k: k for k in range(6)}
    gates = []
    for i, (g, a, b, c, lut) in enumerate(circ.gates):
        ren[g] = 6 + i
        gates.append((6 + i, ren[a], ren[b], ren[c], lut))
    return Circ(gates, {o: (ren[g], inv) for o, (g, inv) in circ.outs.items()})


def improve_once(box, circ, timeout_s, max_cone, log):
    tt = circ.tts()
    hs = sorted({g for g, *_ in circ.gates}, reverse=True)
    for h in hs:
        cone = circ.mffc(h)
        k = len(cone)
        if k < 3 or k > max_cone:
            continue
        tfo = circ.tfo(h)
        cand_ids = [x for x in list(range(6)) + [g for g, *_ in circ.gates] if x not in cone and x not in tfo]
        t0 = time.time()
        res = synth([tt[x] for x in cand_ids], tt[h], k - 1, timeout_s)
        log(f"box {box} gate {h}: cone {k} over {len(cand_ids)} signals -> "
            f"{'found ' + str(k - 1) if res else 'no'} ({time.time() - t0:.1f} s)")
        if not res:
            continue
        c2 = splice(box, circ, h, cone, cand_ids, res)
        if c2 is None:
            log("  splice failed")
            continue
        c2 = sweep(c2)
        verify(box, c2)
        return c2
    return None


def main():
    box = int(sys.argv[1])
    src, dst = sys.argv[2], sys.argv[3]
    timeout_s = float(sys.argv[4]) if len(sys.argv) > 4 else 120
    max_cone = int(sys.argv[5]) if len(sys.argv) > 5 else 7
    gates, outs = G.load_circuit(box, src)
    circ = Circ(gates, outs)
    verify(box, circ)
    log = lambda m: print(m, file=sys.stderr, flush=True)
    log(f"box {box}: {len(circ.gates)} gates")
    while True:
        c2 = improve_once(box, circ, timeout_s, max_cone, log)
        if c2 is None:
            break
        circ = c2
        log(f"box {box}: now {len(circ.gates)} gates")
        dump(dst, box, circ)
    log(f"box {box}: done at {len(circ.gates)} gates")


if __name__ == "__main__":
    main()
