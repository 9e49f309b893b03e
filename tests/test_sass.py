"""The shipped binary against the instruction counts the roofline quotes
(no GPU needed: cuobjdump reads the built sm_100a library).

bench.py reports `executed_alu_lane_ops_per_block` = 48 x (S-box LOP3 + 32)
/ 32 + the slice transposes / 32, computed from the generated S-box circuits;
these tests pin that figure to the SASS: the 2-round loop body issues exactly
2 x (T3_SBOX_LOP3_TOTAL + 32) LOP3 and nothing else on the ALU pipe, and the
tile prologue/epilogue (the four 32x32 transposes) 4 x 64 PRMT plus ~4 x 96
LOP3 and ~4 x 48 SHF.  Opcode histograms: profiles/r2/sass_histogram.txt
(scripts/sass_histogram.py)."""
import importlib.util
import os
import re
import shutil

import pytest

from tests.oracle_util import ROOT

spec = importlib.util.spec_from_file_location("sass_histogram", os.path.join(ROOT, "scripts", "sass_histogram.py"))
S = importlib.util.module_from_spec(spec)
spec.loader.exec_module(S)

pytestmark = pytest.mark.skipif(not shutil.which(S.CUOBJDUMP) and not os.path.exists(S.CUOBJDUMP),
                                reason="cuobjdump not available")


def sbox_total() -> int:
    with open(os.path.join(ROOT, "paper_1305_4376_b200", "csrc", "generated", "bitslice_rounds.cuh")) as f:
        return int(re.search(r"T3_SBOX_LOP3_TOTAL (\d+)", f.read()).group(1))


@pytest.fixture(scope="module")
def funcs(engine_lib):
    return S.sass_functions()


@pytest.mark.parametrize("label", ["bitsliced (shipped, OPT 5, 48 rounds)", "bitsliced, collapsed EDE (16 rounds)"])
def test_round_loop_body_lop3_count(funcs, label):
    ins = funcs[S.SHIPPED[label]]
    rl = S.round_loop(ins)
    body = rl["body"]
    assert body["LOP3"] == 2 * (sbox_total() + 32)
    # the rounds are pure LOP3 + FMA-pipe corrections: no shifts, byte
    # permutes or register moves on the ALU pipe
    assert body["SHF"] == 0 and body["PRMT"] == 0 and body.get("MOV", 0) == 0
    assert body["IMAD"] <= 2 * 24  # 16 E-duplicate corrections + whitening per round


def test_transposes_and_executed_alu_figure(funcs):
    ins = funcs[S.SHIPPED["bitsliced (shipped, OPT 5, 48 rounds)"]]
    rl = S.round_loop(ins)
    out = rl["outside"]
    assert out["PRMT"] == 4 * 64
    assert 4 * 96 <= out["LOP3"] <= 4 * 96 + 8
    assert 4 * 48 - 8 <= out["SHF"] <= 4 * 48 + 8
    per_block = 48 * (sbox_total() + 32) / 32 + (out["LOP3"] + out["PRMT"] + out["SHF"]) / 32
    import bench

    assert abs(per_block - bench.executed_alu_ops_per_block()) < 1.0, per_block


def test_tma_bulk_copy_in_shipped_kernel(funcs):
    h = S.histogram(funcs[S.SHIPPED["bitsliced (shipped, OPT 5, 48 rounds)"]])
    assert h["UBLKCP"] >= 1 and h["SYNCS"] >= 1  # cp.async.bulk + mbarrier
    assert h["LDS"] == 16 and h["STG"] == 16     # 16 x 128-bit per lane per tile
