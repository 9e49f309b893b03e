"""SURVEY §8f-4, key-specialised kernels: MEASURED, NOT SHIPPED.

scripts/gen_keyed.py folds one key's 48 round keys into the lop3 immediates
of a fully unrolled cipher (gen_bitslice.gen_keyed_cipher); building the
engine with -DT3_KEYED_EXPERIMENT makes its TMA kernel run that cipher
(encrypt under that key only).  It measured equal to the shipped
table-driven kernel (2.67 vs 2.66 ms/GiB, profiles/r1/keyed_experiment_r1g.txt,
DESIGN §3.7), so it is not shipped; this test keeps the experiment buildable
and bit-exact so the finding stays reproducible.  The experiment library is
built into tests/native/_build/keyed/ (never the product path) and driven in
a subprocess."""
import os
import subprocess
import sys

import numpy as np
import pytest

from tests.oracle_util import ROOT

KEY = "133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57"
CSRC = os.path.join(ROOT, "paper_1305_4376_b200", "csrc")
OUT = os.path.join(ROOT, "tests", "native", "_build", "keyed", "libt3des_b200.so")

DRIVER = r'''
import ctypes, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from tests.oracle_util import Oracle
o = Oracle.load()
lib = ctypes.CDLL(sys.argv[2])
key = sys.argv[3]
s = o.schedule_hex(key)
ctx = ctypes.c_void_p()
assert lib.t3des_cu_create(0, ctypes.byref(ctx)) == 0
assert lib.t3des_cu_set_schedule(ctx, s) == 0
assert lib.t3des_cu_set_variant(ctx, 0) == 0   # BITSLICE -> the keyed kernel in this build
import torch
tiles = 148 * 16 * 2                              # every warp runs the same number of tiles
n = tiles * 1024
x = o.splitmix(0, n, 0x3DE5C0DE)
src = torch.from_numpy(x).cuda()
dst = torch.empty_like(src)
lib.t3des_cu_ecb_device.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
assert lib.t3des_cu_ecb_device(ctx, 0, src.data_ptr(), dst.data_ptr(), x.nbytes, None) == 0
torch.cuda.synchronize()
assert np.array_equal(dst.cpu().numpy(), o.ecb(x, s, 0)), "keyed cipher mismatch"
print("ok", n)
'''


def build_keyed() -> str:
    subprocess.check_call([sys.executable, os.path.join(ROOT, "scripts", "gen_keyed.py"), KEY])
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    if os.path.exists(OUT):
        os.remove(OUT)  # keyed.cuh is not a make dependency: force this one target
    subprocess.check_call(["make", "-s", "-C", CSRC, f"OUT={OUT}", f"LOG={OUT}.ptxas.log",
                           "EXTRA_NVFLAGS=-DT3_KEYED_EXPERIMENT", OUT], stdout=subprocess.DEVNULL)
    return OUT


def test_keyed_experiment_builds_for_sm100a():
    """The experiment compiles (nvcc cross-compiles; no GPU) and contains the
    keyed kernel."""
    lib = build_keyed()
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    assert "t3_bs_keyed_kernel" in sass


@pytest.mark.gpu
def test_keyed_experiment_bit_exact_on_device():
    lib = OUT if os.path.exists(OUT) else build_keyed()
    env = dict(os.environ, T3_KEYED_GRID="148")
    p = subprocess.run([sys.executable, "-c", DRIVER, ROOT, lib, KEY], capture_output=True, text=True, env=env,
                       timeout=600)
    assert p.returncode == 0 and p.stdout.startswith("ok"), p.stdout + p.stderr
