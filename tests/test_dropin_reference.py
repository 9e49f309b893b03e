"""The drop-in, end to end: the reference library itself, patched with
integration/reference_backend_cuda.patch, runs its own encrypt_batch /
decrypt_batch / encrypt_stream / decrypt_stream on Backend::Cuda (the engine's
C ABI) and must match its own Backend::Threaded byte for byte."""
import os
import subprocess

import pytest

from tests.oracle_util import ROOT

BIN = os.path.join(ROOT, "integration", "_build", "dropin_check")
PATCH = os.path.join(ROOT, "integration", "reference_backend_cuda.patch")


def test_patch_is_small_and_targets_the_dispatch_layer():
    txt = open(PATCH).read()
    files = sorted({l.split()[1].split("/", 1)[1] for l in txt.splitlines() if l.startswith("+++ ")})
    assert files == ["include/t3des/dispatch.hpp", "src/bench.cpp", "src/dispatch.cpp", "tools/t3des_cli.cpp"]
    added = [l for l in txt.splitlines() if l.startswith("+") and not l.startswith("+++")]
    assert len(added) < 60


@pytest.mark.skipif(not os.path.exists(BIN), reason="patched reference not built (no /root/reference at build time)")
@pytest.mark.skipif("__import__('torch').cuda.is_available()")
def test_patched_reference_fails_loudly_without_a_device():
    p = subprocess.run([BIN], capture_output=True, text=True)
    assert p.returncode != 0 and "no usable sm_100 CUDA device" in p.stderr


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(BIN), reason="patched reference not built (no /root/reference at build time)")
def test_patched_reference_runs_on_the_engine():
    p = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0 and p.stdout.strip() == "ok", (p.stdout, p.stderr)
