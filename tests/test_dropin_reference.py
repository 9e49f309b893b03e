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
    assert files == ["CMakeLists.txt", "include/t3des/dispatch.hpp", "src/bench.cpp", "src/dispatch.cpp",
                     "tools/t3des_cli.cpp"]
    added = [l for l in txt.splitlines() if l.startswith("+") and not l.startswith("+++")]
    assert len(added) < 75


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj/src"), reason="needs the reference tree")
def test_patched_reference_builds_with_its_own_cmake():
    """The maintainer's path: the reference's own CMakeLists (patched:
    option T3DES_WITH_CUDA, T3DES_B200_ROOT) configures and builds its
    library and acceptance program against libt3des_b200.so."""
    import shutil

    if not shutil.which("cmake"):
        pytest.skip("cmake not installed")
    p = subprocess.run(["bash", os.path.join(ROOT, "integration", "cmake_patched_reference.sh")],
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, (p.stdout[-2000:], p.stderr[-2000:])
    assert "libt3des_b200.so" in p.stdout and "cmake build ok" in p.stdout


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
