"""The t3des_b200 CLI, mirroring the reference's CLI smoke test
(proj/tests/cli_smoke.cmake) and exit codes (t3des_cli.cpp:22-28)."""
import os
import subprocess

import pytest

from tests.oracle_util import ROOT

CLI = os.path.join(ROOT, "paper_1305_4376_b200", "t3des_b200")
KEY = "133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57"


@pytest.fixture(scope="module")
def cli(engine_lib):
    if not os.path.exists(CLI):
        subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "paper_1305_4376_b200", "csrc")])
    return CLI


def run(cli, *args, **kw):
    return subprocess.run([cli, *args], capture_output=True, **kw)


def test_usage_and_host_side_exit_codes(cli, tmp_path):
    f = tmp_path / "in.bin"
    f.write_bytes(b"\0" * 64)
    assert run(cli).returncode == 2
    assert run(cli, "--help").returncode == 0
    assert run(cli, "frobnicate").returncode == 2
    assert run(cli, "encrypt", "--nope", str(f), str(tmp_path / "x")).returncode == 2       # unknown flag
    assert run(cli, "encrypt", "--key", "zz23456789ABCDEF", str(f), str(tmp_path / "x")).returncode == 3
    assert run(cli, "encrypt", str(f), str(tmp_path / "x")).returncode == 3                 # no key
    assert run(cli, "encrypt", "--key", "0023456789ABCDEF", "--check-parity", str(f),
               str(tmp_path / "x")).returncode == 6
    assert run(cli, "encrypt", "--key", "0101010101010101", "--strict-keys", str(f),
               str(tmp_path / "x")).returncode == 3
    assert run(cli, "encrypt", "--key", KEY, str(tmp_path / "missing"), str(tmp_path / "x")).returncode == 1
    assert run(cli, "encrypt", "--key-file", str(tmp_path / "nokey"), str(f), str(tmp_path / "x")).returncode == 1
    assert run(cli, "bench", "--sweep", "nope").returncode == 2
    assert run(cli, "encrypt", "--key", KEY, "--backend", "threaded", str(f), str(tmp_path / "x")).returncode == 2


@pytest.mark.gpu
def test_cli_smoke_on_device(cli, oracle, tmp_path):
    import numpy as np

    data = b"0123456789abcdef" * 512 * 128  # 1 MiB, cli_smoke.cmake
    src, enc, dec = tmp_path / "in.bin", tmp_path / "enc.bin", tmp_path / "dec.bin"
    src.write_bytes(data)
    assert run(cli, "encrypt", "--key", KEY, str(src), str(enc)).returncode == 0
    assert run(cli, "decrypt", "--key", KEY, str(enc), str(dec)).returncode == 0
    assert dec.read_bytes() == data and enc.read_bytes() != data
    assert enc.read_bytes() == oracle.ecb(np.frombuffer(data, np.uint8), oracle.schedule_hex(KEY), 0).tobytes()
    assert run(cli, "encrypt", "--key", KEY, "--chunk-blocks", "4096", "--variant", "sptable", str(src),
               str(tmp_path / "enc2")).returncode == 0
    assert (tmp_path / "enc2").read_bytes() == enc.read_bytes()
    rag = tmp_path / "rag"
    rag.write_bytes(b"nine bytes!")
    assert run(cli, "encrypt", "--key", KEY, "--pkcs7", str(rag), str(tmp_path / "rag.enc")).returncode == 0
    assert run(cli, "decrypt", "--key", KEY, "--pkcs7", str(tmp_path / "rag.enc"),
               str(tmp_path / "rag.dec")).returncode == 0
    assert (tmp_path / "rag.dec").read_bytes() == b"nine bytes!"
    assert run(cli, "encrypt", "--key", KEY, str(rag), str(tmp_path / "x")).returncode == 4
    short = tmp_path / "short"
    short.write_bytes(b"123456789")
    assert run(cli, "decrypt", "--key", KEY, str(short), str(tmp_path / "x")).returncode == 4
    assert run(cli, "decrypt", "--key", KEY, "--pkcs7", str(enc), str(tmp_path / "x")).returncode == 5
    kf = tmp_path / "k.key"
    kf.write_text(KEY + "\n")
    assert run(cli, "encrypt", "--key-file", str(kf), str(src), str(tmp_path / "kf.enc")).returncode == 0
    assert (tmp_path / "kf.enc").read_bytes() == enc.read_bytes()
    # stdin/stdout
    p = run(cli, "encrypt", "--key", KEY, input=data)
    assert p.returncode == 0 and p.stdout == enc.read_bytes()
    v = run(cli, "verify")
    assert v.returncode == 0 and b"FAIL" not in v.stdout, v.stdout
    csv = tmp_path / "b.csv"
    b = run(cli, "bench", "--sweep", "chunk", "--values", "1024,131072", "--payload-mb", "8", "--reps", "1",
            "--out", str(csv))
    assert b.returncode == 0, b.stderr
    lines = csv.read_text().splitlines()
    assert lines[0] == ("backend,workers,chunk_blocks,work_group,payload_bytes,compute_seconds,io_seconds,"
                        "throughput_mb_s,speedup_vs_baseline,ok")
    assert len(lines) == 3 and all(l.endswith(",ok") for l in lines[1:])


@pytest.mark.gpu
def test_cli_bench_device_mode_on_last_device(cli, tmp_path):
    """`bench --mode device --device D` allocates, times and checks on device
    D (it used to allocate on the current device)."""
    import torch

    d = torch.cuda.device_count() - 1
    out = tmp_path / "b.csv"
    p = run(cli, "bench", "--mode", "device", "--device", str(d), "--sweep", "chunk", "--values", "0,65536",
            "--payload-mb", "8", "--reps", "1", "--format", "csv", "--out", str(out), timeout=300)
    assert p.returncode == 0, p.stderr
    rows = out.read_text().strip().splitlines()[1:]
    assert len(rows) == 2 and all(r.split(",")[-1] == "ok" for r in rows), rows
