"""NUMA placement helpers of the multi-GPU host path (hoststage.cpp:
parse_cpulist, numa_node_of_pci over sysfs, NumaBind), exercised on a fake
sysfs tree on CPU.  The GPU boxes of this run have one NUMA node, where the
helpers must be no-ops."""
import os
import subprocess

from tests.oracle_util import ROOT

CSRC = os.path.join(ROOT, "paper_1305_4376_b200", "csrc")


def _fake_sysfs(root, nodes: dict[int, str], dev_node: int):
    d = root / "bus" / "pci" / "devices" / "0000:1b:00.0"
    d.mkdir(parents=True)
    (d / "numa_node").write_text(f"{dev_node}\n")
    for k, cpus in nodes.items():
        nd = root / "devices" / "system" / "node" / f"node{k}"
        nd.mkdir(parents=True)
        (nd / "cpulist").write_text(cpus + "\n")
    return str(root)


def test_numa_helpers_on_fake_sysfs(tmp_path):
    if len(os.sched_getaffinity(0)) < 8 or not all(c in os.sched_getaffinity(0) for c in range(4, 8)):
        import pytest

        pytest.skip("needs CPUs 4-7 in this process's affinity mask")
    two = _fake_sysfs(tmp_path / "two", {0: "0-3", 1: "4-7"}, 1)
    one = _fake_sysfs(tmp_path / "one", {0: "0-7"}, 0)
    exe = tmp_path / "numa_host"
    subprocess.check_call(["/usr/bin/g++", "-std=c++17", "-O1", "-I" + CSRC, "-I/usr/local/cuda/include",
                           os.path.join(ROOT, "tests", "native", "numa_host.cpp"), os.path.join(CSRC, "hoststage.cpp"),
                           "-L/usr/local/cuda/lib64", "-lcudart", "-lpthread",
                           "-Wl,-rpath,/usr/local/cuda/lib64", "-o", str(exe)])
    p = subprocess.run([str(exe), two, one], capture_output=True, text=True, timeout=60)
    assert p.returncode == 0 and p.stdout.strip().endswith("ok"), p.stdout + p.stderr
