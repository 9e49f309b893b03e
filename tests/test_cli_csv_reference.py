"""The CLI's bench CSV (paper_1305_4376_b200/t3des_b200 bench --format csv)
is the reference's own report format: the reference library's
bench::parse_csv reads it and bench::emit_report writes it back byte for byte
(proj/src/bench.cpp:151-232; the patched reference knows the "cuda" backend
name, integration/reference_backend_cuda.patch).  Uses GPU sweep CSVs the CLI
wrote on a B200 (profiles/r2/tables/).  CPU only; needs the reference headers
(build container) and the patched reference library."""
import glob
import os
import subprocess

import pytest

from tests.oracle_util import ROOT

REF_INC = "/root/reference/proj/include"
LIB = os.path.join(ROOT, "integration", "_build", "libt3des_ref_cuda.so")

DRIVER = r'''
#include <fstream>
#include <iostream>
#include <sstream>
#include "t3des/bench.hpp"
int main(int argc, char** argv) {
    std::ifstream f(argv[1]);
    std::stringstream ss;
    ss << f.rdbuf();
    const auto recs = t3des::bench::parse_csv(ss.str());
    std::cout << t3des::bench::emit_report(recs, t3des::bench::ReportFormat::Csv);
    return recs.empty() ? 2 : 0;
}
'''


@pytest.mark.skipif(not (os.path.isdir(REF_INC) and os.path.exists(LIB)),
                    reason="needs the reference headers and the patched reference library")
def test_cli_csv_round_trips_through_the_reference(tmp_path):
    src = tmp_path / "rt.cpp"
    src.write_text(DRIVER)
    exe = tmp_path / "rt"
    subprocess.check_call(["/usr/bin/g++", "-std=c++20", "-I" + REF_INC, str(src), LIB, "-fopenmp",
                           "-Wl,-rpath," + os.path.dirname(LIB), "-Wl,-rpath," + os.path.join(ROOT, "paper_1305_4376_b200"),
                           "-o", str(exe)])
    csvs = sorted(glob.glob(os.path.join(ROOT, "profiles", "r2", "tables", "table*_*.csv")))
    csvs = [c for c in csvs if "reference_cpu" not in c]
    assert csvs
    for c in csvs:
        with open(c) as f:
            text = f.read()
        p = subprocess.run([str(exe), c], capture_output=True, text=True, timeout=60)
        assert p.returncode == 0, (c, p.stderr)
        assert p.stdout == text, c
