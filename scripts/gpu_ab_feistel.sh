#!/bin/bash
# A/B of the Feistel-top code path: the shipped generation vs every S-box
# output forced into the Feistel-top form (T3_GEN_FEISTEL_ALL=1: no gate
# saved, C applied as 32 extra IMADs per round on the FMA pipe).  Measures
# what the FMA-pipe C costs when nothing is gained on the ALU pipe.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-extra-configs"
timeout 300 $B > gpurun_out/ab_base.json 2> gpurun_out/ab_base.err; echo "base rc=$?"
T3_GEN_FEISTEL_ALL=1 python paper_1305_4376_b200/csrc/gen_bitslice.py
make -s -C paper_1305_4376_b200/csrc > gpurun_out/ab_make.log 2>&1; echo "make rc=$?"
timeout 300 $B > gpurun_out/ab_fall.json 2> gpurun_out/ab_fall.err; echo "fall rc=$?"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "kat or golden or edge" > gpurun_out/ab_fall_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/ab_fall_pytest.log
python - <<'PY'
import json
for n in ("ab_base", "ab_fall"):
    d = json.load(open(f"gpurun_out/{n}.json"))
    print(n, d["value"], d["variants"], d["roofline"]["alu_pipe_frac"])
PY
