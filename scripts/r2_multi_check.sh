#!/bin/bash
# N>1 bench paths on a one-GPU box: gloo ranks sharing the GPU, self-launched; reference arm at N=2; smoke
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
T3DES_BENCH_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 5 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo "n2 rc=$?"
T3DES_BENCH_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 4 --steps 5 --no-e2e > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err; echo "n4 rc=$?"
timeout 900 python bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/bench_ref_n2.json 2> gpurun_out/bench_ref_n2.err; echo "ref n2 rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
