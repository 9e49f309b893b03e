#!/bin/bash
# GPU tests + bench + reference arm + ncu launch list + ncu --set full of the
# shipped kernel.  Usage: TAG=r1b bash scripts/gpu_full.sh
cd "$GRAFT_REPO_ROOT" || exit 1
TAG=${TAG:-run}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 30 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?" >> gpurun_out/bench_$TAG.err
cat gpurun_out/bench_$TAG.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?" >> gpurun_out/bench_ref_$TAG.err
cat gpurun_out/bench_ref_$TAG.json
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$B > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $B > gpurun_out/ncu_bench.log 2>&1
echo "launch list rc=$?"
P="python scripts/profile_kernels.py"
$P bitslice bitslice_ldg > gpurun_out/plain_profile.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:t3_bs_tma_kernel -s 1 -c 1 -o gpurun_out/prof_bstma_$TAG $P bitslice > gpurun_out/ncu_full.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:t3_bs_kernel -s 1 -c 1 -o gpurun_out/prof_bsldg_$TAG $P bitslice_ldg > gpurun_out/ncu_full2.log 2>&1
echo "ncu full rc=$?"
cat gpurun_out/plain_profile.log
