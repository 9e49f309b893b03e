#!/bin/bash
# round-2 final evidence: GPU tests, bench N=1 (+ reference arm), N=2 gloo, smoke, ncu launch list of the bench
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out/final
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final/smoke.log
timeout 900 python bench.py --impl reference > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err
timeout 900 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err
T3DES_BENCH_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 > gpurun_out/final/bench_n2_gloo.json 2> gpurun_out/final/bench_n2.err
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launches.csv $B > gpurun_out/final/ncu_bench.log 2>&1
echo "ncu rc=$?" >> gpurun_out/final/ncu_bench.log
tail -2 gpurun_out/final/pytest_gpu.log
