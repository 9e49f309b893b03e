#!/bin/bash
# round-2 first GPU call: golden 64 GiB checksum from the reference, GPU tests, bench N=1 and N=2 (gloo, shared GPU)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
{ nproc; free -g; lscpu | grep -i "model name\|numa\|socket"; nvidia-smi --query-gpu=name,pci.bus_id,memory.total --format=csv; nvidia-smi topo -m; } > gpurun_out/host_info.txt 2>&1
timeout 900 python tests/golden/make_c3_checksum.py --out gpurun_out/c3_checksum.json > gpurun_out/golden.log 2>&1
cp gpurun_out/c3_checksum.json tests/golden/c3_checksum.json
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err
echo "bench rc=$?" >> gpurun_out/bench_n1.err
T3DES_BENCH_DIST_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 5 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
echo "bench2 rc=$?" >> gpurun_out/bench_n2.err
tail -3 gpurun_out/pytest_gpu.log
