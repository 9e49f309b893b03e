#!/bin/bash
# round-2 GPU call 2: e2e ceiling probe; ncu launch list of bench.py and full captures of the two kernels
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 600 python scripts/e2e_ceiling_probe.py > gpurun_out/e2e_probe.jsonl 2> gpurun_out/e2e_probe.err
echo "probe rc=$?"
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 $B > gpurun_out/plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2.csv $B > gpurun_out/ncu_bench.log 2>&1
echo "launch list rc=$?"
P="python scripts/profile_kernels.py"
timeout 300 $P > gpurun_out/plain_profile.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:t3_bs_tma_kernel -s 1 -c 1 -o gpurun_out/prof_bstma_r2 $P bitslice > gpurun_out/ncu_full_bs.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:t3_sp_kernel -s 1 -c 1 -o gpurun_out/prof_sp_r2 $P sptable > gpurun_out/ncu_full_sp.log 2>&1
echo "ncu full rc=$?"
ls -la gpurun_out
