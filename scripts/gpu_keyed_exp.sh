#!/bin/bash
# Experiment: key-specialised (fully unrolled, key folded into lop3
# immediates) cipher vs the table-driven shipped kernel, bench key, 1 GiB.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python scripts/profile_kernels.py bitslice > gpurun_out/keyed_base.log 2>&1
python scripts/gen_keyed.py
make -B -s -C paper_1305_4376_b200/csrc EXTRA_NVFLAGS=-DT3_KEYED_EXPERIMENT > gpurun_out/keyed_make.log 2>&1; echo "make rc=$?"
python scripts/profile_kernels.py bitslice > gpurun_out/keyed_exp.log 2>&1
python - <<'PY' > gpurun_out/keyed_check.log 2>&1
import torch, paper_1305_4376_b200 as t3
e = t3.Engine(0)
e.set_schedule(t3.triple_schedule(t3.parse_hex_key("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57")))
n = (64 << 20) // 8
src = torch.empty(8 * n, dtype=torch.uint8, device="cuda"); s = torch.cuda.current_stream().cuda_stream
e.fill_splitmix(src.data_ptr(), 0, n, 1234, s)
a = torch.empty_like(src); b = torch.empty_like(src)
e.set_variant(t3.VARIANT_BITSLICE); e.ecb_device(0, src.data_ptr(), a.data_ptr(), 8 * n, s)
e.set_variant(t3.VARIANT_SPTABLE); e.ecb_device(0, src.data_ptr(), b.data_ptr(), 8 * n, s)
torch.cuda.synchronize()
print("keyed == sptable:", bool(torch.equal(a, b)))
PY
cat gpurun_out/keyed_check.log
ncu --set full --clock-control none -k regex:t3_bs_tma_kernel -s 1 -c 1 -o gpurun_out/prof_keyed python scripts/profile_kernels.py bitslice > gpurun_out/keyed_ncu.log 2>&1; echo "ncu rc=$?"
cat gpurun_out/keyed_base.log gpurun_out/keyed_exp.log
