#!/bin/bash
# Where the CLI's wall clock goes: process + CUDA start-up vs the stream work.
cd "$GRAFT_REPO_ROOT" || exit 1
K=133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57
C=paper_1305_4376_b200/t3des_b200
printf 'abcdefgh' > /tmp/t3_8.bin
t() { local s=$(date +%s.%N); "$@" > /dev/null 2>&1; local rc=$?; local e=$(date +%s.%N); echo "rc=$rc $(python -c "print(f'{$e-$s:.3f} s')") : $*"; }
for i in 1 2 3; do t $C encrypt --key $K /tmp/t3_8.bin /tmp/t3_8.out; done
t $C verify
t nvidia-smi -L
CUDA_MODULE_LOADING=EAGER t $C encrypt --key $K /tmp/t3_8.bin /tmp/t3_8.out
CUDA_MODULE_LOADING=LAZY t $C encrypt --key $K /tmp/t3_8.bin /tmp/t3_8.out
cat > /tmp/init.cu <<'CU'
#include <cuda_runtime.h>
#include <cstdio>
#include <chrono>
int main() { auto a = std::chrono::steady_clock::now(); cudaFree(0); auto b = std::chrono::steady_clock::now();
  printf("cudaFree(0) init: %.3f s\n", std::chrono::duration<double>(b - a).count()); }
CU
nvcc -o /tmp/init /tmp/init.cu && t /tmp/init && /tmp/init
T3DES_TRACE_INIT=1 $C encrypt --key $K /tmp/t3_8.bin /tmp/t3_8.out
