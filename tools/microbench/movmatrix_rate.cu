// microbenchmark: LOP3 chains alone vs interleaved with movmatrix / PRMT
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(uint32_t* out, int iters) {
    uint32_t x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 0x9E3779B9u + i;
    uint32_t y = threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[i]) : "r"(x[(i + 1) & 7]), "r"(x[(i + 3) & 7]));
            if (MODE == 1 && (i & 1) == 0) asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %0;" : "+r"(y));
            if (MODE == 2 && (i & 1) == 0) asm volatile("prmt.b32 %0, %0, %1, 0x5410;" : "+r"(y) : "r"(x[i]));
            if (MODE == 3) asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %0;" : "+r"(y));
        }
    }
    uint32_t s = y;
    for (int i = 0; i < 8; ++i) s ^= x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    uint32_t* d;
    cudaMalloc(&d, 148 * 8 * 256 * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 4096;
    const char* names[] = {"lop3 only (8 per iter)", "lop3 + movmatrix 2:1 (4 per iter)", "lop3 + prmt 2:1", "lop3 + movmatrix 1:1"};
    for (int mode = 0; mode < 4; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            if (mode == 0) k<0><<<148 * 8, 256>>>(d, iters);
            if (mode == 1) k<1><<<148 * 8, 256>>>(d, iters);
            if (mode == 2) k<2><<<148 * 8, 256>>>(d, iters);
            if (mode == 3) k<3><<<148 * 8, 256>>>(d, iters);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep) printf("%-36s %.3f ms  (lop3 warp-instr/clk/SMSP at 1.965 GHz: %.3f)\n", names[mode], ms,
                            148.0 * 8 * 8 * 8.0 * iters / 4 / 148 / (ms * 1e-3 * 1.965e9));
        }
    }
    return 0;
}
