// Issue-rate microbenchmark for the instruction forms the bitsliced kernel
// uses: LOP3 with 3 register sources / an immediate / a constant-bank
// operand, IMAD in the same forms, and LOP3+IMAD interleaved.  Prints warp
// instructions per clock per SMSP (1.0 = one per cycle, 0.5 = half rate).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CHAINS 16
template <int FORM>
__global__ void __launch_bounds__(256) k(uint32_t* out, int iters, uint32_t cval) {
    uint32_t x[CHAINS], y = threadIdx.x * 0x9E3779B9u, z = threadIdx.x ^ 0x5bd1e995u;
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) x[i] = threadIdx.x * (i + 1);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CHAINS; ++i) {
            if (FORM == 0) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[i]) : "r"(y), "r"(z));
            if (FORM == 1) asm volatile("lop3.b32 %0, %0, %1, 0x0F0F0F0F, 0xE4;" : "+r"(x[i]) : "r"(y));
            if (FORM == 2) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[i]) : "r"(y), "r"(cval));
            if (FORM == 3) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[i]) : "r"(y), "r"(z));
            if (FORM == 4) asm volatile("mad.lo.u32 %0, %0, 3, %1;" : "+r"(x[i]) : "r"(z));
            if (FORM == 5) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[i]) : "r"(cval), "r"(z));
            if (FORM == 6) {  // LOP3 and IMAD interleaved 1:1 (independent)
                if (i & 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[i]) : "r"(cval), "r"(z));
                else asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[i]) : "r"(y), "r"(z));
            }
            if (FORM == 7) {  // LOP3 : IMAD = 3 : 1
                if ((i & 3) == 3) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[i]) : "r"(cval), "r"(z));
                else asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[i]) : "r"(y), "r"(z));
            }
            if (FORM == 8) asm volatile("lop3.b32 %0, %0, %1, 0, 0x3C;" : "+r"(x[i]) : "r"(y));  // 2-input xor
            if (FORM == 9) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(x[i]) : "r"(cval));  // IMAD.HI
            if (FORM == 10) {  // IMAD.WIDE: 64-bit product, both halves kept live
                uint64_t w;
                asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(w) : "r"(x[i]), "r"(cval));
                x[i] = uint32_t(w) ^ uint32_t(w >> 32);
            }
            if (FORM == 11) {  // LOP3 and IMAD.HI interleaved 1:1
                if (i & 1) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(x[i]) : "r"(cval));
                else asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[i]) : "r"(y), "r"(z));
            }
            if (FORM == 12) {  // LOP3 : IMAD.SHL-style mad by a register power of two, 1:1
                if (i & 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[i]) : "r"(cval), "r"(z));
                else asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[i]) : "r"(y), "r"(z));
            }
        }
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) s ^= x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int FORM>
void run(const char* name, uint32_t* d, int sms, int clk_khz) {
    const int iters = 4096, grid = sms * 8, block = 256;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k<FORM><<<grid, block>>>(d, 16, 7u);
    cudaEventRecord(a);
    k<FORM><<<grid, block>>>(d, iters, 7u);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double warp_instr = double(grid) * (block / 32) * iters * CHAINS;
    const double cycles = ms * 1e-3 * clk_khz * 1e3;
    printf("%-34s %8.3f ms  %.3f warp-instr/clk/SMSP\n", name, ms, warp_instr / (cycles * sms * 4));
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("%s, %d SMs, clock %d MHz (assumed during the run)\n", p.name, p.multiProcessorCount, clk / 1000);
    uint32_t* d;
    cudaMalloc(&d, 1 << 24);
    run<0>("LOP3 R,R,R,R", d, p.multiProcessorCount, clk);
    run<1>("LOP3 R,R,imm,R", d, p.multiProcessorCount, clk);
    run<2>("LOP3 R,R,R,c[] (param)", d, p.multiProcessorCount, clk);
    run<8>("LOP3 R,R,imm0 (2-input xor)", d, p.multiProcessorCount, clk);
    run<3>("IMAD R,R,R,R", d, p.multiProcessorCount, clk);
    run<4>("IMAD R,R,imm,R", d, p.multiProcessorCount, clk);
    run<5>("IMAD R,R,c[],R (param)", d, p.multiProcessorCount, clk);
    run<6>("LOP3 + IMAD 1:1", d, p.multiProcessorCount, clk);
    run<7>("LOP3 + IMAD 3:1", d, p.multiProcessorCount, clk);
    run<9>("IMAD.HI R,R,R (mul.hi)", d, p.multiProcessorCount, clk);
    run<10>("IMAD.WIDE R,R,R (+lop3 fold)", d, p.multiProcessorCount, clk);
    run<11>("LOP3 + IMAD.HI 1:1", d, p.multiProcessorCount, clk);
    return 0;
}
