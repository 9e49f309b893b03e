// Key-specialised bitsliced 3DES: the source NVRTC compiles
// at run time for one key sequence (csrc/keyed.cpp).  Before including this
// header the translation unit defines
//
//   constexpr uint64_t T3_KSEQ[T3_KROUNDS];  // round keys, execution order
//   constexpr int T3_KROUNDS;                // 48, or 16 for collapsed EDE
//
// and every round is t3_keyed_round<T3_KSEQ[t]> (generated/keyed_rounds.cuh):
// the key bits live in the LOP3 immediates, so the kernel reads no key table
// and runs no whitening or FMA-pipe key corrections.  The tile layout, IP/FP
// renaming and transposes are the table-driven kernel's (t3des_core.cuh).
//
// The 48 unrolled rounds are ~180 KB of SASS, more than the instruction
// caches hold, so warps that drift apart thrash them (measured: 3.26 ms/GiB
// with free-running 4-warp CTAs, profiles/r1/keyed_experiment_r1g.txt).  A
// CTA is therefore 16 warps, one per SM, re-aligned by CTA barriers pinned at
// the pass boundaries, so all warps of an SM fetch from one window of the
// code.  Every warp of the grid runs the same number of passes; a pass's
// tiles go warp-major over the CTAs, and in the last (partial) pass a warp
// past the last tile takes only the barriers, so the live warps are spread
// over all SMs and get their issue slots (+0.35%, keyed_ab5_r2z.jsonl).
//
// Also compiles as plain host C++ (tests/native/keyed_host.cpp): the rounds
// and tile function then run on the CPU for the parity tests.
#pragma once
#include "t3des_core.cuh"
#include "tma.cuh"
#include "generated/keyed_rounds.cuh"

#ifndef T3_KEYED_WARPS
#define T3_KEYED_WARPS 16  // warps per CTA (one CTA per SM)
#endif
// CTA barriers every T3K_SYNC rounds: at the pass boundaries (rounds 16 and
// 32) of the 48-round cipher, mid-way through a collapsed 16-round one.
#ifdef T3_KEYED_SYNC_EVERY  // (experiments)
constexpr int T3K_SYNC_EVERY = T3_KEYED_SYNC_EVERY;
#else
constexpr int T3K_SYNC_EVERY = 16;  // scripts/r2_keyed_ab{3,4}.sh
#endif
constexpr int T3K_SYNC = T3_KROUNDS <= T3K_SYNC_EVERY ? T3_KROUNDS / 2 : T3K_SYNC_EVERY;

#ifdef __CUDA_ARCH__
// A plain __syncthreads constrains no register dataflow, and ptxas hoists
// every one of them to the top of the cipher (measured: all BAR.SYNC within
// the first 0.5 KB of the ~180 KB body).  This barrier is pinned between its
// rounds by a data dependency instead: its predicate reads the state and its
// result feeds the state back through `z`, a kernel-parameter zero the
// compiler cannot fold (one SEL + one LOP3 per barrier).
#define T3_KEYED_SYNC_AB(A, B, z)                               \
    {                                                           \
        const int r_ = __syncthreads_or((B)[0] == 0x9E3779B9u); \
        (A)[0] ^= r_ ? (z) : 0u;                                \
    }
#else
#define T3_KEYED_SYNC_AB(A, B, z) ((void)(z))
#endif

template <int T>
T3_FI void t3_keyed_rounds(uint32_t (&A)[32], uint32_t (&B)[32], uint32_t z) {
    if constexpr (T < T3_KROUNDS) {
        if constexpr (T3K_ROLE[T] == 0)
            t3_keyed_round<T3_KSEQ[T]>(A, B);
        else
            t3_keyed_round<T3_KSEQ[T]>(B, A);
        if constexpr ((T + 1) % T3K_SYNC == 0 && T + 1 < T3_KROUNDS) T3_KEYED_SYNC_AB(A, B, z);
        t3_keyed_rounds<T + 1>(A, B, z);
    }
}

// 32 blocks per thread: lo/hi = the big-endian halves as loaded (t3_tile32)
T3_FI void t3_keyed_tile(uint32_t (&lo)[32], uint32_t (&hi)[32], uint32_t z = 0) {
    t3_transpose32<0>(lo);
    t3_transpose32<0>(hi);
    uint32_t A[32] = T3_GATHER_A(lo, hi);
    uint32_t B[32] = T3_GATHER_B(lo, hi);
    t3_keyed_rounds<0>(A, B, z);
    uint32_t olo[32] = T3_SCATTER_LO(A, B);
    uint32_t ohi[32] = T3_SCATTER_HI(A, B);
#pragma unroll
    for (int k = 0; k < 32; ++k) {
        lo[k] = olo[k];
        hi[k] = ohi[k];
    }
    t3_transpose32<0>(lo);
    t3_transpose32<0>(hi);
}

#ifdef __CUDACC__
// ntiles full 1024-block warp tiles of 16-byte aligned in/out; dynamic
// shared memory T3_KEYED_WARPS * 8 KiB (each warp's next tile streams in by
// TMA while it computes, as in t3_bs_tma_kernel).
extern "C" __global__ void __launch_bounds__(T3_KEYED_WARPS * 32, 1)
t3_keyed_kernel(const uint8_t* in, uint8_t* out, uint64_t ntiles, uint32_t zero) {
    extern __shared__ __align__(128) uint4 kslot[];  // [T3_KEYED_WARPS][512]
    __shared__ __align__(8) uint64_t bar[T3_KEYED_WARPS];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint64_t nwarps = uint64_t(gridDim.x) * T3_KEYED_WARPS;
    const uint64_t iters = (ntiles + nwarps - 1) / nwarps;  // the same for every warp: uniform barriers
    // a pass's tiles warp-major over the CTAs, so the live warps of the
    // last (partial) pass are spread over all SMs
    uint64_t tile = uint64_t(wib) * gridDim.x + blockIdx.x;
    const uint32_t sbar = t3_smem_addr(&bar[wib]);
    const uint32_t sdst = t3_smem_addr(&kslot[wib * 512]);
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (tile < ntiles) t3_tma_fetch(sdst, in + tile * (T3_TILE_BLOCKS * 8), T3_TILE_BLOCKS * 8, sbar);
    }
    __syncwarp();
    uint32_t parity = 0;
    for (uint64_t it = 0; it < iters; ++it, tile += nwarps) {
        const bool live = tile < ntiles;  // warp-uniform
        if (!live) {  // past the last tile: only the cipher's barriers (pass-uniform)
#pragma unroll 1
            for (int b = 0; b < (T3_KROUNDS - 1) / T3K_SYNC; ++b) (void)__syncthreads_or(0);
            continue;
        }
        t3_mbar_wait(sbar, parity);
        parity ^= 1u;
        uint32_t lo[32], hi[32];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const uint4 v = kslot[wib * 512 + 32 * j + lane];
            lo[2 * j] = v.x;
            hi[2 * j] = v.y;
            lo[2 * j + 1] = v.z;
            hi[2 * j + 1] = v.w;
        }
        __syncwarp();
        const uint64_t next = tile + nwarps;
        if (lane == 0 && next < ntiles) {
            // this warp's generic-proxy reads of the slot before the TMA overwrite
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            t3_tma_fetch(sdst, in + next * (T3_TILE_BLOCKS * 8), T3_TILE_BLOCKS * 8, sbar);
        }
        t3_keyed_tile(lo, hi, zero);
        uint4* dst = reinterpret_cast<uint4*>(out + tile * (T3_TILE_BLOCKS * 8)) + lane;
#pragma unroll
        for (int j = 0; j < 16; ++j)
            __stcs(dst + 32 * j, make_uint4(lo[2 * j], hi[2 * j], lo[2 * j + 1], hi[2 * j + 1]));
    }
}
#endif  // __CUDACC__
