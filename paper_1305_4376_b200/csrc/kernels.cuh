// sm_100a kernels of the B200 3DES-ECB engine.
//
//   t3_bs_tma_kernel  bitsliced 3DES, the shipped kernel: one warp owns a
//                 tile of 1024 blocks (8 KiB), each thread 32 blocks held as
//                 64 slice words; the warp's next tile streams into shared
//                 memory by TMA (cp.async.bulk) while it computes; the rounds
//                 are LOP3 circuits on the integer pipe with key/whitening
//                 constants from constant bank 0 (__grid_constant__ table).
//   t3_bs_kernel  the same cipher with direct 128-bit (or 64-bit, for
//                 8-byte-aligned buffers) loads, and the predicated tail tile.
//   t3_sp_kernel  SP-table variant (measured alternative; AUTO uses it for
//                 small launches and partial tiles): one block per thread per
//                 step, the 8 fused S/P tables replicated per lane in shared
//                 memory (64 KiB, bank = lane: conflict-free).
//   helpers       splitmix payload generator, order-sensitive checksum.
//
// Replaces the reference's Threaded backend inner loop
// (/root/reference/proj/src/dispatch.cpp:60-86 -> run_blocks_fast :47-56
// -> tdes_{en,de}crypt_block_fast, tdes.cpp:177-185).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "t3des_core.cuh"
#include "tma.cuh"

#ifndef T3_BS_THREADS
#define T3_BS_THREADS 128  // CTA size of the bitsliced kernels
#endif
#ifndef T3_BS_MIN_CTAS
#define T3_BS_MIN_CTAS 4  // resident CTAs per SM the register budget is sized for
#endif
#define T3_SP_THREADS 256        // SP-table CTA size for small batches
#define T3_SP_THREADS_BIG 1024  // ... and for batches of >= 16384 blocks
#ifndef T3_OPT_DEFAULT
#define T3_OPT_DEFAULT T3_OPT_DFMA  // for the LDG/tail kernels; the TMA kernel's mask is per context
#endif

// ---- bitsliced kernel --------------------------------------------------
// VEC = 4: lane t of the warp loads blocks (64j + 2t, 64j + 2t + 1), j < 16,
//          with one LDG.128 per j (512 contiguous bytes per instruction).
// VEC = 2: lane t loads block 32k + t, k < 32, with LDG.64.
// TAIL:    the final partial tile; missing blocks read as zero and are not
//          stored (only VEC = 2).
template <int VEC, bool TAIL, int OPT = T3_OPT_DEFAULT>
__global__ void __launch_bounds__(T3_BS_THREADS, T3_BS_MIN_CTAS)
t3_bs_kernel(const uint8_t* in, uint8_t* out, uint64_t first_tile, uint64_t ntiles,
             uint64_t nblocks, const __grid_constant__ T3BsTable tab) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t tile = first_tile + warp; tile < first_tile + ntiles; tile += nwarps) {
        const uint64_t base = tile * T3_TILE_BLOCKS;
        uint32_t lo[32], hi[32];
        if (VEC == 4) {
            const uint4* src = reinterpret_cast<const uint4*>(in + base * 8) + lane;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const uint4 v = __ldcs(src + 32 * j);
                lo[2 * j] = v.x;
                hi[2 * j] = v.y;
                lo[2 * j + 1] = v.z;
                hi[2 * j + 1] = v.w;
            }
        } else {
            const uint2* src = reinterpret_cast<const uint2*>(in + base * 8) + lane;
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                uint2 v = make_uint2(0u, 0u);
                if (!TAIL || base + 32 * k + lane < nblocks) v = __ldcs(src + 32 * k);
                lo[k] = v.x;
                hi[k] = v.y;
            }
        }
        t3_tile32<OPT>(lo, hi, tab.w);
        if (VEC == 4) {
            uint4* dst = reinterpret_cast<uint4*>(out + base * 8) + lane;
#pragma unroll
            for (int j = 0; j < 16; ++j)
                __stcs(dst + 32 * j, make_uint4(lo[2 * j], hi[2 * j], lo[2 * j + 1], hi[2 * j + 1]));
        } else {
            uint2* dst = reinterpret_cast<uint2*>(out + base * 8) + lane;
#pragma unroll
            for (int k = 0; k < 32; ++k)
                if (!TAIL || base + 32 * k + lane < nblocks) __stcs(dst + 32 * k, make_uint2(lo[k], hi[k]));
        }
    }
}

// ---- bitsliced kernel with TMA prefetch (aligned full tiles) ----------
// OPT (T3_OPT_* bitmask) selects which small pieces of work move from the
// saturated ALU pipe to the FMA pipe; T3_OPT_DEFAULT is the measured best.
// Each warp owns an 8 KiB shared-memory slot and an mbarrier.  While the
// warp runs the 48 rounds of tile t, the TMA engine (cp.async.bulk, SASS
// UBLKCP) streams tile t+1 from HBM into the slot, so the warps' load phases
// never stall the integer pipe (without it all warps of an SM reach their
// loads in lockstep and the ALU idles ~10%, ncu profiles/r1).  Requires
// 16-byte aligned in/out.
template <int OPT, int ROUNDS = 48>
__global__ void __launch_bounds__(T3_BS_THREADS, T3_BS_MIN_CTAS)
t3_bs_tma_kernel(const uint8_t* in, uint8_t* out, uint64_t ntiles, const __grid_constant__ T3BsTable tab) {
    __shared__ __align__(128) uint4 slot[T3_BS_THREADS / 32][T3_TILE_BLOCKS / 2];
    __shared__ __align__(8) uint64_t bar[T3_BS_THREADS / 32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    uint64_t tile = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint32_t sbar = t3_smem_addr(&bar[wib]);
    const uint32_t sdst = t3_smem_addr(&slot[wib][0]);
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (tile < ntiles) t3_tma_fetch(sdst, in + tile * (T3_TILE_BLOCKS * 8), T3_TILE_BLOCKS * 8, sbar);
    }
    __syncwarp();
    uint32_t parity = 0;
    for (; tile < ntiles; tile += nwarps) {
        t3_mbar_wait(sbar, parity);
        parity ^= 1u;
        uint32_t lo[32], hi[32];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const uint4 v = slot[wib][32 * j + lane];
            lo[2 * j] = v.x;
            hi[2 * j] = v.y;
            lo[2 * j + 1] = v.z;
            hi[2 * j + 1] = v.w;
        }
        __syncwarp();
        const uint64_t next = tile + nwarps;
        if (lane == 0 && next < ntiles) {
            // order this warp's generic-proxy reads of the slot before the
            // async-proxy (TMA) overwrite
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            t3_tma_fetch(sdst, in + next * (T3_TILE_BLOCKS * 8), T3_TILE_BLOCKS * 8, sbar);
        }
        t3_tile32<OPT, ROUNDS>(lo, hi, tab.w);
        uint4* dst = reinterpret_cast<uint4*>(out + tile * (T3_TILE_BLOCKS * 8)) + lane;
#pragma unroll
        for (int j = 0; j < 16; ++j)
            __stcs(dst + 32 * j, make_uint4(lo[2 * j], hi[2 * j], lo[2 * j + 1], hi[2 * j + 1]));
    }
}

// ---- SP-table kernel ---------------------------------------------------
__device__ __forceinline__ void t3_dswap(uint32_t& a, uint32_t& b, int s, uint32_t m) {
    const uint32_t w = ((a >> s) ^ b) & m;
    b ^= w;
    a ^= w << s;
}

// Code-generation options of the SP-table kernel (template bitmask SPV).
// Per round the kernel extracts 8 six-bit windows of R (rotate), XORs the
// round-key chunk and masks (one lop3), adds the lane's table column, loads,
// and merges the 8 table words into L.  Everything but the loads runs on the
// ALU pipe unless these options move work to the (otherwise idle) FMA pipe.
// Measured (scripts/sp_variant_sweep.py, profiles/r1/sp_variants_r1k.txt).
enum : int {
    T3_SPV_LANEFMA = 1,  // lane column added as IMAD (else a lop3 OR)
    T3_SPV_MERGE6 = 2,   // the 8 table words summed by 6 IMADs (disjoint bits: + = |), 1 lop3 into L
    T3_SPV_MERGE4 = 4,   // 4 IMADs + 2 lop3 (else 4 lop3)
    T3_SPV_SHLFMA = 8,   // S-box 6's window (a left shift by 4) as IMAD, else a funnel rotate
    T3_SPV_SHRFMA = 16,  // S-boxes 1-4 windows (right shifts) as IMAD.HI, else funnel rotates
    T3_SPV_KEYPARAM = 32, // 48 rounds unrolled, round keys as uniform constant-bank operands (LDCU)
    T3_SPV_KEY2 = 64,     // key XOR on R (2 words, t3b::SpKeys::k2) instead of on the 8 windows;
                          // the lane column then merges into the mask lop3
    T3_SPV_PREFETCH = 128, // a thread's first block loaded before the table fill, each next
                           // block before the current one's rounds
    T3_SPV_PDL = 256,      // programmatic dependent launch: the table fill overlaps the previous
                           // kernel on the stream; input is touched only after griddepcontrol.wait
};

// Opaque multipliers of the FMA-pipe forms (kernel parameter: ptxas cannot
// strength-reduce a multiply by an unknown value back into an ALU shift/OR).
struct T3SpMul {
    uint32_t one;   // 1
    uint32_t m[8];  // S-box i: 2^(32-s) for the right shift s = 20-4i (i = 1..4), 16 for i = 6
};

__device__ __forceinline__ uint32_t t3_mad(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}
__device__ __forceinline__ uint32_t t3_mulhi(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}

// Shared-memory table layout: word (i * 64 + six) * 32 + lane, i.e. byte
// offset i*8192 + six*128 + lane*4.  Keys arrive pre-shifted to bits 7..12.
// Returns L ^ f(R, k) (f = the fused S/P round function).
template <int SPV>
__device__ __forceinline__ uint32_t t3_sp_round(uint32_t l, uint32_t r, const uint32_t* ks, const char* smem,
                                                uint32_t lane4, const T3SpMul& mul) {
    // the round's 8 key words: two broadcast LDS.128 (shared) or uniform
    // constant-bank operands (kernel parameter, compile-time round index)
    if (SPV & T3_SPV_KEY2) {  // ks -> {Ka, Kb}
        const uint32_t ra = r ^ ks[0], rb = r ^ ks[1];
        uint32_t v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint32_t ri = (i & 1) ? rb : ra;
            uint32_t y;
            if ((SPV & T3_SPV_SHLFMA) && i == 6)
                y = t3_mad(ri, mul.m[6], 0u);  // ri << 4
            else
                y = __funnelshift_r(ri, ri, (20 - 4 * i) & 31);
            const uint32_t col = (y & 0x1F80u) | lane4;  // one lop3
            v[i] = *reinterpret_cast<const uint32_t*>(smem + i * 8192 + col);
        }
        if (SPV & T3_SPV_MERGE6) {
            const uint32_t a = t3_mad(t3_mad(v[0], mul.one, v[1]), mul.one, t3_mad(v[2], mul.one, v[3]));
            const uint32_t b = t3_mad(t3_mad(v[4], mul.one, v[5]), mul.one, t3_mad(v[6], mul.one, v[7]));
            return l ^ a ^ b;
        }
        if (SPV & T3_SPV_MERGE4) {
            const uint32_t a = t3_mad(v[0], mul.one, v[1]), b = t3_mad(v[2], mul.one, v[3]);
            const uint32_t c = t3_mad(v[4], mul.one, v[5]), d = t3_mad(v[6], mul.one, v[7]);
            return l ^ (a | b | c) ^ d;
        }
        return l ^ ((v[0] | v[1] | v[2]) | (v[3] | v[4] | v[5]) | (v[6] | v[7]));
    }
    uint32_t k[8];
    if (SPV & T3_SPV_KEYPARAM) {
#pragma unroll
        for (int i = 0; i < 8; ++i) k[i] = ks[i];
    } else {
        const uint4 ka = reinterpret_cast<const uint4*>(ks)[0], kb = reinterpret_cast<const uint4*>(ks)[1];
        k[0] = ka.x, k[1] = ka.y, k[2] = ka.z, k[3] = ka.w, k[4] = kb.x, k[5] = kb.y, k[6] = kb.z, k[7] = kb.w;
    }
    uint32_t v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        // E window of S-box i moved so its 6 bits sit at bits 7..12.
        uint32_t y;
        if ((SPV & T3_SPV_SHRFMA) && i >= 1 && i <= 4)
            y = t3_mulhi(r, mul.m[i]);  // r >> (20 - 4i)
        else if ((SPV & T3_SPV_SHLFMA) && i == 6)
            y = t3_mad(r, mul.m[6], 0u);  // r << 4
        else
            y = __funnelshift_r(r, r, (20 - 4 * i) & 31);
        const uint32_t off = (y ^ k[i]) & 0x1F80u;
        const uint32_t col = (SPV & T3_SPV_LANEFMA) ? t3_mad(off, mul.one, lane4) : (off | lane4);
        v[i] = *reinterpret_cast<const uint32_t*>(smem + i * 8192 + col);
    }
    // the 8 words have disjoint bits (each S-box owns 4 output bits): sums are ORs
    if (SPV & T3_SPV_MERGE6) {
        const uint32_t a = t3_mad(t3_mad(v[0], mul.one, v[1]), mul.one, t3_mad(v[2], mul.one, v[3]));
        const uint32_t b = t3_mad(t3_mad(v[4], mul.one, v[5]), mul.one, t3_mad(v[6], mul.one, v[7]));
        return l ^ a ^ b;
    }
    if (SPV & T3_SPV_MERGE4) {
        const uint32_t a = t3_mad(v[0], mul.one, v[1]), b = t3_mad(v[2], mul.one, v[3]);
        const uint32_t c = t3_mad(v[4], mul.one, v[5]), d = t3_mad(v[6], mul.one, v[7]);
        return l ^ (a | b | c) ^ d;
    }
    return l ^ ((v[0] | v[1] | v[2]) | (v[3] | v[4] | v[5]) | (v[6] | v[7]));
}

// The 48 x 8 round-key words are staged in shared memory next to the tables
// (from a device copy): read from the constant bank, every round's keys miss
// the constant cache once per CTA, which dominates small launches.
#define T3_SPK(kp, t) ((SPV & T3_SPV_KEY2) ? (kp).k2[t] : (kp).k[t])
#define T3_SKS(t) ((SPV & T3_SPV_KEY2) ? ks2 + 2 * (t) : ks + 8 * (t))
template <int SPV>
__global__ void __launch_bounds__(1024)
t3_sp_kernel(const uint2* in, uint2* out, uint64_t nblocks, const uint32_t* __restrict__ sp_global,
             int passes, const uint32_t* __restrict__ keys_global, const __grid_constant__ T3SpMul mul,
             const __grid_constant__ T3SpKeyParam kp, int pdl) {
    extern __shared__ __align__(16) uint32_t t3_sp_smem[];
    uint32_t* ks = t3_sp_smem + 8 * 64 * 32;  // [48][8]
    uint32_t* sp = ks + sizeof(T3SpKeyParam) / 4;  // the 2 KiB table, staged once
    // one global round trip: every thread issues its few loads together, then
    // the 32-fold lane replication is a shared-memory copy (a fill loop of 64
    // dependent-latency global loads per thread cost ~7 us per launch)
    if (SPV & T3_SPV_PDL) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const uint64_t b0 = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    uint2 vnext = make_uint2(0u, 0u);
    // pdl: launched with programmatic serialisation (host decides per launch);
    // the input may still be being written by the previous kernel until the wait
    if ((SPV & T3_SPV_PREFETCH) && !pdl && b0 < nblocks) vnext = __ldcs(in + b0);  // overlaps the fill
    if (!(SPV & T3_SPV_KEYPARAM))
        for (int w = threadIdx.x; w < int(sizeof(T3SpKeyParam) / 4); w += blockDim.x) ks[w] = __ldg(keys_global + w);
    const uint32_t* ks2 = ks + 48 * 8;  // T3SpKeyParam::k2
    for (int w = threadIdx.x; w < 8 * 64; w += blockDim.x) sp[w] = __ldg(sp_global + w);
    __syncthreads();
    // lane replication: each table word fills 32 consecutive words (8 x 16 B)
    uint4* fill = reinterpret_cast<uint4*>(t3_sp_smem);
#pragma unroll 4
    for (int w = threadIdx.x; w < 8 * 64 * 8; w += blockDim.x) {
        const uint32_t v = sp[w >> 3];
        fill[w] = make_uint4(v, v, v, v);
    }
    __syncthreads();
    if ((SPV & T3_SPV_PDL) && pdl) {  // the previous grid on the stream has completed from here on
        asm volatile("griddepcontrol.wait;" ::: "memory");
        if ((SPV & T3_SPV_PREFETCH) && b0 < nblocks) vnext = __ldcs(in + b0);
    }
    const char* smem = reinterpret_cast<const char*>(t3_sp_smem);
    const uint32_t lane4 = (threadIdx.x & 31) * 4;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t b = b0; b < nblocks; b += stride) {
        uint2 v;
        if (SPV & T3_SPV_PREFETCH) {
            v = vnext;
            if (b + stride < nblocks) vnext = __ldcs(in + b + stride);  // read before any write: in place is safe
        } else {
            v = __ldcs(in + b);
        }
        uint32_t x = __byte_perm(v.x, 0, 0x0123);  // big-endian high word
        uint32_t y = __byte_perm(v.y, 0, 0x0123);
        // IP as five delta swaps (verified against the FIPS table in tests).
        t3_dswap(x, y, 4, 0x0F0F0F0Fu);
        t3_dswap(x, y, 16, 0x0000FFFFu);
        t3_dswap(y, x, 2, 0x33333333u);
        t3_dswap(y, x, 8, 0x00FF00FFu);
        t3_dswap(x, y, 1, 0x55555555u);
        if (SPV & T3_SPV_KEYPARAM) {
#pragma unroll
            for (int t = 0; t < 16; t += 2) {
                x = t3_sp_round<SPV>(x, y, T3_SPK(kp, t), smem, lane4, mul);
                y = t3_sp_round<SPV>(y, x, T3_SPK(kp, t + 1), smem, lane4, mul);
            }
            if (passes == 3) {
#pragma unroll
                for (int t = 16; t < 32; t += 2) {
                    y = t3_sp_round<SPV>(y, x, T3_SPK(kp, t), smem, lane4, mul);
                    x = t3_sp_round<SPV>(x, y, T3_SPK(kp, t + 1), smem, lane4, mul);
                }
#pragma unroll
                for (int t = 32; t < 48; t += 2) {
                    x = t3_sp_round<SPV>(x, y, T3_SPK(kp, t), smem, lane4, mul);
                    y = t3_sp_round<SPV>(y, x, T3_SPK(kp, t + 1), smem, lane4, mul);
                }
            }
        } else {
#pragma unroll 1
        for (int t = 0; t < 16; t += 2) {
            x = t3_sp_round<SPV>(x, y, T3_SKS(t), smem, lane4, mul);
            y = t3_sp_round<SPV>(y, x, T3_SKS(t + 1), smem, lane4, mul);
        }
        if (passes == 3) {  // 1 = collapsed EDE (single DES)
#pragma unroll 1
            for (int t = 16; t < 32; t += 2) {  // pass 2: roles swapped
                y = t3_sp_round<SPV>(y, x, T3_SKS(t), smem, lane4, mul);
                x = t3_sp_round<SPV>(x, y, T3_SKS(t + 1), smem, lane4, mul);
            }
#pragma unroll 1
            for (int t = 32; t < 48; t += 2) {
                x = t3_sp_round<SPV>(x, y, T3_SKS(t), smem, lane4, mul);
                y = t3_sp_round<SPV>(y, x, T3_SKS(t + 1), smem, lane4, mul);
            }
        }
        }
        // preoutput = y || x, then FP = the IP swaps in reverse order.
        uint32_t hi = y, lo = x;
        t3_dswap(hi, lo, 1, 0x55555555u);
        t3_dswap(lo, hi, 8, 0x00FF00FFu);
        t3_dswap(lo, hi, 2, 0x33333333u);
        t3_dswap(hi, lo, 16, 0x0000FFFFu);
        t3_dswap(hi, lo, 4, 0x0F0F0F0Fu);
        __stcs(out + b, make_uint2(__byte_perm(hi, 0, 0x0123), __byte_perm(lo, 0, 0x0123)));
    }
}

// ---- helpers -----------------------------------------------------------
__device__ __forceinline__ uint64_t t3_splitmix(uint64_t seed, uint64_t i) {
    uint64_t z = (seed ^ i) + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Block i (global index first_block + i) = splitmix64(seed ^ index),
// serialised big-endian (same as oracle_splitmix_payload).
__global__ void t3_fill_splitmix_kernel(uint2* out, uint64_t first_block, uint64_t n, uint64_t seed) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint64_t v = t3_splitmix(seed, first_block + i);
        out[i] = make_uint2(__byte_perm(uint32_t(v >> 32), 0, 0x0123), __byte_perm(uint32_t(v), 0, 0x0123));
    }
}

// Order-sensitive, shard-additive checksum: sum_i splitmix(word_i ^ gidx_i)
// mod 2^64 where word_i is the little-endian 64-bit load of block i.
__global__ void t3_checksum_kernel(const unsigned long long* in, uint64_t first_block, uint64_t n,
                                   unsigned long long* acc) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    unsigned long long s = 0;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        s += t3_splitmix(in[i] ^ (first_block + i), 0x3DE5C0DEull);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(acc, s);
}
