// Bitsliced 3DES core for sm_100a: 32x32 slice transposes, the 48-round
// cipher over 64 slice words, and the whitening-table layout.
//
// Portable between device code and a host test build (tests/native): the
// only device-specific pieces are lop3 and prmt, which fall back to plain C
// when __CUDA_ARCH__ is not defined.  The host build exists so the test
// suite can check the generated round code on a CPU; the product path is
// the CUDA kernel in bitslice_kernel.cuh and never runs this on the host.
//
// Reference path replaced: fused_tdes / run_pass / round_f
// (/root/reference/proj/src/tdes.cpp:132-173) and the per-block loop
// run_blocks_fast (dispatch.cpp:47-56).
#pragma once
#include <stdint.h>

#define T3_TILE_BLOCKS 1024  // blocks per warp tile (32 lanes x 32 blocks)

#ifdef __CUDACC__
#define T3_FI __host__ __device__ __forceinline__
#else
#define T3_FI inline
#endif

template <unsigned LUT>
T3_FI uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
#ifdef __CUDA_ARCH__
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(LUT));
    return d;
#else
    uint32_t r = 0;
#pragma unroll
    for (int m = 0; m < 8; ++m)
        if ((LUT >> m) & 1u)
            r |= ((m & 4) ? a : ~a) & ((m & 2) ? b : ~b) & ((m & 1) ? c : ~c);
    return r;
#endif
}

template <unsigned SEL>
T3_FI uint32_t prmt(uint32_t a, uint32_t b) {
#ifdef __CUDA_ARCH__
    return __byte_perm(a, b, SEL);
#else
    const uint64_t v = ((uint64_t)b << 32) | a;
    uint32_t r = 0;
    for (int i = 0; i < 4; ++i) r |= (uint32_t)((v >> (8 * ((SEL >> (4 * i)) & 7))) & 0xFF) << (8 * i);
    return r;
#endif
}

// Code-generation options of the bitsliced core (template bitmask OPT).
enum : int {
    T3_OPT_DFMA = 1,    // E-duplicate key corrections as IMAD (FMA pipe)
    T3_OPT_SHRFMA = 2,  // transpose right shifts as IMAD.HI (FMA pipe)
    T3_OPT_WFMA = 4,    // pre/re/post whitening XORs as IMAD (FMA pipe)
};

// x ^ d for a key-correction word d in {0, ~0}.  OPT & DFMA computes it as
// x * s + d with s = d | 1 (= +1 or -1): an IMAD on the FMA pipe, which is
// otherwise idle, instead of a LOP3 on the saturated ALU pipe.
template <int OPT>
T3_FI uint32_t t3_dfix(uint32_t x, uint32_t d, uint32_t s) {
#ifdef __CUDA_ARCH__
    if (OPT & T3_OPT_DFMA) {
        uint32_t r;
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(s), "r"(d));
        return r;
    }
#endif
    (void)s;
    return x ^ d;
}

// x ^ c for a warp-uniform word c in {0, ~0}, entirely on the FMA pipe and
// with c as the only per-round operand (a uniform register, no LDC):
//   x ^ c = c * (2x + 1) + x      (c = 0: x;  c = -1: -x - 1 = ~x)
// Both IMADs take the opaque registers two/one (read from the table) so
// ptxas cannot strength-reduce 2x + 1 into an ALU LEA.  Used where an
// S-box output's last gate is merged into the Feistel lop3 (gen_bitslice.py
// "Feistel tops"), which leaves no lop3 input free for the C word.
struct T3Fk {
    uint32_t two, one;
};
T3_FI uint32_t t3_cfix(uint32_t x, uint32_t c, T3Fk fk) {
#ifdef __CUDA_ARCH__
    uint32_t t, r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(t) : "r"(x), "r"(fk.two), "r"(fk.one));
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(t), "r"(c), "r"(x));
    return r;
#else
    (void)fk;
    return x ^ c;
#endif
}

// a >> S; OPT & SHRFMA uses IMAD.HI (a * 2^(32-S) >> 32) on the FMA pipe.
template <int S, int OPT>
T3_FI uint32_t t3_shr(uint32_t a) {
#ifdef __CUDA_ARCH__
    if (OPT & T3_OPT_SHRFMA) {
        uint32_t r;
        asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(1u << (32 - S)));
        return r;
    }
#endif
    return a >> S;
}

#include "generated/bitslice_rounds.cuh"

// ---- whitening/key table (built on the host, schedule.cpp) --------------
// Word offsets inside the 3458-word table that travels as the kernel's
// __grid_constant__ parameter (constant bank 0, read through LDCU).
enum : int {
    T3_TAB_PRE = 0,            // 64: initial whitening, half A then half B
    T3_TAB_ROUND = 64,         // 48 rounds x 64 words (32 C + 16 D + 16 S)
    T3_ROUND_WORDS = 64,
    T3_TAB_RW1 = 64 + 48 * T3_ROUND_WORDS, // 32: re-whitening of A between pass 1 and 2
    T3_TAB_RW2 = T3_TAB_RW1 + 32,  // 32: re-whitening of B between pass 2 and 3
    T3_TAB_POST = T3_TAB_RW2 + 32, // 64: final un-whitening, A then B
    T3_TAB_WS = T3_TAB_POST + 64,  // 192: S = D | 1 for PRE(64), RW1(32), RW2(32), POST(64)
    T3_TAB_FK = T3_TAB_WS + 192,   // 2: the opaque constants 2, 1 of t3_cfix
    T3_TAB_WORDS = T3_TAB_FK + 2,
};

struct T3BsTable {
    uint32_t w[T3_TAB_WORDS];
};

// Per-round 6-bit key chunks of the SP-table kernel (pre-shifted, see
// t3b::build_sp_keys).
struct T3SpKeyParam {
    uint32_t k[48][8];
    uint32_t k2[48][2];  // t3b::SpKeys::k2
};

#ifndef T3_SPV_DEFAULT
#define T3_SPV_DEFAULT 490  // T3_SPV_* mask of the SP-table kernel (kernels.cuh): KEY2|KEYPARAM|SHLFMA|MERGE6|PREFETCH|PDL
#endif

// In-register transpose of a 32x32 bit matrix: afterwards x[k] bit m is the
// old x[m] bit k.  Stages 16 and 8 are byte moves (PRMT); stages 4, 2, 1
// are mask-select swaps (two shifts + two lop3 per pair).
template <int OPT>
T3_FI void t3_transpose32(uint32_t (&x)[32]) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        const uint32_t a = x[r], b = x[r + 16];
        x[r] = prmt<0x5410>(a, b);
        x[r + 16] = prmt<0x7632>(a, b);
    }
#pragma unroll
    for (int r = 0; r < 32; ++r) {
        if (r & 8) continue;
        const uint32_t a = x[r], b = x[r + 8];
        x[r] = prmt<0x6240>(a, b);
        x[r + 8] = prmt<0x7351>(a, b);
    }
#pragma unroll
    for (int r = 0; r < 32; ++r) {
        if (r & 4) continue;
        const uint32_t a = x[r], b = x[r + 4];
        x[r] = lop3<0xE4>(a, b << 4, 0x0F0F0F0Fu);  // 0xE4: c ? a : b
        x[r + 4] = lop3<0xE4>(t3_shr<4, OPT>(a), b, 0x0F0F0F0Fu);
    }
#pragma unroll
    for (int r = 0; r < 32; ++r) {
        if (r & 2) continue;
        const uint32_t a = x[r], b = x[r + 2];
        x[r] = lop3<0xE4>(a, b << 2, 0x33333333u);
        x[r + 2] = lop3<0xE4>(t3_shr<2, OPT>(a), b, 0x33333333u);
    }
#pragma unroll
    for (int r = 0; r < 32; r += 2) {
        const uint32_t a = x[r], b = x[r + 1];
        x[r] = lop3<0xE4>(a, b << 1, 0x55555555u);
        x[r + 1] = lop3<0xE4>(t3_shr<1, OPT>(a), b, 0x55555555u);
    }
}

// h ^= table words k (0/~0); with WFMA as IMAD h*s+k, s = the matching S words.
template <int OPT, class KP>
T3_FI void t3_xor_table(uint32_t (&h)[32], const KP k, const KP s) {
#pragma unroll
    for (int q = 0; q < 32; ++q) h[q] = (OPT & T3_OPT_WFMA) ? t3_dfix<T3_OPT_DFMA>(h[q], k[q], s[q]) : (h[q] ^ k[q]);
}

#ifndef T3_BODY_ROUNDS
#define T3_BODY_ROUNDS 2  // rounds per loop iteration (2 or 4)
#endif

// All 48 rounds (3 passes of 16) on halves A (initial L) and B (initial R).
// The pass-final half swaps of the reference (tdes.cpp:151-159) are role
// renamings: pass 2 runs with the roles of A and B exchanged.
template <int OPT, int ROUNDS = 48, class KP>
T3_FI void t3_cipher(uint32_t (&A)[32], uint32_t (&B)[32], const KP w) {
    // A is written (round 1) before it is ever read, so its initial whitening
    // is 0 by construction (checked in build_bitslice_table); only B needs it.
    const T3Fk fk{w[T3_TAB_FK], w[T3_TAB_FK + 1]};
    t3_xor_table<OPT>(B, w + T3_TAB_PRE + 32, w + T3_TAB_WS + 32);
    if (ROUNDS == 16) {  // collapsed EDE (single DES): one pass, [A<-B, B<-A] x 8
#pragma unroll 1
        for (int r = 0; r < 16; r += 2) {
            t3_round<OPT>(A, B, fk, w + T3_TAB_ROUND + r * T3_ROUND_WORDS);
            t3_round<OPT>(B, A, fk, w + T3_TAB_ROUND + (r + 1) * T3_ROUND_WORDS);
        }
        t3_xor_table<OPT>(A, w + T3_TAB_POST, w + T3_TAB_WS + 128);
        return;
    }
    // Rounds as one shared 2-round body: pass 1 = [A<-B, B<-A] x 8; pass 2
    // (roles swapped) = B<-A, [A<-B, B<-A] x 7, A<-B; pass 3 = [A<-B, B<-A] x 8.
    // One loop of 23 bodies with the two single rounds (and the
    // re-whitenings) behind uniform branches keeps 4 rounds of code instead
    // of 6 (instruction-cache footprint).
#if T3_BODY_ROUNDS == 4
    // 4-round body: [AB AB]x4, B, [AB AB]x3, [AB], A, [AB AB]x4
    auto body2 = [&](int r) {
        t3_round<OPT>(A, B, fk, w + T3_TAB_ROUND + r * T3_ROUND_WORDS);
        t3_round<OPT>(B, A, fk, w + T3_TAB_ROUND + (r + 1) * T3_ROUND_WORDS);
    };
    int r = 0;
#pragma unroll 1
    for (int it = 0; it < 11; ++it) {
        body2(r);
        body2(r + 2);
        r += 4;
        if (it == 3) {  // after round 15
            t3_xor_table<OPT>(A, w + T3_TAB_RW1, w + T3_TAB_WS + 64);
            t3_round<OPT>(B, A, fk, w + T3_TAB_ROUND + 16 * T3_ROUND_WORDS);
            r = 17;
        } else if (it == 6) {  // rounds 17..28 done: 29, 30, then 31 = A <- B
            body2(29);
            t3_round<OPT>(A, B, fk, w + T3_TAB_ROUND + 31 * T3_ROUND_WORDS);
            t3_xor_table<OPT>(B, w + T3_TAB_RW2, w + T3_TAB_WS + 96);
            r = 32;
        }
    }
#else
    int r = 0;
#pragma unroll 1
    for (int it = 0; it < 23; ++it) {
        t3_round<OPT>(A, B, fk, w + T3_TAB_ROUND + r * T3_ROUND_WORDS);
        t3_round<OPT>(B, A, fk, w + T3_TAB_ROUND + (r + 1) * T3_ROUND_WORDS);
        r += 2;
        if (it == 7) {  // after round 15: pass 2 starts with B <- A
            t3_xor_table<OPT>(A, w + T3_TAB_RW1, w + T3_TAB_WS + 64);
            t3_round<OPT>(B, A, fk, w + T3_TAB_ROUND + 16 * T3_ROUND_WORDS);
            r = 17;
        } else if (it == 14) {  // after round 30: pass 2 ends with A <- B
            t3_round<OPT>(A, B, fk, w + T3_TAB_ROUND + 31 * T3_ROUND_WORDS);
            t3_xor_table<OPT>(B, w + T3_TAB_RW2, w + T3_TAB_WS + 96);
            r = 32;
        }
    }
#endif
    // B is never read after round 48, so its final whitening is 0 (checked
    // on the host); only A is un-whitened.
    t3_xor_table<OPT>(A, w + T3_TAB_POST, w + T3_TAB_WS + 128);
}

// One thread's 32 blocks: lo[m]/hi[m] are the little-endian words holding
// bytes 0..3 / 4..7 of block m.  Transforms in place.
template <int OPT, int ROUNDS = 48, class KP>
T3_FI void t3_tile32(uint32_t (&lo)[32], uint32_t (&hi)[32], const KP w) {
    t3_transpose32<OPT>(lo);
    t3_transpose32<OPT>(hi);
    uint32_t A[32] = T3_GATHER_A(lo, hi);
    uint32_t B[32] = T3_GATHER_B(lo, hi);
    t3_cipher<OPT, ROUNDS>(A, B, w);
    {
        uint32_t olo[32] = T3_SCATTER_LO(A, B);
        uint32_t ohi[32] = T3_SCATTER_HI(A, B);
#pragma unroll
        for (int k = 0; k < 32; ++k) {
            lo[k] = olo[k];
            hi[k] = ohi[k];
        }
    }
    t3_transpose32<OPT>(lo);
    t3_transpose32<OPT>(hi);
}

