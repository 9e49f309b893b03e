// TEST INFRASTRUCTURE — host build of the bitsliced core (t3des_core.cuh)
// so the CPU test suite can check the generated round code, the slice
// transposes and the whitening tables against the oracle without a GPU.
// The product never runs this; it is the same source compiled for x86.
#include <cstdint>
#include <cstring>

#include "schedule.hpp"

extern "C" int bs_host_ecb(const std::uint8_t* in, std::uint8_t* out, std::size_t nblocks,
                           const std::uint64_t sub48[48], int decrypt) {
    if (nblocks % 32) return 1;
    std::uint64_t seq[48];
    t3b::key_sequence(sub48, decrypt != 0, seq);
    static T3BsTable tab;
    t3b::build_bitslice_table(seq, tab);
    for (std::size_t base = 0; base < nblocks; base += 32) {
        std::uint32_t lo[32], hi[32];
        for (int m = 0; m < 32; ++m) {
            std::memcpy(&lo[m], in + 8 * (base + m), 4);
            std::memcpy(&hi[m], in + 8 * (base + m) + 4, 4);
        }
        t3_tile32<0>(lo, hi, static_cast<const std::uint32_t*>(tab.w));
        for (int m = 0; m < 32; ++m) {
            std::memcpy(out + 8 * (base + m), &lo[m], 4);
            std::memcpy(out + 8 * (base + m) + 4, &hi[m], 4);
        }
    }
    return 0;
}

// Same, through the collapsed (single-DES) path when the schedule allows it
// (K1 = K2 or K2 = K3); returns the round count used.
extern "C" int bs_host_ecb_collapse(const std::uint8_t* in, std::uint8_t* out, std::size_t nblocks,
                                    const std::uint64_t sub48[48], int decrypt) {
    if (nblocks % 32) return -1;
    std::uint64_t seq[48] = {};
    const int rounds = t3b::collapsed_sequence(sub48, decrypt != 0, seq);
    if (rounds != 16) return bs_host_ecb(in, out, nblocks, sub48, decrypt) == 0 ? 48 : -1;
    static T3BsTable tab;
    t3b::build_bitslice_table(seq, tab, 16);
    for (std::size_t base = 0; base < nblocks; base += 32) {
        std::uint32_t lo[32], hi[32];
        for (int m = 0; m < 32; ++m) {
            std::memcpy(&lo[m], in + 8 * (base + m), 4);
            std::memcpy(&hi[m], in + 8 * (base + m) + 4, 4);
        }
        t3_tile32<0, 16>(lo, hi, static_cast<const std::uint32_t*>(tab.w));
        for (int m = 0; m < 32; ++m) {
            std::memcpy(out + 8 * (base + m), &lo[m], 4);
            std::memcpy(out + 8 * (base + m) + 4, &hi[m], 4);
        }
    }
    return 16;
}

extern "C" int bs_host_table(const std::uint64_t sub48[48], int decrypt, std::uint32_t* words) {
    std::uint64_t seq[48];
    t3b::key_sequence(sub48, decrypt != 0, seq);
    static T3BsTable tab;
    t3b::build_bitslice_table(seq, tab);
    std::memcpy(words, tab.w, sizeof tab.w);
    return T3_TAB_WORDS;
}
