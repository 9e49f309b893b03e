// Host build of the key-specialised cipher (keyed_kernel.cuh) for the CPU
// parity tests (tests/test_keyed.py): the same t3_keyed_round<K> templates
// NVRTC instantiates at run time, compiled by g++ for one key sequence given
// on the command line (-DT3K_SEQ=..., -DT3K_ROUNDS=48|16).  Reads blocks from
// stdin (a multiple of 32), writes the transformed blocks to stdout.
#include <cstdint>
#include <cstdio>
#include <vector>

constexpr uint64_t T3_KSEQ[] = {T3K_SEQ};
constexpr int T3_KROUNDS = T3K_ROUNDS;
static_assert(sizeof(T3_KSEQ) / sizeof(T3_KSEQ[0]) == T3_KROUNDS, "key sequence length");
#include "keyed_kernel.cuh"

int main() {
    std::vector<uint32_t> w;
    uint32_t buf[64];
    while (std::fread(buf, sizeof buf, 1, stdin) == 1) {
        uint32_t lo[32], hi[32];
        for (int k = 0; k < 32; ++k) {  // block k = (lo[k], hi[k]) as the kernel's 16-byte loads see it
            lo[k] = buf[2 * k];
            hi[k] = buf[2 * k + 1];
        }
        t3_keyed_tile(lo, hi);
        for (int k = 0; k < 32; ++k) {
            buf[2 * k] = lo[k];
            buf[2 * k + 1] = hi[k];
        }
        if (std::fwrite(buf, sizeof buf, 1, stdout) != 1) return 1;
    }
    return 0;
}
