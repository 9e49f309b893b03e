// Host keying for the B200 3DES engine (see schedule.hpp).
#include "schedule.hpp"

#include <cstdlib>
#include <cstring>

#include "generated/bitslice_tables.h"

namespace t3b {
namespace {

// FIPS 46-3 key-schedule and P tables, stored 0-based (source bit index
// counted from the MSB).  Same data as reference des.cpp:31-41.
constexpr std::uint8_t kPC1[56] = {
    56, 48, 40, 32, 24, 16, 8, 0, 57, 49, 41, 33, 25, 17,
    9, 1, 58, 50, 42, 34, 26, 18, 10, 2, 59, 51, 43, 35,
    62, 54, 46, 38, 30, 22, 14, 6, 61, 53, 45, 37, 29, 21,
    13, 5, 60, 52, 44, 36, 28, 20, 12, 4, 27, 19, 11, 3};
constexpr std::uint8_t kPC2[48] = {
    13, 16, 10, 23, 0, 4, 2, 27, 14, 5, 20, 9, 22, 18, 11, 3,
    25, 7, 15, 6, 26, 19, 12, 1, 40, 51, 30, 36, 46, 54, 29, 39,
    50, 44, 32, 47, 43, 48, 38, 55, 33, 52, 45, 41, 49, 35, 28, 31};
constexpr std::uint8_t kRot[16] = {1, 1, 2, 2, 2, 2, 2, 2, 1, 2, 2, 2, 2, 2, 2, 1};
constexpr std::uint8_t kP[32] = {
    15, 6, 19, 20, 28, 11, 27, 16, 0, 14, 22, 25, 4, 17, 30, 9,
    1, 7, 23, 13, 31, 26, 2, 8, 18, 12, 29, 5, 21, 10, 3, 24};
constexpr std::uint8_t kSbox[8][64] = {
    {14, 4, 13, 1, 2, 15, 11, 8, 3, 10, 6, 12, 5, 9, 0, 7, 0, 15, 7, 4, 14, 2, 13, 1, 10, 6, 12, 11, 9, 5, 3, 8,
     4, 1, 14, 8, 13, 6, 2, 11, 15, 12, 9, 7, 3, 10, 5, 0, 15, 12, 8, 2, 4, 9, 1, 7, 5, 11, 3, 14, 10, 0, 6, 13},
    {15, 1, 8, 14, 6, 11, 3, 4, 9, 7, 2, 13, 12, 0, 5, 10, 3, 13, 4, 7, 15, 2, 8, 14, 12, 0, 1, 10, 6, 9, 11, 5,
     0, 14, 7, 11, 10, 4, 13, 1, 5, 8, 12, 6, 9, 3, 2, 15, 13, 8, 10, 1, 3, 15, 4, 2, 11, 6, 7, 12, 0, 5, 14, 9},
    {10, 0, 9, 14, 6, 3, 15, 5, 1, 13, 12, 7, 11, 4, 2, 8, 13, 7, 0, 9, 3, 4, 6, 10, 2, 8, 5, 14, 12, 11, 15, 1,
     13, 6, 4, 9, 8, 15, 3, 0, 11, 1, 2, 12, 5, 10, 14, 7, 1, 10, 13, 0, 6, 9, 8, 7, 4, 15, 14, 3, 11, 5, 2, 12},
    {7, 13, 14, 3, 0, 6, 9, 10, 1, 2, 8, 5, 11, 12, 4, 15, 13, 8, 11, 5, 6, 15, 0, 3, 4, 7, 2, 12, 1, 10, 14, 9,
     10, 6, 9, 0, 12, 11, 7, 13, 15, 1, 3, 14, 5, 2, 8, 4, 3, 15, 0, 6, 10, 1, 13, 8, 9, 4, 5, 11, 12, 7, 2, 14},
    {2, 12, 4, 1, 7, 10, 11, 6, 8, 5, 3, 15, 13, 0, 14, 9, 14, 11, 2, 12, 4, 7, 13, 1, 5, 0, 15, 10, 3, 9, 8, 6,
     4, 2, 1, 11, 10, 13, 7, 8, 15, 9, 12, 5, 6, 3, 0, 14, 11, 8, 12, 7, 1, 14, 2, 13, 6, 15, 0, 9, 10, 4, 5, 3},
    {12, 1, 10, 15, 9, 2, 6, 8, 0, 13, 3, 4, 14, 7, 5, 11, 10, 15, 4, 2, 7, 12, 9, 5, 6, 1, 13, 14, 0, 11, 3, 8,
     9, 14, 15, 5, 2, 8, 12, 3, 7, 0, 4, 10, 1, 13, 11, 6, 4, 3, 2, 12, 9, 5, 15, 10, 11, 14, 1, 7, 6, 0, 8, 13},
    {4, 11, 2, 14, 15, 0, 8, 13, 3, 12, 9, 7, 5, 10, 6, 1, 13, 0, 11, 7, 4, 9, 1, 10, 14, 3, 5, 12, 2, 15, 8, 6,
     1, 4, 11, 13, 12, 3, 7, 14, 10, 15, 6, 8, 0, 5, 9, 2, 6, 11, 13, 8, 1, 4, 10, 7, 9, 5, 0, 15, 14, 2, 3, 12},
    {13, 2, 8, 4, 6, 15, 11, 1, 10, 9, 3, 14, 5, 0, 12, 7, 1, 15, 13, 8, 10, 3, 7, 4, 12, 5, 6, 11, 0, 14, 9, 2,
     7, 11, 4, 1, 9, 12, 14, 2, 0, 6, 10, 13, 15, 3, 5, 8, 2, 1, 14, 7, 4, 10, 8, 13, 15, 12, 9, 0, 3, 5, 6, 11}};

// Gather bits: result bit (n-1-i) = source bit (w-1-src[i]), MSB-first.
std::uint64_t gather_bits(std::uint64_t v, int w, const std::uint8_t* src, int n) {
    std::uint64_t r = 0;
    for (int i = 0; i < n; ++i) r |= ((v >> (w - 1 - src[i])) & 1u) << (n - 1 - i);
    return r;
}

int hexval(char c) {
    if (c >= '0' && c <= '9') return c - '0';
    c = static_cast<char>(c | 0x20);
    if (c >= 'a' && c <= 'f') return c - 'a' + 10;
    return -1;
}

// Bit j (0 = FIPS slot 1) of a 48-bit round key, as a slice mask.
inline std::uint32_t kbit(std::uint64_t k48, int j) {
    return ((k48 >> (47 - j)) & 1u) ? 0xFFFFFFFFu : 0u;
}

}  // namespace

int parse_hex_key(const char* hex, std::size_t len, std::uint64_t keys[3]) {
    if (len != 16 && len != 32 && len != 48) return -1;
    std::uint64_t k[3] = {0, 0, 0};
    for (std::size_t i = 0; i < len; ++i) {
        const int v = hexval(hex[i]);
        if (v < 0) return -2;
        k[i >> 4] = (k[i >> 4] << 4) | static_cast<unsigned>(v);
    }
    keys[0] = k[0];
    keys[1] = len >= 32 ? k[1] : k[0];
    keys[2] = len == 48 ? k[2] : k[0];
    return len == 48 ? 1 : (len == 32 ? 2 : 3);
}

void des_key_schedule(std::uint64_t key, std::uint64_t ks[16]) {
    const std::uint64_t cd = gather_bits(key, 64, kPC1, 56);
    std::uint32_t c = static_cast<std::uint32_t>(cd >> 28);
    std::uint32_t d = static_cast<std::uint32_t>(cd) & 0x0FFFFFFFu;
    for (int r = 0; r < 16; ++r) {
        const int s = kRot[r];
        c = ((c << s) | (c >> (28 - s))) & 0x0FFFFFFFu;
        d = ((d << s) | (d >> (28 - s))) & 0x0FFFFFFFu;
        ks[r] = gather_bits((static_cast<std::uint64_t>(c) << 28) | d, 56, kPC2, 48);
    }
}

void triple_schedule(const std::uint64_t keys[3], std::uint64_t sub48[48]) {
    for (int p = 0; p < 3; ++p) des_key_schedule(keys[p], sub48 + 16 * p);
}

void key_sequence(const std::uint64_t sub48[48], bool decrypt, std::uint64_t seq[48]) {
    std::uint64_t enc[48];
    for (int i = 0; i < 16; ++i) {
        enc[i] = sub48[i];
        enc[16 + i] = sub48[31 - i];
        enc[32 + i] = sub48[32 + i];
    }
    for (int t = 0; t < 48; ++t) seq[t] = decrypt ? enc[47 - t] : enc[t];
}

// Whitening simulation.  Round t (0-based) updates the half in the L role
// and reads the half in the R role.  Pass 1 and 3 start with L = A; pass 2
// starts with L = B (the reference's pass-final swap, tdes.cpp:158).
// A half that is read as R in round t must be stored XORed with the round
// key bit of each bit's primary E slot; this function tracks the stored
// whitening of both halves and emits the constants that keep it so.
void build_bitslice_table(const std::uint64_t seq[48], T3BsTable& tab, int nrounds) {
    std::memset(&tab, 0, sizeof tab);
    auto l_role = [](int t) -> int {  // 0 = A, 1 = B
        const int pass = t / 16, loc = t % 16;
        int a = (loc % 2 == 0) ? 0 : 1;
        return pass == 1 ? 1 - a : a;
    };
    auto prim = [&](int t, int q) { return kbit(seq[t], T3_PRIM_SLOT[q]); };
    // Whitening a half should carry after being written at time t: the
    // primary key bits of the next round reading it, unless it is written
    // again first (then 0).
    auto target_after = [&](int half, int t, std::uint32_t out[32]) {
        for (int t2 = t + 1; t2 < nrounds; ++t2) {
            if (l_role(t2) == half) break;  // overwritten before any read
            for (int q = 0; q < 32; ++q) out[q] = prim(t2, q);
            return;
        }
        for (int q = 0; q < 32; ++q) out[q] = 0;
    };
    std::uint32_t wh[2][32];
    for (int h = 0; h < 2; ++h) {
        target_after(h, -1, wh[h]);
        for (int q = 0; q < 32; ++q) tab.w[T3_TAB_PRE + 32 * h + q] = wh[h][q];
    }
    for (int t = 0; t < nrounds; ++t) {
        const int lh = l_role(t), rh = 1 - lh;
        if (t == 16 || t == 32) {
            // The R half was already read in round t-1 with that round's
            // whitening; re-whiten it for round t (kernel: RW1 on A, RW2 on B).
            const int off = t == 16 ? T3_TAB_RW1 : T3_TAB_RW2;
            for (int q = 0; q < 32; ++q) {
                const std::uint32_t want = prim(t, q);
                tab.w[off + q] = wh[rh][q] ^ want;
                wh[rh][q] = want;
            }
        }
        std::uint32_t* rk = tab.w + T3_TAB_ROUND + T3_ROUND_WORDS * t;
        for (int d = 0; d < 16; ++d) {
            const int j = T3_SECONDARY_SLOT[d];
            const int q = T3_E[j] - 1;
            rk[32 + d] = kbit(seq[t], j) ^ wh[rh][q];
            rk[48 + d] = rk[32 + d] | 1u;  // multiplier of the FMA form
        }
        std::uint32_t nxt[32];
        target_after(lh, t, nxt);
        for (int q = 0; q < 32; ++q) {
            rk[q] = wh[lh][q] ^ nxt[q];
            wh[lh][q] = nxt[q];
        }
    }
    for (int h = 0; h < 2; ++h)
        for (int q = 0; q < 32; ++q) tab.w[T3_TAB_POST + 32 * h + q] = wh[h][q];
    // The kernel skips the XORs that are zero by construction: half A's
    // initial whitening (A is written before it is read) and half B's final
    // one (B is not read after the last round).
    for (int q = 0; q < 32; ++q)
        if (tab.w[T3_TAB_PRE + q] != 0 || tab.w[T3_TAB_POST + 32 + q] != 0) std::abort();
    // multipliers of the FMA form of the whitening XORs (S = D | 1)
    for (int i = 0; i < 64; ++i) tab.w[T3_TAB_WS + i] = tab.w[T3_TAB_PRE + i] | 1u;
    for (int i = 0; i < 32; ++i) tab.w[T3_TAB_WS + 64 + i] = tab.w[T3_TAB_RW1 + i] | 1u;
    for (int i = 0; i < 32; ++i) tab.w[T3_TAB_WS + 96 + i] = tab.w[T3_TAB_RW2 + i] | 1u;
    for (int i = 0; i < 64; ++i) tab.w[T3_TAB_WS + 128 + i] = tab.w[T3_TAB_POST + i] | 1u;
    tab.w[T3_TAB_FK] = 2u;  // t3_cfix's opaque constants
    tab.w[T3_TAB_FK + 1] = 1u;
}

int collapsed_sequence(const std::uint64_t sub48[48], bool decrypt, std::uint64_t seq16[16]) {
    const std::uint64_t* p1 = sub48;
    const std::uint64_t* p2 = sub48 + 16;
    const std::uint64_t* p3 = sub48 + 32;
    const std::uint64_t* single = nullptr;
    if (std::memcmp(p1, p2, 16 * 8) == 0) single = p3;       // E_k3(D_k2(E_k1 x)) = E_k3 x
    else if (std::memcmp(p2, p3, 16 * 8) == 0) single = p1;  // = E_k1 x
    if (!single) return 48;
    for (int t = 0; t < 16; ++t) seq16[t] = decrypt ? single[15 - t] : single[t];
    return 16;
}

void build_sp_keys(const std::uint64_t seq[48], SpKeys& out) {
    for (int t = 0; t < 48; ++t) {
        out.k2[t][0] = out.k2[t][1] = 0;
        for (int i = 0; i < 8; ++i) {
            const std::uint32_t kc = static_cast<std::uint32_t>((seq[t] >> (42 - 6 * i)) & 0x3F) << 7;
            out.k[t][i] = kc;
            // the kernel reads window i as rotr(R, s) bits 7..12, s = (20 - 4i) mod 32
            const int s = (20 - 4 * i) & 31;
            out.k2[t][i & 1] |= s ? (kc << s) | (kc >> (32 - s)) : kc;
        }
    }
}

void build_sp_tables(std::uint32_t sp[8][64]) {
    for (int i = 0; i < 8; ++i)
        for (int x = 0; x < 64; ++x) {
            const int row = ((x >> 4) & 2) | (x & 1), col = (x >> 1) & 0xF;
            const std::uint32_t placed = static_cast<std::uint32_t>(kSbox[i][row * 16 + col])
                                         << (28 - 4 * i);
            sp[i][x] = static_cast<std::uint32_t>(gather_bits(placed, 32, kP, 32));
        }
}

// ---- key hygiene ----------------------------------------------------------
// Parity: FIPS 46-3 DES keys carry odd parity in the LSB of each byte.
bool has_odd_parity(std::uint64_t key) {
    for (int i = 0; i < 8; ++i)
        if (!__builtin_parity(static_cast<unsigned>((key >> (8 * i)) & 0xFFu))) return false;
    return true;
}

std::uint64_t normalize_parity(std::uint64_t key) {
    for (int i = 0; i < 8; ++i)
        if (!__builtin_parity(static_cast<unsigned>((key >> (8 * i)) & 0xFFu))) key ^= std::uint64_t(1) << (8 * i);
    return key;
}

// Weak and semi-weak keys, characterised by what makes them weak instead of
// listed: after PC-1 (which drops the parity bits) each 28-bit register C, D
// is invariant under the schedule's rotations (all zeros or all ones: the 16
// subkeys are identical, the 4 weak keys) or 2-periodic (0101... / 1010...:
// the subkeys alternate between two values).  The 4 x 4 combinations minus
// the 4 weak ones are the 12 semi-weak keys of the reference's table
// (des.cpp:180-191); tests/test_capi_host.py checks the two agree.
namespace {
int register_class(std::uint32_t r) {  // 0: constant, 1: 2-periodic, -1: other
    if (r == 0 || r == 0x0FFFFFFFu) return 0;
    if (r == 0x05555555u || r == 0x0AAAAAAAu) return 1;
    return -1;
}
}  // namespace

bool is_weak_key(std::uint64_t key) {
    const std::uint64_t cd = gather_bits(key, 64, kPC1, 56);
    return register_class(static_cast<std::uint32_t>(cd >> 28)) == 0 &&
           register_class(static_cast<std::uint32_t>(cd) & 0x0FFFFFFFu) == 0;
}

bool is_semiweak_key(std::uint64_t key) {
    const std::uint64_t cd = gather_bits(key, 64, kPC1, 56);
    const int c = register_class(static_cast<std::uint32_t>(cd >> 28));
    const int d = register_class(static_cast<std::uint32_t>(cd) & 0x0FFFFFFFu);
    return c >= 0 && d >= 0 && (c | d) == 1;
}

}  // namespace t3b
