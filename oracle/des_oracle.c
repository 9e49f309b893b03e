/*
 * TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * CPU oracle for the 3DES-ECB hot path: a plain-C restatement of the
 * reference algorithm (/root/reference/proj, "t3des").  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load this library, and only as the checker (or the timed CPU
 * baseline) — never as the product path.
 *
 * Parity pinning: tests/test_oracle.py checks this file against the
 * reference's embedded known-answer vectors (proj/src/verify.cpp:15-40,
 * copied as data into tests/golden/kats.json), against golden batch
 * vectors produced by the reference library itself (oracle/_ref, generator
 * tests/golden/make_golden.py), and — when oracle/_ref is built — against
 * the reference's encrypt_batch/decrypt_batch on random inputs.
 *
 * Bit conventions (reference des.hpp:8-15): a block is a uint64 with FIPS
 * bit 1 in machine bit 63; bytes are big-endian on the wire.
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* FIPS 46-3 tables (data; reference des.cpp:8-75). 1-based, MSB-first. */
static const uint8_t T_IP[64] = {
    58, 50, 42, 34, 26, 18, 10, 2, 60, 52, 44, 36, 28, 20, 12, 4,
    62, 54, 46, 38, 30, 22, 14, 6, 64, 56, 48, 40, 32, 24, 16, 8,
    57, 49, 41, 33, 25, 17, 9, 1, 59, 51, 43, 35, 27, 19, 11, 3,
    61, 53, 45, 37, 29, 21, 13, 5, 63, 55, 47, 39, 31, 23, 15, 7};
static const uint8_t T_FP[64] = {
    40, 8, 48, 16, 56, 24, 64, 32, 39, 7, 47, 15, 55, 23, 63, 31,
    38, 6, 46, 14, 54, 22, 62, 30, 37, 5, 45, 13, 53, 21, 61, 29,
    36, 4, 44, 12, 52, 20, 60, 28, 35, 3, 43, 11, 51, 19, 59, 27,
    34, 2, 42, 10, 50, 18, 58, 26, 33, 1, 41, 9, 49, 17, 57, 25};
static const uint8_t T_E[48] = {
    32, 1, 2, 3, 4, 5, 4, 5, 6, 7, 8, 9, 8, 9, 10, 11,
    12, 13, 12, 13, 14, 15, 16, 17, 16, 17, 18, 19, 20, 21, 20, 21,
    22, 23, 24, 25, 24, 25, 26, 27, 28, 29, 28, 29, 30, 31, 32, 1};
static const uint8_t T_P[32] = {
    16, 7, 20, 21, 29, 12, 28, 17, 1, 15, 23, 26, 5, 18, 31, 10,
    2, 8, 24, 14, 32, 27, 3, 9, 19, 13, 30, 6, 22, 11, 4, 25};
static const uint8_t T_PC1[56] = {
    57, 49, 41, 33, 25, 17, 9, 1, 58, 50, 42, 34, 26, 18,
    10, 2, 59, 51, 43, 35, 27, 19, 11, 3, 60, 52, 44, 36,
    63, 55, 47, 39, 31, 23, 15, 7, 62, 54, 46, 38, 30, 22,
    14, 6, 61, 53, 45, 37, 29, 21, 13, 5, 28, 20, 12, 4};
static const uint8_t T_PC2[48] = {
    14, 17, 11, 24, 1, 5, 3, 28, 15, 6, 21, 10, 23, 19, 12, 4,
    26, 8, 16, 7, 27, 20, 13, 2, 41, 52, 31, 37, 47, 55, 30, 40,
    51, 45, 33, 48, 44, 49, 39, 56, 34, 53, 46, 42, 50, 36, 29, 32};
static const uint8_t T_SHIFTS[16] = {1, 1, 2, 2, 2, 2, 2, 2, 1, 2, 2, 2, 2, 2, 2, 1};
static const uint8_t T_SBOX[8][64] = {
    {14, 4, 13, 1, 2, 15, 11, 8, 3, 10, 6, 12, 5, 9, 0, 7,
     0, 15, 7, 4, 14, 2, 13, 1, 10, 6, 12, 11, 9, 5, 3, 8,
     4, 1, 14, 8, 13, 6, 2, 11, 15, 12, 9, 7, 3, 10, 5, 0,
     15, 12, 8, 2, 4, 9, 1, 7, 5, 11, 3, 14, 10, 0, 6, 13},
    {15, 1, 8, 14, 6, 11, 3, 4, 9, 7, 2, 13, 12, 0, 5, 10,
     3, 13, 4, 7, 15, 2, 8, 14, 12, 0, 1, 10, 6, 9, 11, 5,
     0, 14, 7, 11, 10, 4, 13, 1, 5, 8, 12, 6, 9, 3, 2, 15,
     13, 8, 10, 1, 3, 15, 4, 2, 11, 6, 7, 12, 0, 5, 14, 9},
    {10, 0, 9, 14, 6, 3, 15, 5, 1, 13, 12, 7, 11, 4, 2, 8,
     13, 7, 0, 9, 3, 4, 6, 10, 2, 8, 5, 14, 12, 11, 15, 1,
     13, 6, 4, 9, 8, 15, 3, 0, 11, 1, 2, 12, 5, 10, 14, 7,
     1, 10, 13, 0, 6, 9, 8, 7, 4, 15, 14, 3, 11, 5, 2, 12},
    {7, 13, 14, 3, 0, 6, 9, 10, 1, 2, 8, 5, 11, 12, 4, 15,
     13, 8, 11, 5, 6, 15, 0, 3, 4, 7, 2, 12, 1, 10, 14, 9,
     10, 6, 9, 0, 12, 11, 7, 13, 15, 1, 3, 14, 5, 2, 8, 4,
     3, 15, 0, 6, 10, 1, 13, 8, 9, 4, 5, 11, 12, 7, 2, 14},
    {2, 12, 4, 1, 7, 10, 11, 6, 8, 5, 3, 15, 13, 0, 14, 9,
     14, 11, 2, 12, 4, 7, 13, 1, 5, 0, 15, 10, 3, 9, 8, 6,
     4, 2, 1, 11, 10, 13, 7, 8, 15, 9, 12, 5, 6, 3, 0, 14,
     11, 8, 12, 7, 1, 14, 2, 13, 6, 15, 0, 9, 10, 4, 5, 3},
    {12, 1, 10, 15, 9, 2, 6, 8, 0, 13, 3, 4, 14, 7, 5, 11,
     10, 15, 4, 2, 7, 12, 9, 5, 6, 1, 13, 14, 0, 11, 3, 8,
     9, 14, 15, 5, 2, 8, 12, 3, 7, 0, 4, 10, 1, 13, 11, 6,
     4, 3, 2, 12, 9, 5, 15, 10, 11, 14, 1, 7, 6, 0, 8, 13},
    {4, 11, 2, 14, 15, 0, 8, 13, 3, 12, 9, 7, 5, 10, 6, 1,
     13, 0, 11, 7, 4, 9, 1, 10, 14, 3, 5, 12, 2, 15, 8, 6,
     1, 4, 11, 13, 12, 3, 7, 14, 10, 15, 6, 8, 0, 5, 9, 2,
     6, 11, 13, 8, 1, 4, 10, 7, 9, 5, 0, 15, 14, 2, 3, 12},
    {13, 2, 8, 4, 6, 15, 11, 1, 10, 9, 3, 14, 5, 0, 12, 7,
     1, 15, 13, 8, 10, 3, 7, 4, 12, 5, 6, 11, 0, 14, 9, 2,
     7, 11, 4, 1, 9, 12, 14, 2, 0, 6, 10, 13, 15, 3, 5, 8,
     2, 1, 14, 7, 4, 10, 8, 13, 15, 12, 9, 0, 3, 5, 6, 11}};

/* Generic FIPS permutation (reference des.cpp:77-84): output bit i+1 (from
 * the MSB of the table-length-bit result) is input bit tab[i], counted
 * 1-based from the MSB of a w-bit input. */
static uint64_t fips_permute(uint64_t v, int w, const uint8_t* tab, int n) {
    uint64_t r = 0;
    for (int i = 0; i < n; i++) r = (r << 1) | ((v >> (w - tab[i])) & 1u);
    return r;
}

/* Feistel f on the plain tables (reference des.cpp:86-96). */
static uint32_t feistel_plain(uint32_t half, uint64_t k48) {
    uint64_t x = fips_permute(half, 32, T_E, 48) ^ k48;
    uint32_t s = 0;
    for (int i = 0; i < 8; i++) {
        unsigned six = (unsigned)(x >> (42 - 6 * i)) & 0x3Fu;
        unsigned row = ((six >> 4) & 2u) | (six & 1u);
        unsigned col = (six >> 1) & 0xFu;
        s = (s << 4) | T_SBOX[i][row * 16 + col];
    }
    return (uint32_t)fips_permute(s, 32, T_P, 32);
}

/* One DES block, 16 rounds (reference des.cpp:104-118). */
static uint64_t des_plain(uint64_t blk, const uint64_t ks[16], int inverse) {
    uint64_t p = fips_permute(blk, 64, T_IP, 64);
    uint32_t l = (uint32_t)(p >> 32), r = (uint32_t)p;
    for (int i = 0; i < 16; i++) {
        uint32_t nr = l ^ feistel_plain(r, ks[inverse ? 15 - i : i]);
        l = r;
        r = nr;
    }
    return fips_permute(((uint64_t)r << 32) | l, 64, T_FP, 64);
}

/* Key schedule (reference des.cpp:135-149): PC-1, 16 x (rotl28, PC-2). */
void oracle_key_schedule(uint64_t key, uint64_t ks[16]) {
    uint64_t cd = fips_permute(key, 64, T_PC1, 56);
    uint32_t c = (uint32_t)(cd >> 28), d = (uint32_t)(cd & 0x0FFFFFFFu);
    for (int i = 0; i < 16; i++) {
        int s = T_SHIFTS[i];
        c = ((c << s) | (c >> (28 - s))) & 0x0FFFFFFFu;
        d = ((d << s) | (d >> (28 - s))) & 0x0FFFFFFFu;
        ks[i] = fips_permute(((uint64_t)c << 28) | d, 56, T_PC2, 48);
    }
}

/* triple_schedule (reference tdes.cpp:84-87): pass-major 48 subkeys. */
void oracle_triple_schedule(uint64_t k1, uint64_t k2, uint64_t k3, uint64_t sub48[48]) {
    oracle_key_schedule(k1, sub48);
    oracle_key_schedule(k2, sub48 + 16);
    oracle_key_schedule(k3, sub48 + 32);
}

/* Hex key parse (reference tdes.cpp:32-59).  Returns the keying option
 * (1, 2, 3) or -1 on a length error, -2 on a bad hex character. */
int oracle_parse_hex_key(const char* hex, size_t len, uint64_t out[3]) {
    if (len != 48 && len != 32 && len != 16) return -1;
    uint64_t k[3] = {0, 0, 0};
    for (size_t i = 0; i < len; i++) {
        char ch = hex[i];
        int v = (ch >= '0' && ch <= '9') ? ch - '0'
              : (ch >= 'a' && ch <= 'f') ? ch - 'a' + 10
              : (ch >= 'A' && ch <= 'F') ? ch - 'A' + 10 : -1;
        if (v < 0) return -2;
        k[i / 16] = (k[i / 16] << 4) | (uint64_t)v;
    }
    if (len == 32) k[2] = k[0];
    if (len == 16) k[1] = k[2] = k[0];
    memcpy(out, k, sizeof k);
    return len == 48 ? 1 : (len == 32 ? 2 : 3);
}

uint64_t oracle_des_block(uint64_t blk, uint64_t key, int inverse) {
    uint64_t ks[16];
    oracle_key_schedule(key, ks);
    return des_plain(blk, ks, inverse);
}

/* Reference EDE (tdes.cpp:89-99). */
uint64_t oracle_tdes_block(uint64_t blk, const uint64_t sub48[48], int decrypt) {
    if (!decrypt)
        return des_plain(des_plain(des_plain(blk, sub48, 0), sub48 + 16, 1), sub48 + 32, 0);
    return des_plain(des_plain(des_plain(blk, sub48 + 32, 1), sub48 + 16, 0), sub48, 1);
}

/* ---- fused SP-table route (reference tdes.cpp:101-185) ------------------
 * Same function as the plain route; kept as the faster CPU checker for
 * large batches and for the CPU-baseline port. */
static uint32_t g_sp[8][64];
static int g_sp_ready = 0;

static void sp_init(void) {
    if (g_sp_ready) return;
    for (int i = 0; i < 8; i++)
        for (unsigned x = 0; x < 64; x++) {
            unsigned row = ((x >> 4) & 2u) | (x & 1u), col = (x >> 1) & 0xFu;
            uint32_t placed = (uint32_t)T_SBOX[i][row * 16 + col] << (28 - 4 * i);
            g_sp[i][x] = (uint32_t)fips_permute(placed, 32, T_P, 32);
        }
    g_sp_ready = 1;
}

static inline uint32_t f_sp(uint32_t r, uint64_t k) {
    uint64_t v = ((uint64_t)(r & 1u) << 33) | ((uint64_t)r << 1) | (r >> 31);
    uint32_t o = 0;
    for (int i = 0; i < 8; i++)
        o |= g_sp[i][(unsigned)((v >> (28 - 4 * i)) ^ (k >> (42 - 6 * i))) & 0x3Fu];
    return o;
}

/* seq48: the flattened 48-key execution sequence (a7 in SURVEY §8a). */
static void key_sequence(const uint64_t sub48[48], int decrypt, uint64_t seq[48]) {
    for (int i = 0; i < 16; i++) {
        if (!decrypt) {
            seq[i] = sub48[i];            /* k1 forward */
            seq[16 + i] = sub48[16 + 15 - i]; /* k2 reversed */
            seq[32 + i] = sub48[32 + i];  /* k3 forward */
        } else {
            seq[i] = sub48[32 + 15 - i];  /* k3 reversed */
            seq[16 + i] = sub48[16 + i];  /* k2 forward */
            seq[32 + i] = sub48[15 - i];  /* k1 reversed */
        }
    }
}

static inline uint64_t tdes_sp(uint64_t blk, const uint64_t seq[48]) {
    uint64_t p = fips_permute(blk, 64, T_IP, 64);
    uint32_t l = (uint32_t)(p >> 32), r = (uint32_t)p;
    for (int pass = 0; pass < 3; pass++) {
        for (int i = 0; i < 16; i++) {
            uint32_t nr = l ^ f_sp(r, seq[pass * 16 + i]);
            l = r;
            r = nr;
        }
        uint32_t t = l; l = r; r = t; /* pass-final swap (tdes.cpp:151-159) */
    }
    return fips_permute(((uint64_t)l << 32) | r, 64, T_FP, 64);
}

static inline uint64_t load_be(const uint8_t* p) {
    uint64_t b = 0;
    for (int i = 0; i < 8; i++) b = (b << 8) | p[i];
    return b;
}
static inline void store_be(uint64_t b, uint8_t* p) {
    for (int i = 0; i < 8; i++) p[i] = (uint8_t)(b >> (56 - 8 * i));
}

/* Batch ECB, reference semantics (dispatch.cpp:88-109): returns 0 ok,
 * 1 if len % 8 != 0, 3 if buffers partially overlap.  route 0 = plain
 * tables (ScalarReference), 1 = fused SP tables. threads <= 0: all. */
int oracle_ecb(const uint8_t* in, uint8_t* out, size_t len, const uint64_t sub48[48],
               int decrypt, int route, int threads) {
    if (len % 8) return 1;
    if (out != in && out < in + len && out + len > in) return 3;
    size_t n = len / 8;
    uint64_t seq[48];
    key_sequence(sub48, decrypt, seq);
    sp_init();
#ifdef _OPENMP
    int nt = threads > 0 ? threads : omp_get_max_threads();
#pragma omp parallel for schedule(static, 4096) num_threads(nt)
#endif
    for (long long i = 0; i < (long long)n; i++) {
        uint64_t b = load_be(in + 8 * i);
        uint64_t c = route == 0 ? oracle_tdes_block(b, sub48, decrypt) : tdes_sp(b, seq);
        store_be(c, out + 8 * i);
    }
    (void)threads;
    return 0;
}

/* ---- payload generators ---------------------------------------------------
 * make_payload (reference bench.cpp:41-51): std::mt19937_64(seed), one draw
 * per 8 bytes, emitted little-endian.  MT19937-64 restated from its
 * published definition (the C++ standard's std::mt19937_64 parameters). */
typedef struct { uint64_t mt[312]; int idx; } mt64_t;

static void mt64_seed(mt64_t* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; i++)
        s->mt[i] = 6364136223846793005ull * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->idx = 312;
}

static uint64_t mt64_next(mt64_t* s) {
    const uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull;
    if (s->idx >= 312) {
        for (int i = 0; i < 312; i++) {
            uint64_t x = (s->mt[i] & UM) | (s->mt[(i + 1) % 312] & LM);
            uint64_t xa = x >> 1;
            if (x & 1) xa ^= 0xB5026F5AA96619E9ull;
            s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
        }
        s->idx = 0;
    }
    uint64_t x = s->mt[s->idx++];
    x ^= (x >> 29) & 0x5555555555555555ull;
    x ^= (x << 17) & 0x71D67FFFEDA60000ull;
    x ^= (x << 37) & 0xFFF7EEE000000000ull;
    x ^= x >> 43;
    return x;
}

void oracle_make_payload(uint8_t* out, size_t bytes, uint64_t seed) {
    mt64_t s;
    mt64_seed(&s, seed);
    size_t i = 0;
    for (; i + 8 <= bytes; i += 8) { /* one draw per 8 bytes, little-endian */
        uint64_t w = mt64_next(&s);
        for (int b = 0; b < 8; b++) out[i + b] = (uint8_t)(w >> (8 * b));
    }
    if (i < bytes) {
        uint64_t w = mt64_next(&s);
        for (int b = 0; i < bytes; i++, b++) out[i] = (uint8_t)(w >> (8 * b));
    }
}

/* Index-addressable payload for shards too large for host RAM
 * (SURVEY §8d C4): block i = splitmix64(seed ^ i), serialised big-endian. */
uint64_t oracle_splitmix_block(uint64_t seed, uint64_t i) {
    uint64_t z = (seed ^ i) + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

void oracle_splitmix_payload(uint8_t* out, uint64_t first_block, size_t nblocks, uint64_t seed) {
#ifdef _OPENMP
#pragma omp parallel for schedule(static, 65536)
#endif
    for (long long i = 0; i < (long long)nblocks; i++)
        store_be(oracle_splitmix_block(seed, first_block + (uint64_t)i), out + 8 * i);
}

/* Host restatement of the engine's shard-additive checksum
 * (t3_checksum_kernel): sum_i splitmix(le64(block i) ^ (first_block + i)),
 * salt 0x3DE5C0DE, mod 2^64.  Lets the full-size parity tests and the
 * 64 GiB golden checksum (tests/golden/make_c3_checksum.py) compare whole
 * outputs without holding two copies. */
uint64_t oracle_checksum(const uint8_t* data, uint64_t first_block, size_t nblocks) {
    uint64_t acc = 0;
#ifdef _OPENMP
#pragma omp parallel for schedule(static, 65536) reduction(+ : acc)
#endif
    for (long long i = 0; i < (long long)nblocks; i++) {
        uint64_t w;
        memcpy(&w, data + 8 * i, 8); /* little-endian load, as the kernel's */
        acc += oracle_splitmix_block(0x3DE5C0DEull, w ^ (first_block + (uint64_t)i));
    }
    return acc;
}

/* ---- helpers exposed for tests ------------------------------------------ */
uint64_t oracle_permute(uint64_t v, int w, int which) {
    switch (which) {
        case 0: return fips_permute(v, w, T_IP, 64);
        case 1: return fips_permute(v, w, T_FP, 64);
        case 2: return fips_permute(v, w, T_E, 48);
        case 3: return fips_permute(v, w, T_P, 32);
        default: return 0;
    }
}

int oracle_sbox(int box, int six) {
    unsigned row = ((six >> 4) & 2u) | (six & 1u), col = (six >> 1) & 0xFu;
    return T_SBOX[box][row * 16 + col];
}
