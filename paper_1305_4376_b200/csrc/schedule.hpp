// Host-side keying for the B200 3DES engine: hex-key parsing, the DES key
// schedule, the 48-key execution sequence and its expansion into the
// constant tables the kernels read.  Pure host C++ (no CUDA calls).
//
// Reference interfaces restated (semantics, not code):
//   parse_hex_key   /root/reference/proj/src/tdes.cpp:32-59
//   key_schedule    /root/reference/proj/src/des.cpp:135-149
//   triple_schedule /root/reference/proj/src/tdes.cpp:84-87 (pass-major)
//   key order of tdes_{en,de}crypt_block_fast, tdes.cpp:177-185
#pragma once
#include <cstddef>
#include <cstdint>

#include "t3des_core.cuh"

namespace t3b {

// Returns 1/2/3 (keying option) or a negative value: -1 bad length,
// -2 bad hex character.  Keys are written k1, k2, k3 (k3=k1 for Option 2,
// all equal for Option 3).
int parse_hex_key(const char* hex, std::size_t len, std::uint64_t keys[3]);

// 16 round keys of 48 bits (FIPS bit 1 of the subkey at machine bit 47).
void des_key_schedule(std::uint64_t key, std::uint64_t ks[16]);

// 48 subkeys, pass-major: k1's 16, then k2's, then k3's.
void triple_schedule(const std::uint64_t keys[3], std::uint64_t sub48[48]);

// The 48 round keys in execution order: encrypt = k1 fwd, k2 rev, k3 fwd;
// decrypt = the exact reverse sequence.
void key_sequence(const std::uint64_t sub48[48], bool decrypt, std::uint64_t seq[48]);

// Whitening/key-constant table of the bitsliced kernel for one execution
// sequence of nrounds (48, or 16 for a collapsed schedule) round keys
// (layout: T3_TAB_* in t3des_core.cuh).
void build_bitslice_table(const std::uint64_t seq[48], T3BsTable& tab, int nrounds = 48);

// EDE collapse: if k1 and k2 (or k2 and k3) have identical schedules, the
// inner E/D pair is the identity and 3DES equals single DES under the
// remaining key.  Writes that 16-key sequence and returns 16, else 48.
int collapsed_sequence(const std::uint64_t sub48[48], bool decrypt, std::uint64_t seq16[16]);

// Per-round 6-bit key chunks for the SP-table kernel: k6[r][i] is the key
// input of S-box i in round r, shifted to bits 7..12 (pre-scaled as a byte
// offset of a 128-byte row).
// k2[r] = {Ka, Kb}: the same chunks placed at the R-word bit positions their
// S-box windows read (windows 0,2,4,6 are disjoint, as are 1,3,5,7), so one
// XOR of R with Ka (Kb) keys four windows at once.
struct SpKeys {
    std::uint32_t k[48][8];
    std::uint32_t k2[48][2];
};
void build_sp_keys(const std::uint64_t seq[48], SpKeys& out);

// The eight S-box/P fused tables (2 KiB): sp[i][six] = P(S_i(six) placed).
void build_sp_tables(std::uint32_t sp[8][64]);

// Key hygiene (reference des.cpp:159-207, semantics restated): every byte
// of odd parity; the LSB of even-parity bytes flipped; membership in the 4
// weak / 12 semi-weak keys with the parity bits masked off.
bool has_odd_parity(std::uint64_t key);
std::uint64_t normalize_parity(std::uint64_t key);
bool is_weak_key(std::uint64_t key);
bool is_semiweak_key(std::uint64_t key);

}  // namespace t3b
