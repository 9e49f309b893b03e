// Single-block transforms, known-answer vectors and the self-check of the
// C++ host API (include/t3des_b200/t3des.hpp), the B200 counterparts of
// the reference's des.hpp:37-39, tdes.hpp:44-54 and verify.hpp:14-37.
//
// There is no CPU cipher here: a "single block" is a one-block batch
// through the engine (encrypt_batch), and single DES is the EDE of one
// schedule repeated three times, which the engine runs as the collapsed
// 16-round kernel.  run_verification checks the same groups as the
// reference's (verify.cpp:65-124) — the walkthrough schedule, DES and 3DES
// vectors, DES round trips and complementation, the EDE collapse — and
// adds the NIST SP 800-67 three-block example as one batch.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <ostream>
#include <random>
#include <sstream>

#include "t3des_b200/t3des.hpp"
#include "t3des_cu.h"

namespace t3des {
namespace {

constexpr std::uint64_t hex_const(std::string_view h) {
    std::uint64_t v = 0;
    for (char c : h) v = v * 16 + static_cast<std::uint64_t>(c <= '9' ? c - '0' : (c | 0x20) - 'a' + 10);
    return v;
}

// Published vectors — the FIPS 46 walkthrough key, NIST SP 500-20 style DES
// vectors, NIST SP 800-67 App. B and the keying-option cases — as the
// reference embeds them (verify.cpp:15-40), so both `verify` commands check
// the same answers.  DES rows: key, plaintext, ciphertext.
constexpr std::string_view kDesRows[] = {
    "133457799BBCDFF1 0123456789ABCDEF 85E813540F0AB405", "0E329232EA6D0D73 8787878787878787 0000000000000000",
    "0101010101010101 0000000000000000 8CA64DE9C1B123A7", "8001010101010101 0000000000000000 95A8D72813DAA94D",
    "7CA110454A1A6E57 01A1D6D039776742 690F5B0D9A26939B", "0131D9619DC1376E 5CD54CA83DEF57DA 7A389D10354BD271",
};

constexpr DesKat des_row(std::string_view r) {
    return DesKat{hex_const(r.substr(0, 16)), hex_const(r.substr(17, 16)), hex_const(r.substr(34, 16))};
}

constexpr DesKat kDes[] = {des_row(kDesRows[0]), des_row(kDesRows[1]), des_row(kDesRows[2]),
                           des_row(kDesRows[3]), des_row(kDesRows[4]), des_row(kDesRows[5])};

constexpr TdesKat kTdes[] = {
    {"0123456789ABCDEF23456789ABCDEF01456789ABCDEF0123", "5468652071756663", "A826FD8CE53B855F"},  // SP 800-67
    {"133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57", "0123456789ABCDEF", "1A493D768C1B9432"},  // option 1
    {"0123456789ABCDEF23456789ABCDEF01", "4E6F772069732074", "B7835779EE26ACB7"},                  // option 2
    {"0123456789ABCDEF", "4E6F772069732074", "3FA40E8A984D4815"},                                  // option 3
};

// the 16 subkeys of key 133457799BBCDFF1, 12 hex digits each
constexpr std::string_view kWalkHex =
    "1B02EFFC7072" "79AED9DBC9E5" "55FC8A42CF99" "72ADD6DB351D" "7CEC07EB53A8" "63A53E507B2F" "EC84B7F618BC"
    "F78A3AC13BFB" "E0DBEBEDE781" "B1F347BA464F" "215FD3DED386" "7571F59467E9" "97C5D1FABA41" "5F43B7F2E73A"
    "BF918D3D3F0A" "CB3D8B0E17F5";

struct WalkTable {
    std::uint64_t k[16];
    constexpr WalkTable() : k{} {
        for (int i = 0; i < 16; ++i) k[i] = hex_const(kWalkHex.substr(12 * i, 12));
    }
};
constexpr WalkTable kWalkTable;
constexpr const std::uint64_t (&kWalk)[16] = kWalkTable.k;

std::uint64_t hex64(std::string_view h) {
    std::uint64_t v = 0;
    for (char c : h) v = (v << 4) | static_cast<unsigned>(c <= '9' ? c - '0' : (c | 0x20) - 'a' + 10);
    return v;
}

std::vector<std::uint8_t> unhex(std::string_view h) {
    std::vector<std::uint8_t> b(h.size() / 2);
    for (std::size_t i = 0; i < b.size(); ++i) b[i] = static_cast<std::uint8_t>(hex64(h.substr(2 * i, 2)));
    return b;
}

Block one_block(Block b, const TripleSchedule& ts, bool decrypt, const DispatchConfig& cfg) {
    std::uint8_t buf[8];
    store_block(b, std::span<std::uint8_t, 8>(buf));
    const std::span<std::uint8_t> io(buf, 8);
    if (decrypt)
        decrypt_batch(io, io, ts, cfg);
    else
        encrypt_batch(io, io, ts, cfg);
    return load_block(std::span<const std::uint8_t, 8>(buf));
}

TripleSchedule single(const RoundKeySet& ks) { return TripleSchedule{ks, ks, ks}; }

bool check(std::ostream& out, const char* name, bool pass) {
    out << (pass ? "ok   " : "FAIL ") << name << '\n';
    return pass;
}

}  // namespace

Block encrypt_block(Block block, const RoundKeySet& ks) { return one_block(block, single(ks), false, {}); }
Block decrypt_block(Block block, const RoundKeySet& ks) { return one_block(block, single(ks), true, {}); }
Block tdes_encrypt_block(Block block, const TripleSchedule& ts) { return one_block(block, ts, false, {}); }
Block tdes_decrypt_block(Block block, const TripleSchedule& ts) { return one_block(block, ts, true, {}); }
Block tdes_encrypt_block_fast(Block block, const TripleSchedule& ts) { return one_block(block, ts, false, {}); }
Block tdes_decrypt_block_fast(Block block, const TripleSchedule& ts) { return one_block(block, ts, true, {}); }

std::span<const DesKat> des_kats() { return kDes; }
std::span<const TdesKat> tdes_kats() { return kTdes; }
std::span<const std::uint64_t> walkthrough_subkeys() { return kWalk; }

bool run_verification(std::ostream& out) { return run_verification(out, DispatchConfig{}); }

bool run_verification(std::ostream& out, const DispatchConfig& cfg) {
    bool all = true;

    const RoundKeySet walk = key_schedule(DesKey{kWalkthroughKey});
    all &= check(out, "key schedule walkthrough", std::equal(walk.begin(), walk.end(), kWalk));

    bool pass = true;
    for (const DesKat& k : kDes) {
        const TripleSchedule ts = single(key_schedule(DesKey{k.key}));
        pass &= one_block(k.plaintext, ts, false, cfg) == k.ciphertext;
        pass &= one_block(k.ciphertext, ts, true, cfg) == k.plaintext;
    }
    all &= check(out, "DES known-answer vectors", pass);

    pass = true;
    for (const TdesKat& k : kTdes) {
        const TripleSchedule ts = triple_schedule(parse_hex_key(k.key_hex));
        pass &= one_block(hex64(k.plaintext_hex), ts, false, cfg) == hex64(k.ciphertext_hex);
        pass &= one_block(hex64(k.ciphertext_hex), ts, true, cfg) == hex64(k.plaintext_hex);
    }
    {  // NIST SP 800-67 App. B: three blocks in one batch
        const TripleSchedule ts = triple_schedule(parse_hex_key("0123456789ABCDEF23456789ABCDEF01456789ABCDEF0123"));
        const auto pt = unhex("54686520717566636B2062726F776E20666F78206A756D70");
        const auto want = unhex("A826FD8CE53B855FCCE21C8112256FE668D5C05DD9B6B900");
        std::vector<std::uint8_t> ct(pt.size()), back(pt.size());
        encrypt_batch(pt, ct, ts, cfg);
        decrypt_batch(ct, back, ts, cfg);
        pass &= ct == want && back == pt;
    }
    all &= check(out, "3DES known-answer vectors (all keying options, SP 800-67 batch)", pass);

    // DES round trips and E_{~k}(~x) = ~E_k(x), 256 random keys: each key's
    // 33 random blocks as one batch
    std::mt19937_64 rng(0xC0FFEE);
    pass = true;
    for (int i = 0; i < 256 && pass; ++i) {
        const std::uint64_t k = rng();
        std::vector<std::uint8_t> x(8 * 33), y(x.size()), z(x.size()), nx(x.size()), ny(x.size());
        for (auto& b : x) b = static_cast<std::uint8_t>(rng());
        for (std::size_t j = 0; j < x.size(); ++j) nx[j] = static_cast<std::uint8_t>(~x[j]);
        const TripleSchedule ts = single(key_schedule(DesKey{k}));
        encrypt_batch(x, y, ts, cfg);
        decrypt_batch(y, z, ts, cfg);
        encrypt_batch(nx, ny, single(key_schedule(DesKey{~k})), cfg);
        pass &= z == x;
        for (std::size_t j = 0; j < x.size(); ++j) pass &= ny[j] == static_cast<std::uint8_t>(~y[j]);
    }
    all &= check(out, "DES round-trip and complementation", pass);

    // Option-3 keys collapse EDE to single DES; 3-key round trips
    pass = true;
    for (int i = 0; i < 256 && pass; ++i) {
        const std::uint64_t k = rng();
        char hex[17];
        std::snprintf(hex, sizeof hex, "%016llX", static_cast<unsigned long long>(k));
        const TripleSchedule ts3 = triple_schedule(parse_hex_key(hex));
        TripleKey key3;
        key3.k1.raw = rng();
        key3.k2.raw = rng();
        key3.k3.raw = rng();
        const TripleSchedule ts1 = triple_schedule(key3);
        std::vector<std::uint8_t> x(8 * 33), a(x.size()), b(x.size()), c(x.size());
        for (auto& v : x) v = static_cast<std::uint8_t>(rng());
        encrypt_batch(x, a, ts3, cfg);
        encrypt_batch(x, b, single(key_schedule(DesKey{k})), cfg);
        pass &= a == b;
        encrypt_batch(x, a, ts1, cfg);
        decrypt_batch(a, c, ts1, cfg);
        pass &= c == x;
    }
    all &= check(out, "EDE collapse and 3-key round trips", pass);

    out << (all ? "verification PASSED\n" : "verification FAILED\n");
    return all;
}

}  // namespace t3des

extern "C" int t3des_cu_run_verification(int device, char* report, std::size_t capacity) {
    std::ostringstream os;
    int rc = T3DES_CU_OK;
    try {
        t3des::DispatchConfig cfg;
        cfg.device = device;
        if (!t3des::run_verification(os, cfg)) rc = T3DES_CU_ERR_ARG;
    } catch (const t3des::CudaError& e) {
        os << "error: " << e.what() << '\n';
        rc = e.status;
    } catch (const std::exception& e) {
        os << "error: " << e.what() << '\n';
        rc = T3DES_CU_ERR_ARG;
    }
    if (report && capacity) {
        const std::string s = os.str();
        const std::size_t n = std::min(s.size(), capacity - 1);
        std::memcpy(report, s.data(), n);
        report[n] = '\0';
    }
    return rc;
}
