// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// extern "C" wrapper around the UNMODIFIED reference library, compiled
// together with /root/reference/proj/src/*.cpp (where they lie) by
// oracle/Makefile into oracle/_ref/libt3des_ref.so.  Used by the tests to
// pin the C oracle against the reference itself, and by bench.py as the
// reference CPU arm (Backend::Threaded, OpenMP over all host cores).
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <sstream>
#include <string>

#include "t3des/bench.hpp"
#include "t3des/dispatch.hpp"
#include "t3des/tdes.hpp"
#include "t3des/verify.hpp"

using namespace t3des;

namespace {

int to_code(const std::exception& e) {
    if (dynamic_cast<const InputLengthError*>(&e)) return 1;
    if (dynamic_cast<const KeyFormatError*>(&e)) return 4;
    return 9;
}

}  // namespace

extern "C" {

// Parse a hex key and write the 48 pass-major subkeys (tdes.hpp:32-42).
int ref_schedule_hex(const char* hex, std::uint64_t sub48[48], int* option) {
    try {
        TripleKey k = parse_hex_key(std::string_view(hex));
        TripleSchedule ts = triple_schedule(k);
        std::memcpy(sub48, ts.pass1.data(), 16 * 8);
        std::memcpy(sub48 + 16, ts.pass2.data(), 16 * 8);
        std::memcpy(sub48 + 32, ts.pass3.data(), 16 * 8);
        if (option) *option = static_cast<int>(k.option) + 1;
        return 0;
    } catch (const std::exception& e) {
        return to_code(e);
    }
}

// encrypt_batch / decrypt_batch (dispatch.hpp:64-69).  backend: 0 scalar
// reference, 1 threaded (OpenMP), 2 no-op copy.
int ref_ecb(const std::uint8_t* in, std::uint8_t* out, std::size_t len,
            const std::uint64_t sub48[48], int decrypt, int backend,
            unsigned workers, std::size_t chunk_blocks, std::size_t work_group) {
    try {
        TripleSchedule ts;
        std::memcpy(ts.pass1.data(), sub48, 16 * 8);
        std::memcpy(ts.pass2.data(), sub48 + 16, 16 * 8);
        std::memcpy(ts.pass3.data(), sub48 + 32, 16 * 8);
        DispatchConfig cfg;
        cfg.backend = backend == 0 ? Backend::ScalarReference
                      : backend == 1 ? Backend::Threaded
                                     : Backend::NoOpCopy;
        cfg.workers = workers;
        if (chunk_blocks) cfg.chunk_blocks = chunk_blocks;
        if (work_group) cfg.work_group = work_group;
        std::span<const std::uint8_t> si(in, len);
        std::span<std::uint8_t> so(out, len);
        if (decrypt)
            decrypt_batch(si, so, ts, cfg);
        else
            encrypt_batch(si, so, ts, cfg);
        return 0;
    } catch (const std::exception& e) {
        return to_code(e);
    }
}

std::uint64_t ref_tdes_block(std::uint64_t b, const std::uint64_t sub48[48], int decrypt,
                             int fast) {
    TripleSchedule ts;
    std::memcpy(ts.pass1.data(), sub48, 16 * 8);
    std::memcpy(ts.pass2.data(), sub48 + 16, 16 * 8);
    std::memcpy(ts.pass3.data(), sub48 + 32, 16 * 8);
    if (fast) return decrypt ? tdes_decrypt_block_fast(b, ts) : tdes_encrypt_block_fast(b, ts);
    return decrypt ? tdes_decrypt_block(b, ts) : tdes_encrypt_block(b, ts);
}

void ref_make_payload(std::uint8_t* out, std::uint64_t bytes, std::uint64_t seed) {
    auto v = bench::make_payload(bytes, seed);
    std::memcpy(out, v.data(), v.size());
}

unsigned ref_resolve_workers(unsigned workers) {
    DispatchConfig cfg;
    cfg.workers = workers;
    return resolve_workers(cfg);
}

// Key hygiene (des.hpp:41-48): bit 0 odd parity, bit 1 weak, bit 2 semi-weak.
int ref_key_flags(std::uint64_t k) {
    const DesKey key{k};
    return (has_odd_parity(key) ? 1 : 0) | (is_weak_key(key) ? 2 : 0) | (is_semiweak_key(key) ? 4 : 0);
}

std::uint64_t ref_normalize_parity(std::uint64_t k) { return normalize_parity(DesKey{k}).raw; }

// to_hex(parse_hex_key(hex)) (tdes.hpp:32-34) into out (>= 49 bytes).
int ref_to_hex(const char* hex, char* out) {
    try {
        const std::string s = to_hex(parse_hex_key(std::string_view(hex)));
        std::memcpy(out, s.c_str(), s.size() + 1);
        return 0;
    } catch (const std::exception& e) {
        return to_code(e);
    }
}

int ref_run_verification(void) {
    std::ostringstream os;
    return run_verification(os) ? 0 : 1;
}

}  // extern "C"
