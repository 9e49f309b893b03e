// C++ host API of the B200 3DES-ECB engine, mirroring the reference's hot
// path API so C++ callers switch by changing the include and the link line:
//
//   reference (/root/reference/proj/include/t3des)    this header
//   tdes.hpp:14-23  KeyingOption, TripleKey          same names
//   tdes.hpp:32     parse_hex_key                    same signature
//   des.hpp:33-35   key_schedule                     same signature
//   tdes.hpp:36-42  TripleSchedule, triple_schedule  same layout (pass-major)
//   des.hpp:30-31   load_block / store_block         same (big-endian)
//   dispatch.hpp:19-30  Backend, DispatchConfig      + Backend::Cuda (default)
//   dispatch.hpp:39-42  plan_dispatch, ChunkSpan     same
//   dispatch.hpp:64-69  encrypt_batch/decrypt_batch  same signatures
//   dispatch.hpp:44-47, tdes.hpp:25-28  InputLengthError, KeyFormatError
//   dispatch.hpp:32,49-91  PaddingMode, PaddingError, IoError, StreamReport,
//                      encrypt_stream/decrypt_stream, pkcs7_pad/pkcs7_unpad
//   dispatch.hpp:94    resolve_workers                  same (GPU shards)
//   tdes.hpp:34        to_hex                           same format
//   des.hpp:25-28,41-48  ParityError, has_odd_parity, normalize_parity,
//                      is_weak_key, is_semiweak_key     same semantics
//   des.hpp:37-39, tdes.hpp:44-54  encrypt_block/decrypt_block,
//                      tdes_{en,de}crypt_block[_fast]   one block through the
//                                                       device (see below)
//   verify.hpp:14-37   DesKat, TdesKat, des_kats, tdes_kats,
//                      walkthrough_subkeys, kWalkthroughKey, run_verification
//
// Backend::Cuda sends the whole batch through the C ABI (t3des_cu.h) in
// one call; there is no CPU cipher in this library (ScalarReference and
// Threaded are the reference's own CPU backends and throw here).
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <iosfwd>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace t3des {

using Block = std::uint64_t;
using RoundKeySet = std::array<std::uint64_t, 16>;

struct DesKey {
    std::uint64_t raw = 0;
};

enum class KeyingOption { Option1, Option2, Option3 };

struct TripleKey {
    DesKey k1, k2, k3;
    KeyingOption option = KeyingOption::Option1;
};

class KeyFormatError : public std::runtime_error {
  public:
    using std::runtime_error::runtime_error;
};

class InputLengthError : public std::runtime_error {
  public:
    using std::runtime_error::runtime_error;
};

class PaddingError : public std::runtime_error {
  public:
    using std::runtime_error::runtime_error;
};

class IoError : public std::runtime_error {
  public:
    IoError(const std::string& what, std::uint64_t offset) : std::runtime_error(what), byte_offset(offset) {}
    std::uint64_t byte_offset;
};

// CUDA runtime / device failures (no device is an error, never a fallback).
class CudaError : public std::runtime_error {
  public:
    CudaError(const std::string& what, int code) : std::runtime_error(what), status(code) {}
    int status;
};

class ParityError : public std::runtime_error {
  public:
    using std::runtime_error::runtime_error;
};

TripleKey parse_hex_key(std::string_view hex);
std::string to_hex(const TripleKey& key);
RoundKeySet key_schedule(DesKey key);

// Key hygiene (host only): odd parity in the LSB of every byte; the 4 weak
// and 12 semi-weak keys compared with the parity bits masked off.
bool has_odd_parity(DesKey key);
DesKey normalize_parity(DesKey key);
bool is_weak_key(DesKey key);
bool is_semiweak_key(DesKey key);

struct TripleSchedule {
    RoundKeySet pass1, pass2, pass3;
};
TripleSchedule triple_schedule(const TripleKey& key);

Block load_block(std::span<const std::uint8_t, 8> bytes);
void store_block(Block b, std::span<std::uint8_t, 8> out);

enum class Backend {
    ScalarReference,  // reference CPU oracle — not in this library
    Threaded,         // reference OpenMP backend — not in this library
    NoOpCopy,         // copy only (timing instrumentation), as in the reference
    Cuda,             // B200 kernels through the C ABI
};

struct DispatchConfig {
    std::size_t chunk_blocks = 131072;  // reference meaning; the CUDA backend sends the
                                        // whole batch per call (blocks per launch only
                                        // when gpu_chunked is set)
    std::size_t work_group = 256;       // CUDA: threads per CTA hint (used when gpu_chunked)
    unsigned workers = 0;               // CUDA: block-range shards, at most one per GPU, from `device` (0 = 1)
    Backend backend = Backend::Cuda;
    int device = 0;                     // first CUDA device
    int variant = 6;                    // T3DES_CU_VARIANT_*: 6 auto (default), 0 bitsliced, 1 SP-table,
                                        // 7 key-specialised (NVRTC at run time, opt-in)
    bool gpu_chunked = false;           // apply chunk_blocks/work_group to launches
};

struct ChunkSpan {
    std::size_t offset;  // in blocks
    std::size_t length;  // in blocks
};

std::vector<ChunkSpan> plan_dispatch(std::size_t total_blocks, const DispatchConfig& cfg);

// Backend::Cuda: the number of block-range shards a batch is split into
// (workers == 0 means 1; each shard runs on its own GPU context).
unsigned resolve_workers(const DispatchConfig& cfg);

void encrypt_batch(std::span<const std::uint8_t> in, std::span<std::uint8_t> out,
                   const TripleSchedule& ts, const DispatchConfig& cfg);
void decrypt_batch(std::span<const std::uint8_t> in, std::span<std::uint8_t> out,
                   const TripleSchedule& ts, const DispatchConfig& cfg);

// Opt-in page-locking of a buffer the caller passes to many batch calls
// (t3des_cu_host_register): the host path then DMAs straight from/to it
// instead of staging it.  RAII: unregisters on destruction, which must come
// before the memory is freed.
class HostRegistration {
  public:
    explicit HostRegistration(std::span<std::uint8_t> buf);
    ~HostRegistration();
    HostRegistration(const HostRegistration&) = delete;
    HostRegistration& operator=(const HostRegistration&) = delete;

  private:
    void* p_ = nullptr;
};

enum class PaddingMode { None, Pkcs7 };

struct StreamReport {
    std::uint64_t bytes_in = 0;
    std::uint64_t bytes_out = 0;
    std::uint64_t chunks = 0;
    double compute_seconds = 0.0;  // engine time not overlapped with I/O
    double io_seconds = 0.0;       // reads and writes
};

// Chunked streams (chunk = cfg.chunk_blocks blocks), Backend::Cuda only:
// chunk k+1 is read while chunk k runs on the GPU.  Same bytes, padding and
// errors as the reference's encrypt_stream/decrypt_stream.
StreamReport encrypt_stream(std::istream& source, std::ostream& sink, const TripleSchedule& ts,
                            const DispatchConfig& cfg, PaddingMode pad);
StreamReport decrypt_stream(std::istream& source, std::ostream& sink, const TripleSchedule& ts,
                            const DispatchConfig& cfg, PaddingMode pad);

// PKCS#7 over 8-byte blocks: always appends 1..8 bytes; unpad throws PaddingError.
void pkcs7_pad(std::vector<std::uint8_t>& data);
void pkcs7_unpad(std::vector<std::uint8_t>& data);

// Single-block transforms with the reference's signatures.  This library
// has no CPU cipher: each call is a one-block batch through the engine on
// device 0 (tens of microseconds), for code ported from the reference that
// checks a block or two; bulk work belongs in encrypt_batch/decrypt_batch.
// encrypt_block/decrypt_block are single DES under one 16-key schedule
// (run as the collapsed EDE (ks, ks, ks)); the _fast names equal the plain
// ones, as the reference's two routes do.
Block encrypt_block(Block block, const RoundKeySet& ks);
Block decrypt_block(Block block, const RoundKeySet& ks);
Block tdes_encrypt_block(Block block, const TripleSchedule& ts);
Block tdes_decrypt_block(Block block, const TripleSchedule& ts);
Block tdes_encrypt_block_fast(Block block, const TripleSchedule& ts);
Block tdes_decrypt_block_fast(Block block, const TripleSchedule& ts);

// Known-answer vectors and the self-check behind the CLI's `verify`.
struct DesKat {
    std::uint64_t key;
    std::uint64_t plaintext;
    std::uint64_t ciphertext;
};

struct TdesKat {
    std::string_view key_hex;
    std::string_view plaintext_hex;  // one block
    std::string_view ciphertext_hex;
};

std::span<const DesKat> des_kats();
std::span<const TdesKat> tdes_kats();
std::span<const std::uint64_t> walkthrough_subkeys();
constexpr std::uint64_t kWalkthroughKey = 0x133457799BBCDFF1ull;

// Runs the vectors and structural properties (round trips, EDE collapse,
// complementation) on the GPU named by cfg (Backend::Cuda); one line per
// group, then "verification PASSED" / "verification FAILED".
bool run_verification(std::ostream& out);
bool run_verification(std::ostream& out, const DispatchConfig& cfg);

}  // namespace t3des
