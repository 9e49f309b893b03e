// C++ host API (include/t3des_b200/t3des.hpp) over the C ABI.
#include "t3des_b200/t3des.hpp"

#include <cstring>
#include <istream>
#include <map>
#include <memory>
#include <ostream>

#include "schedule.hpp"
#include "stream.hpp"
#include "t3des_cu.h"

namespace t3des {
namespace {

[[noreturn]] void raise(int rc) {
    if (rc == T3DES_CU_ERR_LENGTH || rc == T3DES_CU_ERR_OVERLAP)
        throw InputLengthError(t3des_cu_strerror(rc));
    if (rc == T3DES_CU_ERR_KEY) throw KeyFormatError(t3des_cu_strerror(rc));
    if (rc == T3DES_CU_ERR_PADDING) throw PaddingError(t3des_cu_strerror(rc));
    throw CudaError(std::string("t3des_cu: ") + t3des_cu_strerror(rc), rc);
}

struct CtxDeleter {
    void operator()(t3des_cu_ctx* c) const { t3des_cu_destroy(c); }
};

// One context per device per submitting thread (SPEC.md:233 threading).
t3des_cu_ctx* context_for(int device) {
    thread_local std::map<int, std::unique_ptr<t3des_cu_ctx, CtxDeleter>> cache;
    auto it = cache.find(device);
    if (it != cache.end()) return it->second.get();
    t3des_cu_ctx* c = nullptr;
    const int rc = t3des_cu_create(device, &c);
    if (rc) raise(rc);
    cache.emplace(device, std::unique_ptr<t3des_cu_ctx, CtxDeleter>(c));
    return c;
}

void flatten(const TripleSchedule& ts, std::uint64_t sub48[48]) {
    std::memcpy(sub48, ts.pass1.data(), 16 * 8);
    std::memcpy(sub48 + 16, ts.pass2.data(), 16 * 8);
    std::memcpy(sub48 + 32, ts.pass3.data(), 16 * 8);
}

// Reference run_batch (dispatch.cpp:88-109) with the CUDA branch taken
// before the span loop: one C-ABI call per batch.
void run_batch(std::span<const std::uint8_t> in, std::span<std::uint8_t> out, const TripleSchedule& ts,
               const DispatchConfig& cfg, int dir) {
    if (in.size() % 8 != 0)
        throw InputLengthError("batch length " + std::to_string(in.size()) + " is not a multiple of 8 bytes");
    if (out.size() != in.size()) throw InputLengthError("output buffer size mismatch");
    const auto* ib = in.data();
    if (out.data() != ib && out.data() < ib + in.size() && out.data() + out.size() > ib)
        throw InputLengthError("partially overlapping buffers");
    switch (cfg.backend) {
        case Backend::NoOpCopy:
            if (out.data() != ib && !in.empty()) std::memmove(out.data(), ib, in.size());
            return;
        case Backend::ScalarReference:
        case Backend::Threaded:
            throw std::invalid_argument(
                "t3des B200 engine: only Backend::Cuda (and NoOpCopy) are provided; the CPU backends "
                "live in the reference library");
        case Backend::Cuda:
            break;
    }
    if (in.empty()) return;
    std::uint64_t sub48[48];
    flatten(ts, sub48);
    int rc;
    if (cfg.workers > 1) {  // min(workers, GPUs) shards on consecutive GPUs from cfg.device
        rc = t3des_cu_ecb_workers(cfg.workers, cfg.device, sub48, dir, ib, out.data(), in.size());
    } else {
        t3des_cu_ctx* c = context_for(cfg.device);
        rc = t3des_cu_set_schedule(c, sub48);
        if (!rc) rc = t3des_cu_set_variant(c, cfg.variant);
        if (!rc)
            rc = cfg.gpu_chunked ? t3des_cu_set_launch(c, cfg.chunk_blocks, static_cast<int>(cfg.work_group))
                                 : t3des_cu_set_launch(c, 0, 0);
        if (!rc) rc = t3des_cu_ecb_host(c, dir, ib, out.data(), in.size());
    }
    if (rc) raise(rc);
}

struct IstreamSource : t3b::ByteSource {
    std::istream& in;
    explicit IstreamSource(std::istream& s) : in(s) {}
    std::size_t read(std::uint8_t* dst, std::size_t n) override {
        in.read(reinterpret_cast<char*>(dst), static_cast<std::streamsize>(n));
        if (in.bad()) throw std::runtime_error("read failure");
        return static_cast<std::size_t>(in.gcount());
    }
};

struct OstreamSink : t3b::ByteSink {
    std::ostream& out;
    explicit OstreamSink(std::ostream& s) : out(s) {}
    void write(const std::uint8_t* src, std::size_t n) override {
        out.write(reinterpret_cast<const char*>(src), static_cast<std::streamsize>(n));
        if (!out) throw std::runtime_error("write failure");
    }
    void flush() override { out.flush(); }
};

StreamReport run_stream(std::istream& source, std::ostream& sink, const TripleSchedule& ts,
                        const DispatchConfig& cfg, PaddingMode pad, int dir) {
    if (cfg.backend != Backend::Cuda && cfg.backend != Backend::NoOpCopy)
        throw std::invalid_argument("t3des B200 engine: streams run on Backend::Cuda (or NoOpCopy) only");
    if (cfg.chunk_blocks == 0) throw std::invalid_argument("chunk_blocks must be positive");
    std::uint64_t sub48[48];
    flatten(ts, sub48);
    t3des_cu_ctx* c = context_for(cfg.device);
    int rc = t3des_cu_set_schedule(c, sub48);
    if (!rc) rc = t3des_cu_set_variant(c, cfg.variant);
    if (!rc) rc = t3des_cu_set_launch(c, 0, 0);
    if (rc) raise(rc);
    IstreamSource src(source);
    OstreamSink dst(sink);
    try {
        const t3b::StreamStats s = t3b::run_stream(c, dir, src, dst, cfg.chunk_blocks, pad == PaddingMode::Pkcs7, 0,
                                                   cfg.backend == Backend::NoOpCopy);
        return StreamReport{s.bytes_in, s.bytes_out, s.chunks, s.compute_seconds, s.io_seconds};
    } catch (const t3b::StreamFailure& f) {
        switch (f.kind) {
            case t3b::StreamFailure::Length: throw InputLengthError(f.what());
            case t3b::StreamFailure::Padding: throw PaddingError(f.what());
            case t3b::StreamFailure::Io: throw IoError(f.what(), f.byte_offset);
            default: throw CudaError(f.what(), f.status);
        }
    }
}

}  // namespace

StreamReport encrypt_stream(std::istream& source, std::ostream& sink, const TripleSchedule& ts,
                            const DispatchConfig& cfg, PaddingMode pad) {
    return run_stream(source, sink, ts, cfg, pad, T3DES_CU_ENCRYPT);
}

StreamReport decrypt_stream(std::istream& source, std::ostream& sink, const TripleSchedule& ts,
                            const DispatchConfig& cfg, PaddingMode pad) {
    return run_stream(source, sink, ts, cfg, pad, T3DES_CU_DECRYPT);
}

HostRegistration::HostRegistration(std::span<std::uint8_t> buf) {
    if (buf.empty()) return;
    if (int rc = t3des_cu_host_register(buf.data(), buf.size())) raise(rc);
    p_ = buf.data();
}

HostRegistration::~HostRegistration() {
    if (p_) t3des_cu_host_unregister(p_);
}

void pkcs7_pad(std::vector<std::uint8_t>& data) {
    const std::size_t len = data.size();
    data.resize(len + 8 - len % 8);
    std::size_t n = 0;
    t3b::pkcs7_pad_bytes(data.data(), len, &n);
}

void pkcs7_unpad(std::vector<std::uint8_t>& data) {
    try {
        data.resize(t3b::pkcs7_unpad_len(data.data(), data.size()));
    } catch (const t3b::StreamFailure& f) {
        throw PaddingError(f.what());
    }
}

TripleKey parse_hex_key(std::string_view hex) {
    std::uint64_t k[3];
    const int opt = t3b::parse_hex_key(hex.data(), hex.size(), k);
    if (opt == -1)
        throw KeyFormatError("key must be 16, 32 or 48 hex characters, got " + std::to_string(hex.size()));
    if (opt < 0) throw KeyFormatError("invalid hex character in key");
    TripleKey key;
    key.k1.raw = k[0];
    key.k2.raw = k[1];
    key.k3.raw = k[2];
    key.option = opt == 1 ? KeyingOption::Option1 : (opt == 2 ? KeyingOption::Option2 : KeyingOption::Option3);
    return key;
}

// Reference to_hex (tdes.hpp:34): upper-case hex of the keys the option
// carries (k1 k2 k3 / k1 k2 / k1).
std::string to_hex(const TripleKey& key) {
    const int n = key.option == KeyingOption::Option1 ? 3 : (key.option == KeyingOption::Option2 ? 2 : 1);
    const std::uint64_t k[3] = {key.k1.raw, key.k2.raw, key.k3.raw};
    static const char digits[] = "0123456789ABCDEF";
    std::string s;
    for (int i = 0; i < n; ++i)
        for (int nib = 15; nib >= 0; --nib) s += digits[(k[i] >> (4 * nib)) & 0xF];
    return s;
}

bool has_odd_parity(DesKey key) { return t3des_cu_des_key_flags(key.raw) & T3DES_CU_KEY_ODD_PARITY; }
DesKey normalize_parity(DesKey key) { return DesKey{t3des_cu_normalize_parity(key.raw)}; }
bool is_weak_key(DesKey key) { return t3des_cu_des_key_flags(key.raw) & T3DES_CU_KEY_WEAK; }
bool is_semiweak_key(DesKey key) { return t3des_cu_des_key_flags(key.raw) & T3DES_CU_KEY_SEMIWEAK; }

RoundKeySet key_schedule(DesKey key) {
    RoundKeySet ks{};
    t3b::des_key_schedule(key.raw, ks.data());
    return ks;
}

TripleSchedule triple_schedule(const TripleKey& key) {
    return TripleSchedule{key_schedule(key.k1), key_schedule(key.k2), key_schedule(key.k3)};
}

Block load_block(std::span<const std::uint8_t, 8> bytes) {
    Block b = 0;
    for (int i = 0; i < 8; ++i) b |= static_cast<Block>(bytes[i]) << (56 - 8 * i);
    return b;
}

void store_block(Block b, std::span<std::uint8_t, 8> out) {
    for (int i = 0; i < 8; ++i) out[i] = static_cast<std::uint8_t>(b >> (56 - 8 * i));
}

std::vector<ChunkSpan> plan_dispatch(std::size_t total_blocks, const DispatchConfig& cfg) {
    std::vector<ChunkSpan> spans;
    const std::size_t step = cfg.chunk_blocks ? cfg.chunk_blocks : (total_blocks ? total_blocks : 1);
    for (std::size_t off = 0; off < total_blocks; off += step)
        spans.push_back(ChunkSpan{off, step < total_blocks - off ? step : total_blocks - off});
    return spans;
}

unsigned resolve_workers(const DispatchConfig& cfg) { return cfg.workers ? cfg.workers : 1u; }

void encrypt_batch(std::span<const std::uint8_t> in, std::span<std::uint8_t> out, const TripleSchedule& ts,
                   const DispatchConfig& cfg) {
    run_batch(in, out, ts, cfg, T3DES_CU_ENCRYPT);
}

void decrypt_batch(std::span<const std::uint8_t> in, std::span<std::uint8_t> out, const TripleSchedule& ts,
                   const DispatchConfig& cfg) {
    run_batch(in, out, ts, cfg, T3DES_CU_DECRYPT);
}

}  // namespace t3des
