// Drop-in check: the REFERENCE library (patched with
// integration/reference_backend_cuda.patch) running its own public API —
// encrypt_batch/decrypt_batch and encrypt_stream/decrypt_stream — on
// Backend::Cuda, compared byte for byte with its own Backend::Threaded.
// Prints "ok" on success.
#include <cstdio>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "t3des/dispatch.hpp"
#include "t3des/tdes.hpp"

using namespace t3des;

int main() {
    const TripleSchedule ts = triple_schedule(parse_hex_key("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57"));
    std::mt19937_64 rng(7);
    for (std::size_t n : {1ul, 1023ul, 8195ul, 1ul << 20}) {
        std::vector<std::uint8_t> in(8 * n), cpu(in.size()), gpu(in.size()), back(in.size());
        for (auto& b : in) b = static_cast<std::uint8_t>(rng());
        DispatchConfig c_cpu, c_gpu;
        c_cpu.backend = Backend::Threaded;
        c_gpu.backend = Backend::Cuda;
        encrypt_batch(in, cpu, ts, c_cpu);
        encrypt_batch(in, gpu, ts, c_gpu);
        if (gpu != cpu) { std::printf("encrypt mismatch n=%zu\n", n); return 1; }
        decrypt_batch(gpu, back, ts, c_gpu);
        if (back != in) { std::printf("decrypt mismatch n=%zu\n", n); return 1; }
    }
    // cfg.workers > 1: min(workers, GPUs) block-range shards on consecutive
    // GPUs (on a one-GPU box: one shard, whatever workers is)
    for (unsigned w : {2u, 3u}) {
        for (std::size_t n : {1ul, 2047ul, 100003ul, 3ul << 20}) {
            std::vector<std::uint8_t> in(8 * n), cpu(in.size()), gpu(in.size()), back(in.size());
            for (auto& b : in) b = static_cast<std::uint8_t>(rng());
            DispatchConfig c_cpu, c_gpu;
            c_cpu.backend = Backend::Threaded;
            c_gpu.backend = Backend::Cuda;
            c_gpu.workers = w;
            encrypt_batch(in, cpu, ts, c_cpu);
            encrypt_batch(in, gpu, ts, c_gpu);
            if (gpu != cpu) { std::printf("workers=%u encrypt mismatch n=%zu\n", w, n); return 1; }
            decrypt_batch(gpu, back, ts, c_gpu);
            if (back != in) { std::printf("workers=%u decrypt mismatch n=%zu\n", w, n); return 1; }
        }
    }
    // the reference's own stream loop, chunk by chunk on the GPU backend
    std::string payload(100003, '\0');
    for (auto& ch : payload) ch = static_cast<char>(rng());
    DispatchConfig c_gpu, c_cpu;
    c_gpu.backend = Backend::Cuda;
    c_cpu.backend = Backend::Threaded;
    c_gpu.chunk_blocks = c_cpu.chunk_blocks = 1000;
    std::istringstream i1(payload), i2(payload);
    std::ostringstream o1, o2;
    encrypt_stream(i1, o1, ts, c_gpu, PaddingMode::Pkcs7);
    encrypt_stream(i2, o2, ts, c_cpu, PaddingMode::Pkcs7);
    if (o1.str() != o2.str()) { std::puts("stream mismatch"); return 1; }
    std::istringstream i3(o1.str());
    std::ostringstream o3;
    decrypt_stream(i3, o3, ts, c_gpu, PaddingMode::Pkcs7);
    if (o3.str() != payload) { std::puts("stream round trip mismatch"); return 1; }
    // errors keep the reference's types
    std::vector<std::uint8_t> bad(12), bad_out(12);
    try { encrypt_batch(bad, bad_out, ts, c_gpu); std::puts("no length error"); return 1; }
    catch (const InputLengthError&) {}
    std::puts("ok");
    return 0;
}
