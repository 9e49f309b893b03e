// Probe: t3des_cu_ecb_workers on a 64 MiB pageable batch for workers 1/2/4
// (one GPU: several contexts on it), every repetition timed; and the first
// and second run_verification calls of a process.
#include <chrono>
#include <cstdio>
#include <sstream>
#include <vector>

#include "t3des_b200/bench.hpp"
#include "t3des_b200/t3des.hpp"
#include "t3des_cu.h"

int main() {
    using clk = std::chrono::steady_clock;
    auto t0 = clk::now();
    std::ostringstream os;
    bool ok = t3des::run_verification(os);
    double a = std::chrono::duration<double>(clk::now() - t0).count();
    t0 = clk::now();
    ok = ok && t3des::run_verification(os);
    double b = std::chrono::duration<double>(clk::now() - t0).count();
    std::printf("run_verification first %.3f s, second %.3f s, ok %d\n", a, b, int(ok));
    const auto payload = t3des::bench::make_payload(64ull << 20, 1);
    std::vector<std::uint8_t> out(payload.size());
    const auto ts = t3des::triple_schedule(t3des::parse_hex_key("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57"));
    // 8 shards first (8 pooled contexts on one GPU), then the shapes the
    // reference's acceptance criterion 5 sweeps
    for (unsigned w : {8u, 1u, 2u, 4u, 2u, 3u, 1u}) {
        t3des::DispatchConfig cfg;
        cfg.workers = w;
        std::printf("workers %u:", w);
        for (int rep = 0; rep < 5; ++rep) {
            t0 = clk::now();
            t3des::encrypt_batch(payload, out, ts, cfg);
            std::printf(" %.2f", std::chrono::duration<double>(clk::now() - t0).count() * 1e3);
        }
        std::printf(" ms\n");
    }
    return 0;
}
