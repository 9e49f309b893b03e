// C ABI of the B200 3DES-ECB engine (declared in include/t3des_cu.h).
//
// Owns: device selection, per-context streams and staging buffers, the
// host-flattened key tables, kernel launch shaping, the pipelined
// host-buffer paths (pinned DMA pipeline, zero-copy, pageable staging) and
// the utility entries; the multi-GPU entries are in multi.cu, the stream
// entry in stream.cu.  No exception crosses this boundary and there is no
// CPU fallback.
#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <thread>
#include <vector>

#include "kernels.cuh"
#include "schedule.hpp"
#include "t3des_cu.h"

#include "ctx.hpp"
#include "hoststage.hpp"

namespace {

constexpr std::uint64_t kSpMinThreads = 128;  // SP-table CTA size floor for small batches
// pinned host batches up to this size run zero-copy (kernel on the mapped pages)
constexpr std::size_t kZeroCopyMaxBytes = std::size_t(64) << 20;  // scripts/zerocopy_{sweep,big}.py
// pageable batches up to this size run their stages zero-copy on the pinned slots
constexpr std::size_t kStagedZeroCopyMaxBytes = std::size_t(12) << 20;
using t3b::kMaxCopyThreads;
// SP-table launches that may use PDL (scripts/pdl_ab.py: 8-128 KiB enc+dec
// chains 12.3 -> 7.7 us per pair; from 256 KiB the early CTAs cost more)
constexpr std::uint64_t kPdlMaxBlocks = 16384;
// first/last stage size of the pinned DMA pipeline's ramp (large batches)
constexpr std::size_t kRampBytes = std::size_t(8) << 20;  // scripts/ramp_sweep.py
constexpr int kSpSmemBytes = 8 * 64 * 32 * 4 + int(sizeof(T3SpKeyParam)) + 8 * 64 * 4;  // 64 KiB tables, round keys, staging

using t3b::DeviceScope;

#define T3_CK(call)                                   \
    do {                                              \
        if ((call) != cudaSuccess) {                  \
            (void)cudaGetLastError();                 \
            return T3DES_CU_ERR_CUDA;                 \
        }                                             \
    } while (0)

using t3b::partial_overlap;

using t3b::fault_at;

int launch_sptable(t3des_cu_ctx* c, int dir, const std::uint8_t* in, std::uint8_t* out,
                   std::uint64_t nblocks, cudaStream_t s);

int launch_bitslice(t3des_cu_ctx* c, int dir, const std::uint8_t* in, std::uint8_t* out,
                    std::uint64_t nblocks, cudaStream_t s) {
    const std::uint64_t full = nblocks / T3_TILE_BLOCKS;
    const bool tail = (nblocks % T3_TILE_BLOCKS) != 0;
    // AUTO: the partial last tile (< 1024 blocks) runs on the SP-table kernel
    // (one thread per block, ~10 us instead of ~18 us for a 1-warp bitsliced
    // tile) on a side stream, concurrently with the full tiles.
    const bool side_tail =
        tail && full && (c->variant == T3DES_CU_VARIANT_AUTO || c->variant == T3DES_CU_VARIANT_KEYED);
    if (side_tail) {
        const std::uint64_t t0 = full * T3_TILE_BLOCKS;
        T3_CK(cudaEventRecord(c->ev_fork, s));
        T3_CK(cudaStreamWaitEvent(c->tail_st, c->ev_fork, 0));
        if (int rc = launch_sptable(c, dir, in + 8 * t0, out + 8 * t0, nblocks - t0, c->tail_st)) return rc;
        T3_CK(cudaEventRecord(c->ev_join, c->tail_st));
    }
    // work_group is a CTA-size hint; the bitsliced kernels are built for at
    // most T3_BS_THREADS threads (AUTO may pass a larger SP-table size)
    const int threads = c->work_group > 0 ? std::min(c->work_group, T3_BS_THREADS) : T3_BS_THREADS;
    if (full) {
        const std::uint64_t warps_per_cta = std::uint64_t(threads) / 32;
        std::uint64_t grid = (full + warps_per_cta - 1) / warps_per_cta;
        // Oversubscribed grid: ~64 CTAs per SM run as several waves; the
        // hardware CTA scheduler then balances the SMs and de-phases the
        // warps' load/compute cycles (measured: 2.87 ms vs 3.02 ms for a
        // persistent 4-CTA/SM grid on 1 GiB, scripts/grid_sweep.sh).
        // ... and it scales with the batch (about kTilesPerWarp tiles per warp)
        // so that warps never live long enough to fall into lockstep.
        constexpr std::uint64_t kTilesPerWarp = 4;
        const std::uint64_t cap =
            std::max<std::uint64_t>(std::uint64_t(c->sms) * std::uint64_t(c->bs_ctas_per_sm) *
                                        (T3_BS_THREADS / 32) / warps_per_cta,
                                    full / (warps_per_cta * kTilesPerWarp));
        grid = std::min<std::uint64_t>(grid, std::max<std::uint64_t>(cap, 1));
        const bool vec4 = ((reinterpret_cast<std::uintptr_t>(in) |
                            reinterpret_cast<std::uintptr_t>(out)) & 15u) == 0;
        const bool tma = vec4 && threads == T3_BS_THREADS && c->variant != T3DES_CU_VARIANT_BITSLICE_LDG;
        // tuning variants (A/B measurement of the T3_OPT_* code-generation options)
        const int opt = (c->variant == T3DES_CU_VARIANT_BITSLICE || c->variant == T3DES_CU_VARIANT_AUTO ||
                         c->variant == T3DES_CU_VARIANT_KEYED)
                            ? c->bs_opt
                        : c->variant == T3DES_CU_VARIANT_BITSLICE_ALU ? 0
                        : c->variant == T3DES_CU_VARIANT_BITSLICE_DFMA ? T3_OPT_DFMA
                                                                       : T3_OPT_SHRFMA;
        // key-specialised kernel (NVRTC, keyed.cpp): VARIANT_KEYED compiles it
        // on the first launch of a key unless t3des_cu_keyed_prepare ran; AUTO
        // takes it for its bitsliced launches once it has been prepared for the
        // installed schedule and this direction (never compiles on its own)
        const bool keyed = c->variant == T3DES_CU_VARIANT_KEYED ||
                           (c->variant == T3DES_CU_VARIANT_AUTO && c->keyed[dir] != nullptr);
        if (keyed && vec4) {
            if (int rc = t3b::keyed_launch(c, dir, in, out, full, s)) return rc;
        } else if (tma && c->rounds == 16 && opt == T3_OPT_DEFAULT_VALUE) {
            // collapsed EDE (K1 = K2 or K2 = K3): single DES, a third of the work
            t3_bs_tma_kernel<T3_OPT_DEFAULT_VALUE, 16>
                <<<unsigned(grid), threads, 0, s>>>(in, out, full, c->bs16[dir]);
        } else if (tma) {
            switch (opt) {
#define T3_TMA_CASE(O)                                                                                  \
    case O:                                                                                             \
        t3_bs_tma_kernel<O><<<unsigned(grid), threads, 0, s>>>(in, out, full, c->bs[dir]);             \
        break;
                T3_TMA_CASE(0)
                T3_TMA_CASE(1)
                T3_TMA_CASE(2)
                T3_TMA_CASE(3)
                T3_TMA_CASE(5)
                T3_TMA_CASE(7)
#undef T3_TMA_CASE
                default:
                    return T3DES_CU_ERR_ARG;
            }
        } else if (vec4)
            t3_bs_kernel<4, false><<<unsigned(grid), threads, 0, s>>>(in, out, 0, full, nblocks, c->bs[dir]);
        else
            t3_bs_kernel<2, false><<<unsigned(grid), threads, 0, s>>>(in, out, 0, full, nblocks, c->bs[dir]);
        T3_CK(cudaGetLastError());
        ++c->launches;
    }
    if (side_tail) {
        T3_CK(cudaStreamWaitEvent(s, c->ev_join, 0));
    } else if (tail) {
        t3_bs_kernel<2, true><<<1, 32, 0, s>>>(in, out, full, 1, nblocks, c->bs[dir]);
        T3_CK(cudaGetLastError());
        ++c->launches;
    }
    return T3DES_CU_OK;
}

// SP-table kernel instances (T3_SPV_* code-generation masks) compiled in.
#define T3_SPV_LIST(X) X(0) X(T3_SPV_DEFAULT)

const void* sp_kernel_fn(int spv) {
    switch (spv) {
#define T3_SPV_FN(V) \
    case V: return reinterpret_cast<const void*>(&t3_sp_kernel<V>);
        T3_SPV_LIST(T3_SPV_FN)
#undef T3_SPV_FN
        default: return nullptr;
    }
}

T3SpMul sp_mul() {
    T3SpMul m{};
    m.one = 1;
    for (int i = 1; i <= 4; ++i) m.m[i] = 1u << (32 - (20 - 4 * i));
    m.m[6] = 16;
    return m;
}

int launch_sptable(t3des_cu_ctx* c, int dir, const std::uint8_t* in, std::uint8_t* out,
                   std::uint64_t nblocks, cudaStream_t s) {
    // CTA size: 1024 threads (2 CTAs = 64 warps per SM, and the 64 KiB table
    // fill split 4x finer: 1 GiB 160 vs 140 GB/s with 256) once every SM gets
    // a full CTA; below that one CTA per SM with just enough threads, so a
    // small batch spreads over all SMs (scripts/sp_variant_sweep.py).
    const std::uint64_t per_sm = (nblocks + c->sms - 1) / std::uint64_t(c->sms);
    const int threads = c->work_group > 0 ? c->work_group
                        : per_sm >= std::uint64_t(T3_SP_THREADS_BIG)
                            ? T3_SP_THREADS_BIG
                            : int(std::max<std::uint64_t>(kSpMinThreads, (per_sm + 31) / 32 * 32));
    std::uint64_t grid = (nblocks + threads - 1) / threads;
    int occ = threads == T3_SP_THREADS ? c->sp_occ : threads == T3_SP_THREADS_BIG ? c->sp_occ_big : 0;
    if (!occ && grid > std::uint64_t(c->sms) &&
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sp_kernel_fn(c->sp_var), threads, kSpSmemBytes) != cudaSuccess)
        return T3DES_CU_ERR_CUDA;
    if (occ) grid = std::min<std::uint64_t>(grid, std::uint64_t(c->sms) * std::uint64_t(occ));
    const bool single = c->rounds == 16;
    const auto* sin = reinterpret_cast<const uint2*>(in);
    auto* sout = reinterpret_cast<uint2*>(out);
    const int passes = single ? 1 : 3;
    const std::uint32_t* keys = c->d_spk ? c->d_spk + (single ? 2 + dir : dir) * (sizeof(T3SpKeyParam) / 4) : nullptr;
    const T3SpKeyParam& kp = single ? c->sp16[dir] : c->sp[dir];
    static const T3SpMul mul = sp_mul();
    const unsigned g = unsigned(std::max<std::uint64_t>(grid, 1));
    // PDL masks: a launch of at most one CTA per SM may start while the
    // previous kernel on the stream is still running (its table fill overlaps
    // that kernel's tail; the kernel waits for it before touching the data).
    // Larger grids launch normally: early CTAs would hold SM resources.
    std::uint64_t pdl_max = kPdlMaxBlocks;
    if (const char* e = std::getenv("T3DES_PDL_MAX_BLOCKS")) pdl_max = std::strtoull(e, nullptr, 10);  // experiments
    const bool pdl = (c->sp_var & T3_SPV_PDL) && g <= unsigned(c->sms) && nblocks <= pdl_max;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(g);
    cfg.blockDim = dim3(unsigned(threads));
    cfg.dynamicSmemBytes = kSpSmemBytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    switch (c->sp_var) {
#define T3_SPV_CASE(V)                                                                                \
    case V:                                                                                           \
        T3_CK(cudaLaunchKernelEx(&cfg, t3_sp_kernel<V>, sin, sout, nblocks, static_cast<const uint32_t*>(c->d_sp), \
                                 passes, keys, mul, kp, int(pdl)));                                   \
        break;
        T3_SPV_LIST(T3_SPV_CASE)
#undef T3_SPV_CASE
        default:
            return T3DES_CU_ERR_ARG;
    }
    T3_CK(cudaGetLastError());
    ++c->launches;
    return T3DES_CU_OK;
}

int check_batch(t3des_cu_ctx* c, int dir, const void* in, const void* out, std::size_t len) {
    if (!c || (dir != T3DES_CU_ENCRYPT && dir != T3DES_CU_DECRYPT)) return T3DES_CU_ERR_ARG;
    if (len % 8) return T3DES_CU_ERR_LENGTH;
    if (len && (!in || !out)) return T3DES_CU_ERR_ARG;
    if (partial_overlap(in, out, len)) return T3DES_CU_ERR_OVERLAP;
    if (!c->have_schedule) return T3DES_CU_ERR_NO_SCHEDULE;
    return T3DES_CU_OK;
}

// Pipeline stage size for host batches below 64 MiB (pinned and pageable
// alike): enough stages that copies in, kernels and copies out overlap, but
// not so many that per-stage costs dominate (scripts/e2e_small_sweep.py,
// profiles/r1/e2e_small_r1l.txt: 1 MiB best in 2 stages, 4 MiB in 4, 16 MiB
// in 8-16).  0 = not a small batch (the large-batch rules apply).
std::size_t small_batch_stage(std::size_t len) {
    constexpr std::size_t KiB = 1024, MiB = KiB * KiB;
    if (len >= 64 * MiB) return 0;
    std::size_t s = len <= 512 * KiB ? len : len <= 2 * MiB ? len / 2 : len <= 8 * MiB ? len / 4 : len / 8;
    if (s > 8 * T3_TILE_BLOCKS) s -= s % (8 * T3_TILE_BLOCKS);
    return std::max<std::size_t>(s, 8);
}

}  // namespace

namespace t3b {

bool fault_at(std::size_t stage) {
    static const long k = [] {
        const char* e = std::getenv("T3DES_FAULT_AT_STAGE");
        return e ? std::atol(e) : -1L;
    }();
    return k >= 0 && stage == static_cast<std::size_t>(k);
}

int run_device(t3des_cu_ctx* c, int dir, const std::uint8_t* in, std::uint8_t* out, std::uint64_t nblocks,
               cudaStream_t s) {
    if (nblocks == 0) return T3DES_CU_OK;
    const std::uint64_t step = c->chunk_blocks ? c->chunk_blocks : nblocks;
    for (std::uint64_t off = 0; off < nblocks; off += step) {
        const std::uint64_t n = std::min(step, nblocks - off);
        const bool sp = c->variant == T3DES_CU_VARIANT_SPTABLE ||
                        (c->variant == T3DES_CU_VARIANT_AUTO && n <= T3DES_CU_AUTO_SMALL_BLOCKS);
        const int rc = sp ? launch_sptable(c, dir, in + 8 * off, out + 8 * off, n, s)
                          : launch_bitslice(c, dir, in + 8 * off, out + 8 * off, n, s);
        if (rc) return rc;
    }
    return T3DES_CU_OK;
}

int ensure_staging(t3des_cu_ctx* c, std::size_t bytes, int n) {
    bool ok = c->buf_bytes >= bytes;
    for (int i = 0; i < n && ok; ++i) ok = c->buf[i] != nullptr;
    if (ok) return T3DES_CU_OK;
    for (auto& b : c->buf) {
        if (b) cudaFree(b);
        b = nullptr;
    }
    c->buf_bytes = 0;
    for (int i = 0; i < n; ++i) T3_CK(cudaMalloc(&c->buf[i], bytes));
    c->buf_bytes = bytes;
    return T3DES_CU_OK;
}

SpanKind classify_span(const void* p) {
    SpanKind k;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        (void)cudaGetLastError();
        return k;
    }
    k.device_only = a.type == cudaMemoryTypeDevice;
    k.pinned = a.type == cudaMemoryTypeHost;
    if (k.pinned) k.mapped = a.devicePointer;
    return k;
}

// Pageable spans (hoststage.hpp): stage k goes through pinned slot k % R and
// stream st[k % R], R = c->host_slots.  A fill side (this thread, pool_in)
// and a drain side (c->drain, pool_out) run decoupled — see the loop below —
// so up to R - 1 stages are on the GPU while the host threads copy.  A
// pinned side (in or out) skips its host copy and DMAs straight from/to the
// span.
int ecb_host_staged(t3des_cu_ctx* c, int dir, const std::uint8_t* in, std::uint8_t* out, std::size_t len,
                    bool in_pinned, bool out_pinned) {
    const int R = c->host_slots;
    std::size_t S = c->pipe_explicit ? c->pipe_chunk : c->stage_bytes;  // t3des_cu_set_pipeline
    if (!c->pipe_explicit && small_batch_stage(len)) S = small_batch_stage(len);
    if (const char* e = std::getenv("T3DES_HOST_STAGE_MIB")) S = std::size_t(std::max(1, std::atoi(e))) << 20;
    S = std::min(S, len);
    if (S > 8 * T3_TILE_BLOCKS) S -= S % (8 * T3_TILE_BLOCKS);
    const t3b::NumaNode none;
    const t3b::NumaNode& node = c->numa_bind ? c->numa : none;
    if (c->hbuf_bytes < S) {
        for (int i = 0; i < t3des_cu_ctx::kHostSlots; ++i) {
            if (c->hev_live[i]) T3_CK(cudaEventSynchronize(c->hev[i]));
            t3b::host_free_on_node(c->hbuf[i], c->hbuf_bytes, c->hbuf_registered[i]);
            if (c->hdev[i]) cudaFree(c->hdev[i]);
            c->hbuf[i] = c->hdev[i] = nullptr;
        }
        c->hbuf_bytes = 0;
        for (int i = 0; i < R; ++i) {
            void* hp = nullptr;
            if (t3b::host_alloc_on_node(S, node, &hp, &c->hbuf_registered[i]) != 0) {
                for (int j = 0; j < i; ++j) {  // keep the ring all-or-nothing
                    t3b::host_free_on_node(c->hbuf[j], S, c->hbuf_registered[j]);
                    if (c->hdev[j]) cudaFree(c->hdev[j]);
                    c->hbuf[j] = c->hdev[j] = nullptr;
                }
                (void)cudaGetLastError();
                return T3DES_CU_ERR_CUDA;
            }
            c->hbuf[i] = static_cast<std::uint8_t*>(hp);
            T3_CK(cudaMalloc(&c->hdev[i], S));
            if (!c->hev[i]) T3_CK(cudaEventCreateWithFlags(&c->hev[i], cudaEventDisableTiming));
            c->hev_live[i] = false;
        }
        c->hbuf_bytes = S;
    }
    if (!c->pool_in) {
        int total = c->copy_threads;
        if (const char* e = std::getenv("T3DES_HOST_COPY_THREADS")) total = std::atoi(e);
        // measured on the 16-thread B200 hosts (scripts/pageable_ab.py,
        // profiles/r2/pageable_ab_r2k*.txt): 14 threads with 6 MiB stages and
        // cached stores into the slots are best
        if (total <= 0) total = std::clamp(t3b::available_cpus() * 7 / 8, 2, kMaxCopyThreads);
        // Copies out to the caller's buffer use streaming stores (no
        // read-for-ownership; the caller's data is not re-read by this
        // thread).  Copies into the pinned slots choose per batch (below).
        // Overrides for experiments: T3DES_HOST_NT_IN / T3DES_HOST_NT_OUT.
        auto flag = [](const char* n, bool d) { const char* e = std::getenv(n); return e ? std::atoi(e) != 0 : d; };
        int nin = (total + 1) / 2;
        if (const char* e = std::getenv("T3DES_HOST_IN_THREADS")) nin = std::clamp(std::atoi(e), 1, total - 1);  // experiments
        c->pool_in = new t3b::CopyPool(nin, node, flag("T3DES_HOST_NT_IN", true));
        c->pool_out = new t3b::CopyPool(std::max(1, total - nin), node, flag("T3DES_HOST_NT_OUT", true));
    }
    const std::size_t nst = (len + S - 1) / S;
    // One small stage between two pageable spans: copy in, run the SP-table
    // kernel zero-copy on the mapped pinned slot, copy out (no DMA setups).
    if (nst == 1 && !in_pinned && !out_pinned && !c->chunk_blocks &&
        (c->variant == T3DES_CU_VARIANT_AUTO || c->variant == T3DES_CU_VARIANT_SPTABLE)) {
        std::uint8_t* h = c->hbuf[0];
        void* d = nullptr;
        T3_CK(cudaHostGetDevicePointer(&d, h, 0));
        c->pool_in->start(h, in, len);
        c->pool_in->wait();
        int rc0 = launch_sptable(c, dir, static_cast<std::uint8_t*>(d), static_cast<std::uint8_t*>(d), len / 8, c->st[0]);
        if (!rc0 && cudaStreamSynchronize(c->st[0]) != cudaSuccess) rc0 = T3DES_CU_ERR_CUDA;
        if (rc0) {
            (void)cudaGetLastError();
            return rc0;
        }
        c->pool_out->start(out, h, len);
        c->pool_out->wait();
        return T3DES_CU_OK;
    }
    auto off = [&](std::size_t k) { return k * S; };
    auto cnt = [&](std::size_t k) { return std::min(S, len - k * S); };
    // pageable on both sides and at most 12 MiB: stages run zero-copy on their
    // mapped pinned slots (no DMA); above that the host copies and the kernel's
    // PCIe traffic contend and the DMA pipeline is as fast or faster
    // (scripts/zerocopy_big.py with ZC_PAGEABLE=1, profiles/r1/zerocopy_r1n.txt)
    std::size_t zc_max = kStagedZeroCopyMaxBytes;
    if (const char* e = std::getenv("T3DES_ZEROCOPY_MAX")) zc_max = std::strtoull(e, nullptr, 10);  // experiments
    const bool zc = !in_pinned && !out_pinned && len <= zc_max && !c->chunk_blocks &&
                    (c->variant == T3DES_CU_VARIANT_AUTO || c->variant == T3DES_CU_VARIANT_SPTABLE);
    // Slot-store policy of the fill side: batches of >= 256 MiB copy into
    // the slots with ordinary (cached) stores, so a slot is still in the
    // CPU's last-level cache when the H2D DMA reads it (DDIO) — 1 GiB 29.6
    // vs 27.0 GB/s; smaller batches use streaming stores — 16 MiB 17.9 vs
    // 12.9, 64 MiB 23.5 vs 19.1 — (profiles/r2/pageable_policy_r2t.txt;
    // 128 MiB is the crossover).  T3DES_HOST_NT_IN overrides.
    int in_streaming = len >= (std::size_t(256) << 20) ? 0 : 1;
    if (std::getenv("T3DES_HOST_NT_IN")) in_streaming = -1;  // the pool default set from the variable
    // Fill side (this thread) and drain side (c->drain) run decoupled over the
    // ring of R slots: the fill side copies stage k into slot k % R once the
    // drain side has released it, then enqueues H2D -> kernel -> D2H (or the
    // zero-copy kernel) and an event; the drain side waits for stage j's
    // event, copies it out of its slot and releases the slot.  Neither side
    // waits for the other's copy to finish unless the ring is full or empty
    // (the lock-step loop of round 1 ran both copies per step and waited for
    // the slower one).  Errors never return with a copy job in flight: each
    // side waits for its own copies, and the drain side is joined.
    std::mutex mu;
    std::condition_variable cv;
    std::size_t enqueued = 0, released = 0;
    int rc = T3DES_CU_OK, drain_rc = T3DES_CU_OK;
    bool stop = false;
    if (!c->drain) c->drain = new t3b::Worker();
    c->drain->run([&] {
        for (std::size_t j = 0; j < nst; ++j) {
            {
                std::unique_lock<std::mutex> l(mu);
                cv.wait(l, [&] { return stop || enqueued > j; });
                if (enqueued <= j) return;  // the fill side stopped early
            }
            int r = cudaEventSynchronize(c->hev[j % R]) == cudaSuccess ? T3DES_CU_OK : T3DES_CU_ERR_CUDA;
            if (!r && !out_pinned) {
                c->pool_out->start(out + off(j), c->hbuf[j % R], cnt(j));
                c->pool_out->wait();
            }
            std::lock_guard<std::mutex> l(mu);
            if (r) {
                drain_rc = r;
                stop = true;
                cv.notify_all();
                return;
            }
            released = j + 1;
            cv.notify_all();
        }
    });
    for (std::size_t k = 0; k < nst && !rc; ++k) {
        const int slot = int(k % R);
        {
            std::unique_lock<std::mutex> l(mu);
            cv.wait(l, [&] { return stop || k < std::size_t(R) || released + R > k; });
            if (stop) break;
        }
        if (!in_pinned) {  // the slot's last stage has been copied out (or DMA'd to a pinned out)
            c->pool_in->start(c->hbuf[slot], in + off(k), cnt(k), in_streaming);
            c->pool_in->wait();
        }
        cudaStream_t s = c->st[slot];
        const std::uint8_t* src = in_pinned ? in + off(k) : c->hbuf[slot];
        std::uint8_t* dst = out_pinned ? out + off(k) : c->hbuf[slot];
        const std::size_t n = cnt(k);
        if (zc) {  // the SP-table kernel on the mapped pinned slot
            void* d = nullptr;
            if (cudaHostGetDevicePointer(&d, c->hbuf[slot], 0) != cudaSuccess) rc = T3DES_CU_ERR_CUDA;
            if (!rc) rc = launch_sptable(c, dir, static_cast<std::uint8_t*>(d), static_cast<std::uint8_t*>(d), n / 8, s);
        } else {
            if (cudaMemcpyAsync(c->hdev[slot], src, n, cudaMemcpyHostToDevice, s) != cudaSuccess) rc = T3DES_CU_ERR_CUDA;
            if (!rc) rc = fault_at(k) ? T3DES_CU_ERR_CUDA : run_device(c, dir, c->hdev[slot], c->hdev[slot], n / 8, s);
            if (!rc && cudaMemcpyAsync(dst, c->hdev[slot], n, cudaMemcpyDeviceToHost, s) != cudaSuccess)
                rc = T3DES_CU_ERR_CUDA;
        }
        if (!rc && cudaEventRecord(c->hev[slot], s) != cudaSuccess) rc = T3DES_CU_ERR_CUDA;
        c->hev_live[slot] = !rc;
        std::lock_guard<std::mutex> l(mu);
        if (rc) {
            stop = true;
        } else {
            enqueued = k + 1;
        }
        cv.notify_all();
    }
    c->drain->wait();
    if (!rc) rc = drain_rc;
    for (int i = 0; i < R; ++i)
        if (cudaStreamSynchronize(c->st[i]) != cudaSuccess && !rc) rc = T3DES_CU_ERR_CUDA;
    if (rc) (void)cudaGetLastError();
    return rc;
}

}  // namespace t3b

using t3b::run_device;

extern "C" {

int t3des_cu_version(void) { return 1 * 10000 + 0 * 100 + 0; }

const char* t3des_cu_strerror(int code) {
    switch (code) {
        case T3DES_CU_OK: return "ok";
        case T3DES_CU_ERR_LENGTH: return "batch length is not a multiple of 8 bytes";
        case T3DES_CU_ERR_OVERLAP: return "partially overlapping buffers";
        case T3DES_CU_ERR_KEY: return "key must be 16, 32 or 48 hex characters";
        case T3DES_CU_ERR_ARG: return "invalid argument";
        case T3DES_CU_ERR_NO_DEVICE: return "no usable sm_100 CUDA device";
        case T3DES_CU_ERR_CUDA: return "CUDA runtime error";
        case T3DES_CU_ERR_NO_SCHEDULE: return "no key schedule installed";
        case T3DES_CU_ERR_PADDING: return "malformed PKCS#7 padding";
        case T3DES_CU_ERR_IO: return "stream read/write failure";
        case T3DES_CU_ERR_JIT: return "keyed kernel: NVRTC unavailable or compilation failed";
        default: return "unknown error";
    }
}

int t3des_cu_parse_hex_key(const char* hex, std::size_t len, std::uint64_t keys[3], int* option) {
    if (!hex || !keys) return T3DES_CU_ERR_ARG;
    const int opt = t3b::parse_hex_key(hex, len, keys);
    if (opt < 0) return T3DES_CU_ERR_KEY;
    if (option) *option = opt;
    return T3DES_CU_OK;
}

int t3des_cu_triple_schedule(const std::uint64_t keys[3], std::uint64_t sub48[48]) {
    if (!keys || !sub48) return T3DES_CU_ERR_ARG;
    t3b::triple_schedule(keys, sub48);
    return T3DES_CU_OK;
}

int t3des_cu_des_key_flags(std::uint64_t key) {
    return (t3b::has_odd_parity(key) ? T3DES_CU_KEY_ODD_PARITY : 0) | (t3b::is_weak_key(key) ? T3DES_CU_KEY_WEAK : 0) |
           (t3b::is_semiweak_key(key) ? T3DES_CU_KEY_SEMIWEAK : 0);
}

std::uint64_t t3des_cu_normalize_parity(std::uint64_t key) { return t3b::normalize_parity(key); }

int t3des_cu_device_count(int* count) {
    if (!count) return T3DES_CU_ERR_ARG;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        (void)cudaGetLastError();
        n = 0;
    }
    *count = n;
    return T3DES_CU_OK;
}

int t3des_cu_create(int device, t3des_cu_ctx** out) {
    if (!out) return T3DES_CU_ERR_ARG;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) {
        (void)cudaGetLastError();
        return T3DES_CU_ERR_NO_DEVICE;
    }
    cudaDeviceProp prop;
    T3_CK(cudaGetDeviceProperties(&prop, device));
    // built for sm_100a only: another 10.x part would fail every launch later
    if (prop.major != 10 || prop.minor != 0) return T3DES_CU_ERR_NO_DEVICE;
    DeviceScope scope(device);
    auto* c = new (std::nothrow) t3des_cu_ctx();
    if (!c) return T3DES_CU_ERR_ARG;
    c->device = device;
    c->sms = prop.multiProcessorCount;
    {
        char bus[32] = {};
        if (cudaDeviceGetPCIBusId(bus, sizeof bus, device) == cudaSuccess) c->numa = t3b::numa_node_of_pci(bus);
        (void)cudaGetLastError();
        if (const char* e = std::getenv("T3DES_HOST_SLOTS"))  // experiments: pageable ring depth
            c->host_slots = std::clamp(std::atoi(e), 2, t3des_cu_ctx::kHostSlots);
        // T3DES_NUMA=1: place single-device contexts too (multi-GPU contexts always are)
        if (const char* e = std::getenv("T3DES_NUMA")) c->numa_bind = std::atoi(e) == 1;
    }
    int rc = T3DES_CU_OK;
    do {
        int occ_ldg = 1;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c->bs_occ, t3_bs_tma_kernel<T3_OPT_DEFAULT_VALUE>, T3_BS_THREADS, 0) !=
                cudaSuccess ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_ldg, t3_bs_kernel<4, false>, T3_BS_THREADS, 0) !=
                cudaSuccess) {
            rc = T3DES_CU_ERR_CUDA;
            break;
        }
        // Tuning override (experiments only): SP-table code-generation mask.
        if (const char* e = std::getenv("T3DES_SP_VAR")) c->sp_var = std::atoi(e);
        if (!sp_kernel_fn(c->sp_var)) {
            rc = T3DES_CU_ERR_ARG;
            break;
        }
        bool attr_ok = true;
#define T3_SPV_ATTR(V)                                                                               \
    attr_ok = attr_ok && cudaFuncSetAttribute(t3_sp_kernel<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                              kSpSmemBytes) == cudaSuccess;
        T3_SPV_LIST(T3_SPV_ATTR)
#undef T3_SPV_ATTR
        if (!attr_ok ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c->sp_occ, sp_kernel_fn(c->sp_var), T3_SP_THREADS,
                                                          kSpSmemBytes) != cudaSuccess ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c->sp_occ_big, sp_kernel_fn(c->sp_var), T3_SP_THREADS_BIG,
                                                          kSpSmemBytes) != cudaSuccess) {
            rc = T3DES_CU_ERR_CUDA;
            break;
        }
        c->bs_occ = std::max(std::min(c->bs_occ, occ_ldg), 1);
        // Tuning override (experiments only): code-generation options of the
        // default bitsliced variant (T3_OPT_* mask among the compiled ones).
        if (const char* e = std::getenv("T3DES_BS_OPT")) c->bs_opt = std::atoi(e);
        // Tuning override (experiments only): grid size in CTAs per SM.
        if (const char* e = std::getenv("T3DES_BS_CTAS_PER_SM")) {
            const int v = std::atoi(e);
            if (v > 0) c->bs_ctas_per_sm = v;
        }
        c->sp_occ = std::max(c->sp_occ, 1);
        c->sp_occ_big = std::max(c->sp_occ_big, 1);
        std::uint32_t sp[8][64];
        t3b::build_sp_tables(sp);
        if (cudaMalloc(&c->d_sp, sizeof sp) != cudaSuccess ||
            cudaMemcpy(c->d_sp, sp, sizeof sp, cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMalloc(&c->d_acc, sizeof(unsigned long long)) != cudaSuccess) {
            rc = T3DES_CU_ERR_CUDA;
            break;
        }
        for (auto& s : c->st)
            if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) rc = T3DES_CU_ERR_CUDA;
        if (cudaStreamCreateWithFlags(&c->tail_st, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess)
            rc = T3DES_CU_ERR_CUDA;
    } while (false);
    if (rc) {
        (void)cudaGetLastError();
        t3des_cu_destroy(c);
        return rc;
    }
    *out = c;
    return T3DES_CU_OK;
}

int t3des_cu_destroy(t3des_cu_ctx* c) {
    if (!c) return T3DES_CU_ERR_ARG;
    {
        DeviceScope scope(c->device);
        for (auto& s : c->st)
            if (s) cudaStreamDestroy(s);
        if (c->tail_st) cudaStreamDestroy(c->tail_st);
        if (c->ev_fork) cudaEventDestroy(c->ev_fork);
        if (c->ev_join) cudaEventDestroy(c->ev_join);
        for (auto& b : c->buf)
            if (b) cudaFree(b);
        if (c->ubuf) cudaFree(c->ubuf);
        if (c->d_spk) cudaFree(c->d_spk);
        for (int i = 0; i < t3des_cu_ctx::kHostSlots; ++i) {
            t3b::host_free_on_node(c->hbuf[i], c->hbuf_bytes, c->hbuf_registered[i]);
            if (c->hdev[i]) cudaFree(c->hdev[i]);
            if (c->hev[i]) cudaEventDestroy(c->hev[i]);
        }
        delete c->pool_in;
        delete c->pool_out;
        delete c->drain;
        delete c->io_pool;
        if (c->d_sp) cudaFree(c->d_sp);
        if (c->d_acc) cudaFree(c->d_acc);
        (void)cudaGetLastError();
    }
    delete c;
    return T3DES_CU_OK;
}

int t3des_cu_set_schedule(t3des_cu_ctx* c, const std::uint64_t sub48[48]) {
    if (!c || !sub48) return T3DES_CU_ERR_ARG;
    // the same schedule again (the C++/Python batch APIs install it on every
    // call): nothing to rebuild, and no device synchronisation
    if (c->have_schedule && std::memcmp(c->sub48, sub48, sizeof c->sub48) == 0) return T3DES_CU_OK;
    c->have_schedule = false;  // until every table below is rebuilt
    c->keyed[0] = c->keyed[1] = nullptr;  // keyed modules are per key sequence
    c->rounds = 48;
    for (int dir = 0; dir < 2; ++dir) {
        std::uint64_t seq[48];
        t3b::key_sequence(sub48, dir == T3DES_CU_DECRYPT, seq);
        t3b::build_bitslice_table(seq, c->bs[dir]);
        t3b::SpKeys k;
        t3b::build_sp_keys(seq, k);
        std::memcpy(c->sp[dir].k, k.k, sizeof k.k);
        std::memcpy(c->sp[dir].k2, k.k2, sizeof k.k2);
        // K1 = K2 or K2 = K3: the EDE collapses to single DES (16 rounds)
        std::uint64_t seq16[48] = {};
        if (t3b::collapsed_sequence(sub48, dir == T3DES_CU_DECRYPT, seq16) == 16) {
            c->rounds = 16;
            t3b::build_bitslice_table(seq16, c->bs16[dir], 16);
            t3b::build_sp_keys(seq16, k);
            std::memcpy(c->sp16[dir].k, k.k, sizeof k.k);
            std::memcpy(c->sp16[dir].k2, k.k2, sizeof k.k2);
        }
    }
    // device copy of the SP-table kernel's round keys (sp[enc], sp[dec],
    // sp16[enc], sp16[dec]) for the masks that stage them in shared memory;
    // the shipped mask takes them as a kernel parameter (by value, like the
    // bitsliced tables), so a new schedule never waits for launches in flight
    if (!(c->sp_var & T3_SPV_KEYPARAM)) {
        DeviceScope scope(c->device);
        if (!c->d_spk) {
            T3_CK(cudaMalloc(&c->d_spk, 4 * sizeof(T3SpKeyParam)));
        } else {
            T3_CK(cudaDeviceSynchronize());  // no launch may still read the old keys
        }
        const T3SpKeyParam keys[4] = {c->sp[0], c->sp[1], c->sp16[0], c->sp16[1]};
        T3_CK(cudaMemcpy(c->d_spk, keys, sizeof keys, cudaMemcpyHostToDevice));
    }
    std::memcpy(c->sub48, sub48, sizeof c->sub48);
    c->have_schedule = true;
    return T3DES_CU_OK;
}

int t3des_cu_set_variant(t3des_cu_ctx* c, int variant) {
    if (!c || variant < T3DES_CU_VARIANT_BITSLICE || variant > T3DES_CU_VARIANT_KEYED)
        return T3DES_CU_ERR_ARG;
    c->variant = variant;
    return T3DES_CU_OK;
}

int t3des_cu_set_launch(t3des_cu_ctx* c, std::size_t chunk_blocks, int work_group) {
    if (!c || work_group < 0 || work_group > 1024 || (work_group % 32) != 0) return T3DES_CU_ERR_ARG;
    if (work_group > T3_BS_THREADS && c->variant != T3DES_CU_VARIANT_SPTABLE && c->variant != T3DES_CU_VARIANT_AUTO)
        return T3DES_CU_ERR_ARG;
    c->chunk_blocks = chunk_blocks;
    c->work_group = work_group;
    return T3DES_CU_OK;
}

int t3des_cu_ecb_device(t3des_cu_ctx* c, int dir, const void* din, void* dout, std::size_t len,
                        void* stream) {
    const int rc = check_batch(c, dir, din, dout, len);
    if (rc) return rc;
    if (!len) return T3DES_CU_OK;
    DeviceScope scope(c->device);
    const auto* in = static_cast<const std::uint8_t*>(din);
    auto* out = static_cast<std::uint8_t*>(dout);
    auto s = static_cast<cudaStream_t>(stream);
    if (((reinterpret_cast<std::uintptr_t>(in) | reinterpret_cast<std::uintptr_t>(out)) & 7u) == 0)
        return run_device(c, dir, in, out, len / 8, s);
    // Spans that are not 8-byte aligned (the kernels load whole blocks):
    // bounce through an aligned device buffer, chunk by chunk, on the
    // caller's stream; synchronous, so the buffer is free on return.
    constexpr std::size_t kChunk = std::size_t(16) << 20;
    if (!c->ubuf) T3_CK(cudaMalloc(&c->ubuf, kChunk));
    // errors still wait for the queued copies: none may write `out` after return
    int rc2 = T3DES_CU_OK;
    for (std::size_t off = 0; off < len && !rc2; off += kChunk) {
        const std::size_t n = std::min(kChunk, len - off);
        if (cudaMemcpyAsync(c->ubuf, in + off, n, cudaMemcpyDeviceToDevice, s) != cudaSuccess) rc2 = T3DES_CU_ERR_CUDA;
        if (!rc2) rc2 = run_device(c, dir, c->ubuf, c->ubuf, n / 8, s);
        if (!rc2 && cudaMemcpyAsync(out + off, c->ubuf, n, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
            rc2 = T3DES_CU_ERR_CUDA;
    }
    if (cudaStreamSynchronize(s) != cudaSuccess && !rc2) rc2 = T3DES_CU_ERR_CUDA;
    if (rc2) (void)cudaGetLastError();
    return rc2;
}

int t3des_cu_ecb_host(t3des_cu_ctx* c, int dir, const std::uint8_t* in, std::uint8_t* out,
                      std::size_t len) {
    int rc = check_batch(c, dir, in, out, len);
    if (rc) return rc;
    if (!len) return T3DES_CU_OK;
    DeviceScope scope(c->device);
    const t3b::SpanKind ki = t3b::classify_span(in), ko = in == out ? ki : t3b::classify_span(out);
    if (ki.device_only || ko.device_only) return T3DES_CU_ERR_ARG;  // use t3des_cu_ecb_device
    if (!ki.pinned || !ko.pinned) return t3b::ecb_host_staged(c, dir, in, out, len, ki.pinned, ko.pinned);
    // Pinned batches up to 64 MiB: the SP-table kernel reads and writes the
    // mapped host pages directly over PCIe — no DMA setup in either direction,
    // and the kernel (~158 GB/s) stays far ahead of the link.  Larger batches
    // reach more of the link through the copy engines (DMA pipeline below).
    std::size_t zc_max = kZeroCopyMaxBytes;
    if (const char* e = std::getenv("T3DES_ZEROCOPY_MAX")) zc_max = std::strtoull(e, nullptr, 10);  // experiments
    if (len <= zc_max && ki.mapped && ko.mapped && !c->chunk_blocks &&
        ((reinterpret_cast<std::uintptr_t>(ki.mapped) | reinterpret_cast<std::uintptr_t>(ko.mapped)) & 7u) == 0 &&
        (c->variant == T3DES_CU_VARIANT_AUTO || c->variant == T3DES_CU_VARIANT_SPTABLE)) {
        cudaStream_t s = c->st[0];
        if (int rc2 = launch_sptable(c, dir, static_cast<const std::uint8_t*>(ki.mapped),
                                     static_cast<std::uint8_t*>(ko.mapped), len / 8, s))
            return rc2;
        T3_CK(cudaStreamSynchronize(s));
        return T3DES_CU_OK;
    }
    // Stage size: as set, or adapted to the batch — about 8 stages, between
    // 8 and 32 MiB (scripts/e2e_size_sweep.py: 32-64 MiB batches gain ~10-30%
    // from 8 MiB stages, >= 256 MiB batches prefer 32 MiB), whole tiles.
    std::size_t chunk = c->pipe_chunk;
    if (!c->pipe_explicit) {
        chunk = std::min(chunk, std::max(std::size_t(8) << 20, len / 8));
        chunk -= chunk % (8 * T3_TILE_BLOCKS);
        if (const std::size_t s = small_batch_stage(len)) chunk = s;
    }
    chunk = std::min(len, chunk);
    const int ns = c->pipe_streams;
    rc = t3b::ensure_staging(c, chunk, ns);
    if (rc) return rc;
    // Stage k: H2D, kernel, D2H on stream k % ns (in-order per stream, so a
    // stream's buffer is free again when its next stage starts); stages on
    // different streams overlap copies in both directions with kernels.
    // Ramp (large batches, default shape): the first stages grow from
    // kRampBytes to `chunk` and the last ones shrink back, so the pipeline
    // fills and drains in small steps instead of one full stage each way.
    std::size_t ramp = 0;
    if (!c->pipe_explicit && len >= (std::size_t(64) << 20)) ramp = kRampBytes;
    if (const char* e = std::getenv("T3DES_RAMP_KIB")) ramp = std::size_t(std::atoi(e)) << 10;  // experiments
    auto stage_bytes = [&](std::size_t k, std::size_t left) {
        std::size_t n = std::min(chunk, left);
        if (ramp && ramp < chunk) {
            if (k < 16) n = std::min(n, ramp << k);
            if (left < 2 * chunk && left > ramp) {  // tail: halve towards the ramp size
                std::size_t h = (left / 2 + 8 * T3_TILE_BLOCKS - 1) / (8 * T3_TILE_BLOCKS) * (8 * T3_TILE_BLOCKS);
                n = std::min(n, std::max(h, ramp));
            }
        }
        return n;
    };
    // An error stops issuing but still waits for every stream: no queued D2H
    // may write the caller's `out` after this call has returned.
    std::size_t k = 0;
    for (std::size_t off = 0, n = 0; off < len && !rc; off += n, ++k) {
        n = stage_bytes(k, len - off);
        cudaStream_t s = c->st[k % ns];
        std::uint8_t* b = c->buf[k % ns];
        if (cudaMemcpyAsync(b, in + off, n, cudaMemcpyHostToDevice, s) != cudaSuccess) rc = T3DES_CU_ERR_CUDA;
        if (!rc) rc = fault_at(k) ? T3DES_CU_ERR_CUDA : run_device(c, dir, b, b, n / 8, s);
        if (!rc && cudaMemcpyAsync(out + off, b, n, cudaMemcpyDeviceToHost, s) != cudaSuccess) rc = T3DES_CU_ERR_CUDA;
    }
    for (int i = 0; i < ns; ++i)
        if (cudaStreamSynchronize(c->st[i]) != cudaSuccess && !rc) rc = T3DES_CU_ERR_CUDA;
    if (rc) (void)cudaGetLastError();
    return rc;
}

int t3des_cu_set_pipeline(t3des_cu_ctx* c, std::size_t chunk_bytes, int streams) {
    if (!c || streams < 1 || streams > t3des_cu_ctx::kMaxStreams || chunk_bytes < 8 || chunk_bytes % 8)
        return T3DES_CU_ERR_ARG;
    c->pipe_chunk = chunk_bytes;
    c->pipe_streams = streams;
    c->pipe_explicit = true;
    return T3DES_CU_OK;
}

int t3des_cu_host_alloc(std::size_t bytes, void** out) {
    if (!out) return T3DES_CU_ERR_ARG;
    *out = nullptr;
    T3_CK(cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocPortable));
    return T3DES_CU_OK;
}

int t3des_cu_host_free(void* p) {
    if (p) T3_CK(cudaFreeHost(p));
    return T3DES_CU_OK;
}

int t3des_cu_host_register(void* p, std::size_t bytes) {
    if (!p || !bytes) return T3DES_CU_ERR_ARG;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n <= 0) {
        (void)cudaGetLastError();
        return T3DES_CU_ERR_NO_DEVICE;
    }
    // portable: pinned for every context; mapped: the zero-copy small-batch path applies too
    T3_CK(cudaHostRegister(p, bytes, cudaHostRegisterPortable | cudaHostRegisterMapped));
    return T3DES_CU_OK;
}

int t3des_cu_host_unregister(void* p) {
    if (!p) return T3DES_CU_ERR_ARG;
    T3_CK(cudaHostUnregister(p));
    return T3DES_CU_OK;
}

int t3des_cu_fill_splitmix(t3des_cu_ctx* c, void* dptr, std::uint64_t first_block, std::size_t nblocks,
                           std::uint64_t seed, void* stream) {
    if (!c || (nblocks && !dptr)) return T3DES_CU_ERR_ARG;
    if (!nblocks) return T3DES_CU_OK;
    DeviceScope scope(c->device);
    const unsigned grid = unsigned(std::min<std::uint64_t>((nblocks + 255) / 256, std::uint64_t(c->sms) * 8));
    t3_fill_splitmix_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<uint2*>(dptr), first_block, nblocks, seed);
    T3_CK(cudaGetLastError());
    return T3DES_CU_OK;
}

int t3des_cu_checksum(t3des_cu_ctx* c, const void* dptr, std::uint64_t first_block, std::size_t nblocks,
                      std::uint64_t* out, void* stream) {
    if (!c || !out || (nblocks && !dptr)) return T3DES_CU_ERR_ARG;
    DeviceScope scope(c->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    unsigned long long h = 0;
    T3_CK(cudaMemsetAsync(c->d_acc, 0, sizeof h, s));
    if (nblocks) {
        const unsigned grid =
            unsigned(std::min<std::uint64_t>((nblocks + 255) / 256, std::uint64_t(c->sms) * 8));
        t3_checksum_kernel<<<grid, 256, 0, s>>>(static_cast<const unsigned long long*>(dptr), first_block,
                                                nblocks, c->d_acc);
        T3_CK(cudaGetLastError());
    }
    T3_CK(cudaMemcpyAsync(&h, c->d_acc, sizeof h, cudaMemcpyDeviceToHost, s));
    T3_CK(cudaStreamSynchronize(s));
    *out = h;
    return T3DES_CU_OK;
}

int t3des_cu_launch_count(t3des_cu_ctx* c, std::uint64_t* out) {
    if (!c || !out) return T3DES_CU_ERR_ARG;
    *out = c->launches;
    return T3DES_CU_OK;
}

}  // extern "C"
