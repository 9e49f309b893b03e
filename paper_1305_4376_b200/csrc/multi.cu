// Multi-GPU entries of the C ABI (include/t3des_cu.h): block-range sharding
// of host batches over devices (t3des_cu_ecb_multi, t3des_cu_ecb_workers —
// the GPU reading of DispatchConfig.workers) and of device-resident batches
// over NVLink peers (t3des_cu_ecb_multi_device).  No collective: ECB blocks
// are independent (reference SPEC.md:221-223), so each shard is a separate
// single-device transform.
#include <cuda_runtime.h>

#include <algorithm>
#include <iterator>
#include <cstdlib>
#include <mutex>
#include <thread>
#include <vector>

#include "ctx.hpp"
#include "t3des_cu.h"

using t3b::DeviceScope;
using t3b::kMaxCopyThreads;
using t3b::partial_overlap;
using t3b::run_device;

namespace {

// Contexts of the multi-GPU entries (t3des_cu_ecb_multi*), kept across
// calls: creating one costs device queries, table uploads, streams, and its
// staging buffers are allocated on first use, all of which a per-call
// context paid again every call.  A context is handed to one caller at a
// time (calls into a context are serialised).
std::mutex g_pool_mu;
std::vector<t3des_cu_ctx*> g_pool;  // idle contexts, any device

int pool_acquire(int device, t3des_cu_ctx** out) {
    {
        // most recently released first: a caller repeating one shape gets the
        // contexts whose staging rings that shape already sized (handing out
        // the least recently used instead rotated through every pooled
        // context, and each one reallocated its ring for the new shard size:
        // ~30 ms per call, scripts/workers_probe.cpp)
        std::lock_guard<std::mutex> lk(g_pool_mu);
        for (auto it = g_pool.rbegin(); it != g_pool.rend(); ++it)
            if ((*it)->device == device) {
                *out = *it;
                g_pool.erase(std::next(it).base());
                return T3DES_CU_OK;
            }
    }
    return t3des_cu_create(device, out);
}

void pool_release(t3des_cu_ctx* c, bool healthy) {
    if (!c) return;
    if (!healthy) {  // after a CUDA error: do not hand the context out again
        t3des_cu_destroy(c);
        return;
    }
    std::lock_guard<std::mutex> lk(g_pool_mu);
    g_pool.push_back(c);
}

// Block-range cuts of t3des_cu_ecb_multi_device.  With the payload resident
// on `home`, every remote shard crosses the home GPU's NVLink ports twice
// (peer copy out and back), while the home GPU's own shard needs no copy.  So
// the home shard gets the share h that balances its kernel time against the
// remote side's bound: h / r_k = (1 - h) / min(r_link, (n_remote) * r_k), with
// r_k = 396 GB/s (the kernel, bench) and r_link = 770 GB/s per direction (the
// measured B200 peer-copy rate, B200_PROFILING.md) — h = 0.34 for 3+ GPUs, 0.5
// for 2.  Equal shards (t3des_cu_shard_range) when the home GPU is
// not among the devices exactly once, or with T3DES_CU_MULTI_STAGE_ALL.
// T3DES_MULTI_HOME_SHARE overrides h (tests, tuning).  Cuts are whole tiles.
std::vector<std::uint64_t> multi_device_cuts(const int* devices, int ndev, int home, std::uint64_t nblocks,
                                             int flags) {
    std::vector<std::uint64_t> cut(ndev + 1, nblocks);
    int home_idx = -1, homes = 0;
    for (int g = 0; g < ndev; ++g)
        if (devices[g] == home) {
            if (home_idx < 0) home_idx = g;
            ++homes;
        }
    double h = -1.0;
    if (const char* e = std::getenv("T3DES_MULTI_HOME_SHARE")) h = std::atof(e);
    else if (homes == 1 && ndev > 1 && !(flags & T3DES_CU_MULTI_STAGE_ALL)) {
        constexpr double kKernelGBps = 396.0, kLinkGBps = 770.0;
        h = kKernelGBps / (kKernelGBps + std::min(kLinkGBps, (ndev - 1) * kKernelGBps));
    }
    if (home_idx < 0 || ndev == 1 || !(h > 0.0 && h < 1.0)) {
        for (int g = 0; g < ndev; ++g) {
            std::uint64_t f = 0, c = 0;
            t3des_cu_shard_range(nblocks, ndev, g, &f, &c);
            cut[g] = f;
        }
        return cut;
    }
    const double rest = (1.0 - h) / (ndev - 1);
    double acc = 0.0;
    for (int g = 0; g < ndev; ++g) {
        const std::uint64_t b = std::uint64_t(acc * double(nblocks));
        cut[g] = g == 0 ? 0 : std::min(nblocks, b - b % T3_TILE_BLOCKS);
        acc += g == home_idx ? h : rest;
    }
    for (int g = 1; g <= ndev; ++g) cut[g] = std::max(cut[g], cut[g - 1]);  // monotone
    return cut;
}

}  // namespace

extern "C" {

int t3des_cu_shard_range(std::uint64_t nblocks, int ndev, int g, std::uint64_t* first, std::uint64_t* count) {
    if (ndev <= 0 || g < 0 || g >= ndev || !first || !count) return T3DES_CU_ERR_ARG;
    auto cut = [&](int k) -> std::uint64_t {
        if (k >= ndev) return nblocks;
        // 128-bit product: nblocks * k may exceed 2^64 for huge inputs
        const unsigned __int128 p = static_cast<unsigned __int128>(nblocks) * static_cast<unsigned>(k);
        std::uint64_t b = static_cast<std::uint64_t>(p / static_cast<unsigned>(ndev));
        return b - b % T3_TILE_BLOCKS;
    };
    *first = cut(g);
    *count = cut(g + 1) - *first;
    return T3DES_CU_OK;
}

int t3des_cu_ecb_multi(const int* devices, int ndev, const std::uint64_t sub48[48], int dir,
                       const std::uint8_t* in, std::uint8_t* out, std::size_t len) {
    if (!devices || ndev <= 0 || !sub48 || (dir != 0 && dir != 1)) return T3DES_CU_ERR_ARG;
    if (len % 8) return T3DES_CU_ERR_LENGTH;
    if (len && (!in || !out)) return T3DES_CU_ERR_ARG;
    if (partial_overlap(in, out, len)) return T3DES_CU_ERR_OVERLAP;
    if (!len) return T3DES_CU_OK;
    const std::uint64_t nblocks = len / 8;
    // contexts first (pooled), so that each shard's host threads can be sized
    // by how many shards share its device's NUMA node
    std::vector<t3des_cu_ctx*> ctx(ndev, nullptr);
    int rc = T3DES_CU_OK;
    for (int g = 0; g < ndev && !rc; ++g) rc = pool_acquire(devices[g], &ctx[g]);
    if (rc) {
        for (auto* c : ctx) pool_release(c, true);
        return rc;
    }
    const int hw = t3b::available_cpus();
    std::vector<int> rcs(ndev, T3DES_CU_OK);
    std::vector<std::thread> workers;
    for (int g = 0; g < ndev; ++g) {
        t3des_cu_ctx* c = ctx[g];
        c->numa_bind = true;  // pinned ring + copy threads on the device's node (a no-op where unknown)
        if (!c->pool_in) {    // pageable spans: the host's copy threads are shared by the shards
            int same = 0;
            for (auto* o : ctx) same += o->numa.node == c->numa.node;
            const int cpus = c->numa.node >= 0 ? int(c->numa.cpus.size()) : hw;
            c->copy_threads = std::clamp(cpus / std::max(same, 1), 2, kMaxCopyThreads);
        }
        workers.emplace_back([&, g, c] {
            std::uint64_t b0 = 0, cnt = 0;
            t3des_cu_shard_range(nblocks, ndev, g, &b0, &cnt);
            if (!cnt) return;
            t3b::NumaBind bind(c->numa);  // this shard's submitting thread next to its GPU
            int r = t3des_cu_set_schedule(c, sub48);
            if (!r) r = t3des_cu_ecb_host(c, dir, in + 8 * b0, out + 8 * b0, 8 * cnt);
            rcs[g] = r;
        });
    }
    for (auto& w : workers) w.join();
    for (int g = 0; g < ndev; ++g) {
        pool_release(ctx[g], rcs[g] == T3DES_CU_OK || rcs[g] == T3DES_CU_ERR_ARG);
        if (rcs[g] && !rc) rc = rcs[g];
    }
    return rc;
}

int t3des_cu_ecb_workers(unsigned workers, int first_device, const std::uint64_t sub48[48], int dir,
                         const std::uint8_t* in, std::uint8_t* out, std::size_t len) {
    if (!sub48 || (dir != 0 && dir != 1) || workers > 1024) return T3DES_CU_ERR_ARG;
    if (len % 8) return T3DES_CU_ERR_LENGTH;
    if (len && (!in || !out)) return T3DES_CU_ERR_ARG;
    if (partial_overlap(in, out, len)) return T3DES_CU_ERR_OVERLAP;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n <= 0) {
        (void)cudaGetLastError();
        return T3DES_CU_ERR_NO_DEVICE;
    }
    if (first_device < 0 || first_device >= n) return T3DES_CU_ERR_NO_DEVICE;
    if (!len) return T3DES_CU_OK;
    // at most one shard per visible GPU: a reference caller sizes `workers`
    // for CPU threads, and several contexts on one GPU only contend for its
    // PCIe link and the host's copy threads (2 shards on one B200: 4.2 vs
    // 2.7 ms for 64 MiB; 8 of them cost 0.6 s of context creation on first
    // use; scripts/workers_probe.cpp).  t3des_cu_ecb_multi still takes any
    // device list, repeated devices included.
    const int w = workers == 0 ? 1 : int(std::min<unsigned>(workers, unsigned(n)));
    if (w == 1) {
        t3des_cu_ctx* c = nullptr;
        int rc = pool_acquire(first_device, &c);
        if (!rc && !c->pool_in) {
            c->numa_bind = true;
            if (c->numa.node >= 0) c->copy_threads = std::clamp(int(c->numa.cpus.size()) * 7 / 8, 2, kMaxCopyThreads);
        }
        if (!rc) rc = t3des_cu_set_schedule(c, sub48);
        if (!rc) rc = t3des_cu_ecb_host(c, dir, in, out, len);
        pool_release(c, rc == T3DES_CU_OK || rc == T3DES_CU_ERR_ARG);
        return rc;
    }
    std::vector<int> devs(w);
    for (int g = 0; g < w; ++g) devs[g] = (first_device + g) % n;
    return t3des_cu_ecb_multi(devs.data(), w, sub48, dir, in, out, len);
}

int t3des_cu_ecb_multi_device(const int* devices, int ndev, const std::uint64_t sub48[48], int dir,
                              int home, const void* din, void* dout, std::size_t len, int flags) {
    if (!devices || ndev <= 0 || !sub48 || (dir != 0 && dir != 1)) return T3DES_CU_ERR_ARG;
    if (len % 8) return T3DES_CU_ERR_LENGTH;
    if (len && (!din || !dout)) return T3DES_CU_ERR_ARG;
    if (partial_overlap(din, dout, len)) return T3DES_CU_ERR_OVERLAP;
    if (!len) return T3DES_CU_OK;
    const std::uint64_t nblocks = len / 8;
    const auto* in = static_cast<const std::uint8_t*>(din);
    auto* out = static_cast<std::uint8_t*>(dout);
    const bool aligned = ((reinterpret_cast<std::uintptr_t>(in) | reinterpret_cast<std::uintptr_t>(out)) & 7u) == 0;
    std::vector<t3des_cu_ctx*> ctx(ndev, nullptr);
    int rc = T3DES_CU_OK;
    // Issue every shard asynchronously on its device, then wait.  A remote
    // shard runs peer-direct where the devices can map each other's memory
    // (below), else — or with T3DES_CU_MULTI_COPY — as a chunk pipeline
    // over kStreams streams and staging
    // buffers of its context: chunk k = peer copy in -> kernel -> peer copy
    // out on stream k % kStreams, so chunk k's copy in overlaps chunk k-1's
    // kernel and chunk k-2's copy out (NVLink both directions + SMs busy).
    constexpr int kStreams = 3;
    constexpr std::uint64_t kTileBytes = 8 * T3_TILE_BLOCKS;
    std::uint64_t chunk_override = 0;
    if (const char* e = std::getenv("T3DES_MULTI_CHUNK_BYTES")) chunk_override = std::strtoull(e, nullptr, 10);
    const std::vector<std::uint64_t> cut = multi_device_cuts(devices, ndev, home, nblocks, flags);
    for (int g = 0; g < ndev && !rc; ++g) {
        const std::uint64_t first = cut[g], count = cut[g + 1] - cut[g];
        if (!count) continue;
        rc = pool_acquire(devices[g], &ctx[g]);
        if (!rc) rc = t3des_cu_set_schedule(ctx[g], sub48);
        if (rc) break;
        t3des_cu_ctx* c = ctx[g];
        DeviceScope scope(devices[g]);
        const std::uint64_t bytes = 8 * count;
        if (devices[g] == home && !(flags & T3DES_CU_MULTI_STAGE_ALL) && aligned) {
            rc = run_device(c, dir, in + 8 * first, out + 8 * first, count, c->st[0]);
            continue;
        }
        bool peer = false;
        if (devices[g] != home) {
            int can = 0;
            if (cudaDeviceCanAccessPeer(&can, devices[g], home) == cudaSuccess && can) {
                const cudaError_t e = cudaDeviceEnablePeerAccess(home, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) rc = T3DES_CU_ERR_CUDA;
                (void)cudaGetLastError();
                peer = !rc;
            }
        }
        // Peer-direct (NVLink 5 / NVSwitch): the shard's kernel runs on its
        // device straight on the home GPU's buffers — loads and stores cross
        // NVLink inside the kernel, so transfer and compute overlap tile by
        // tile with no staging copies.  Plain 128-bit loads (the LDG variant):
        // the TMA variant's bulk copies are kept to local memory.  Unmeasured
        // on hardware (one GPU per box this round); T3DES_CU_MULTI_COPY
        // selects the copy pipeline below instead.
        if (peer && aligned && !(flags & (T3DES_CU_MULTI_COPY | T3DES_CU_MULTI_STAGE_ALL))) {
            const int v = c->variant;
            c->variant = T3DES_CU_VARIANT_BITSLICE_LDG;
            rc = run_device(c, dir, in + 8 * first, out + 8 * first, count, c->st[0]);
            c->variant = v;
            continue;
        }
        // chunk: about 1/8 of the shard, 8..256 MiB, whole warp tiles
        std::uint64_t chunk =
            std::clamp<std::uint64_t>(bytes / 8, std::uint64_t(8) << 20, std::uint64_t(256) << 20);
        chunk -= chunk % kTileBytes;
        if (chunk_override) chunk = std::max<std::uint64_t>(8, chunk_override - chunk_override % 8);  // tests
        chunk = std::min(chunk, bytes);
        if (!rc) rc = t3b::ensure_staging(c, chunk, kStreams);
        std::uint64_t k = 0;
        for (std::uint64_t off = 0; off < bytes && !rc; off += chunk, ++k) {
            const std::uint64_t n = std::min(chunk, bytes - off);
            cudaStream_t s = c->st[k % kStreams];
            std::uint8_t* b = c->buf[k % kStreams];
            if (cudaMemcpyPeerAsync(b, devices[g], in + 8 * first + off, home, n, s) != cudaSuccess)
                rc = T3DES_CU_ERR_CUDA;
            if (!rc) rc = run_device(c, dir, b, b, n / 8, s);
            if (!rc && cudaMemcpyPeerAsync(out + 8 * first + off, home, b, devices[g], n, s) != cudaSuccess)
                rc = T3DES_CU_ERR_CUDA;
        }
    }
    for (int g = 0; g < ndev; ++g) {
        if (!ctx[g]) continue;
        DeviceScope scope(devices[g]);
        for (int i = 0; i < kStreams; ++i)
            if (cudaStreamSynchronize(ctx[g]->st[i]) != cudaSuccess && !rc) rc = T3DES_CU_ERR_CUDA;
        pool_release(ctx[g], rc == T3DES_CU_OK || rc == T3DES_CU_ERR_ARG);
    }
    (void)cudaGetLastError();
    return rc;
}

int t3des_cu_multi_device_shards(const int* devices, int ndev, int home, std::uint64_t nblocks, int flags,
                                 std::uint64_t* first, std::uint64_t* count) {
    if (!devices || ndev <= 0 || !first || !count) return T3DES_CU_ERR_ARG;
    const std::vector<std::uint64_t> cut = multi_device_cuts(devices, ndev, home, nblocks, flags);
    for (int g = 0; g < ndev; ++g) {
        first[g] = cut[g];
        count[g] = cut[g + 1] - cut[g];
    }
    return T3DES_CU_OK;
}

}  // extern "C"
