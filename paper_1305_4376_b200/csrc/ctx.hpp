// Private: the engine context behind the C ABI's opaque t3des_cu_ctx and
// the internal entry points shared by capi.cu and stream.cu.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "t3des_core.cuh"

#ifndef T3_OPT_DEFAULT_VALUE
#define T3_OPT_DEFAULT_VALUE 5  // T3_OPT_DFMA | T3_OPT_WFMA: measured best (scripts/opt_sweep.sh)
#endif
#include "t3des_cu.h"

#include "hoststage.hpp"

struct t3des_cu_ctx {
    int device = 0;
    int sms = 0;
    int bs_occ = 1;           // resident CTAs per SM (occupancy) of the bitsliced kernel
    int bs_ctas_per_sm = 64;  // grid size of the bitsliced kernel, in CTAs per SM
    int bs_opt = T3_OPT_DEFAULT_VALUE;  // T3_OPT_* mask of the default bitsliced variant
    int sp_occ = 1;      // resident SP-table CTAs per SM at T3_SP_THREADS
    int sp_occ_big = 1;  // ... at T3_SP_THREADS_BIG
    int sp_var = T3_SPV_DEFAULT;  // T3_SPV_* mask of the SP-table kernel
    bool have_schedule = false;
    std::uint64_t sub48[48] = {};  // the installed schedule (pass-major)
    int variant = T3DES_CU_VARIANT_AUTO;
    std::size_t chunk_blocks = 0;
    int work_group = 0;
    T3BsTable bs[2];       // 48-round tables, encrypt / decrypt
    T3SpKeyParam sp[2];
    int rounds = 48;       // 16 when the schedule collapses to single DES
    T3BsTable bs16[2];     // collapsed (16-round) tables
    T3SpKeyParam sp16[2];
    std::uint32_t* d_sp = nullptr;  // 8x64 fused S/P table (2 KiB)
    unsigned long long* d_acc = nullptr;
    static constexpr int kMaxStreams = 8;
    cudaStream_t st[kMaxStreams] = {};
    std::uint8_t* buf[kMaxStreams] = {};
    std::size_t buf_bytes = 0;
    std::size_t pipe_chunk = std::size_t(32) << 20;  // bytes per pipeline stage (upper bound)
    int pipe_streams = 3;
    bool pipe_explicit = false;  // set by t3des_cu_set_pipeline; else stages adapt to the batch
    // pageable-span staging (t3des_cu_ecb_host): pinned ring, one event per
    // slot (the slot's last GPU use), and two host copy pools (in / out)
    static constexpr int kHostSlots = 8;  // ring capacity; host_slots of them are used
    std::uint8_t* hbuf[kHostSlots] = {};
    std::uint8_t* hdev[kHostSlots] = {};
    std::size_t hbuf_bytes = 0;
    cudaEvent_t hev[kHostSlots] = {};
    bool hev_live[kHostSlots] = {};
    bool hbuf_registered[kHostSlots] = {};  // allocated by host_alloc_on_node (mmap + register)
    t3b::CopyPool* pool_in = nullptr;
    t3b::CopyPool* pool_out = nullptr;
    t3b::Worker* drain = nullptr;  // drain side of the pageable ring (copies out)
    t3b::PartPool* io_pool = nullptr;  // parallel pread/pwrite of the stream fd entry
    int host_slots = 4;            // pinned ring slots in use (<= kHostSlots)
    std::size_t stage_bytes = std::size_t(6) << 20;  // pageable stage size (scripts/pageable_ab.py)
    int copy_threads = 0;                            // total host copy threads (0 = auto)
    t3b::NumaNode numa;      // the device's NUMA node (node -1: unknown / single-node host)
    bool numa_bind = false;  // place pinned staging and copy threads on `numa` (multi-GPU contexts)
    std::uint32_t* d_spk = nullptr;  // device copies of sp[2], sp16[2] (48 x 8 words each)
    std::uint8_t* ubuf = nullptr;  // bounce buffer for device spans that are not 8-byte aligned
    std::uint64_t launches = 0;
    cudaStream_t tail_st = nullptr;             // side stream for the partial tile (AUTO)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    const void* keyed[2] = {};  // VARIANT_KEYED: the schedule's loaded module per direction (keyed.cpp)
};

namespace t3b {

// Makes `dev` the current device and restores the caller's on scope exit.
// Every entry point that allocates, launches or synchronises on a context's
// resources opens one (streams, events and buffers belong to c->device).
struct DeviceScope {
    int prev = -1;
    explicit DeviceScope(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        cudaSetDevice(dev);
    }
    ~DeviceScope() {
        if (prev >= 0) cudaSetDevice(prev);
    }
    DeviceScope(const DeviceScope&) = delete;
    DeviceScope& operator=(const DeviceScope&) = delete;
};

// In and out spans overlap without being the same span (the reference's
// InputLengthError case, dispatch.cpp:99-104).
inline bool partial_overlap(const void* a, const void* b, std::size_t len) {
    const auto* x = static_cast<const std::uint8_t*>(a);
    const auto* y = static_cast<const std::uint8_t*>(b);
    return x != y && y < x + len && y + len > x;
}

// host copy threads of the pageable staging path (in + out pools)
constexpr int kMaxCopyThreads = 14;

// Test hook: T3DES_FAULT_AT_STAGE=k makes stage (chunk) k of the host
// pipelines and the stream path fail as a launch would, so their error paths
// can be tested (tests/test_gpu_parity.py, tests/test_streams.py).
bool fault_at(std::size_t stage);

// Transform nblocks device blocks on stream s (in may equal out), honouring
// the context's variant and launch shaping.  Returns a T3DES_CU_* status.
int run_device(t3des_cu_ctx* c, int dir, const std::uint8_t* in, std::uint8_t* out, std::uint64_t nblocks,
               cudaStream_t s);

// Make sure the first n staging buffers hold at least `bytes` each.
int ensure_staging(t3des_cu_ctx* c, std::size_t bytes, int n);

// VARIANT_KEYED (keyed.cpp): load the keyed module of c's schedule for `dir`
// (compiling it on first use of that key sequence), and launch it over
// `ntiles` full warp tiles of 16-byte aligned spans.
int keyed_prepare(t3des_cu_ctx* c, int dir, double* seconds);
int keyed_launch(t3des_cu_ctx* c, int dir, const std::uint8_t* in, std::uint8_t* out, std::uint64_t ntiles,
                 cudaStream_t s);

// What a host-span pointer is, from one attribute query: device-only memory
// (an error for the host entry points), page-locked host memory (DMA-able
// without bouncing), and the device address under which page-locked memory
// is mapped (null if it is not mapped for the current device).
struct SpanKind {
    bool device_only = false, pinned = false;
    void* mapped = nullptr;
};
SpanKind classify_span(const void* p);

// t3des_cu_ecb_host for spans that are not both pinned: pinned ring staging
// with host copy threads (hoststage.hpp).
int ecb_host_staged(t3des_cu_ctx* c, int dir, const std::uint8_t* in, std::uint8_t* out, std::size_t len,
                    bool in_pinned, bool out_pinned);

}  // namespace t3b
