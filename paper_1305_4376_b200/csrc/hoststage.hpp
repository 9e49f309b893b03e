// Private: host-side staging of pageable buffers for t3des_cu_ecb_host.
//
// The reference's callers hand encrypt_batch/decrypt_batch plain
// std::span<uint8_t> memory (dispatch.hpp:64-69) -- pageable, not pinned.
// cudaMemcpyAsync from pageable memory is synchronous and bounces through the
// driver's own staging (7 GB/s end to end on the B200 boxes, against 45 GB/s
// from pinned memory), so the engine stages pageable spans itself: host
// threads copy each stage into a pinned ring slot while the GPU transforms
// the previous ones and other threads copy finished stages out.
#pragma once
#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace t3b {

// NUMA placement of one device's host-side work (multi-GPU end
// to end): the CPUs and memory node local to the GPU's PCIe root.  node < 0:
// unknown, or a single-node host (nothing to place).
struct NumaNode {
    int node = -1;
    std::vector<int> cpus;  // the node's CPUs that this process may run on
};

// CPUs this process may run on (its affinity mask; e.g. a bench rank bound
// to its GPU's node), at least 1.
int available_cpus();

// "0-3,8,10-11" -> {0,1,2,3,8,10,11}; malformed input -> {}.
std::vector<int> parse_cpulist(const char* s);

// The NUMA node of a PCI device ("0000:1B:00.0", any case) from sysfs
// (/sys/bus/pci/devices/<id>/numa_node, /sys/devices/system/node/node<k>/
// cpulist; root overridable with T3DES_SYSFS_ROOT for tests).  Returns
// node -1 on single-node hosts, when sysfs has no answer, or with
// T3DES_NUMA=0.
NumaNode numa_node_of_pci(const char* bus_id);

// Binds the calling thread to a node's CPUs and makes that node its
// preferred memory node; restores both on destruction.  No-op for node < 0.
class NumaBind {
public:
    explicit NumaBind(const NumaNode& n);
    ~NumaBind();
    NumaBind(const NumaBind&) = delete;
    NumaBind& operator=(const NumaBind&) = delete;
    bool active() const { return cpus_bound_; }

private:
    bool cpus_bound_ = false, policy_set_ = false;
    int old_mode_ = 0;
    unsigned long old_mask_[16] = {};
    unsigned char old_cpus_[128] = {};  // cpu_set_t storage
};

// Page-locked host memory on a NUMA node: mmap + mbind(MPOL_PREFERRED) +
// first touch + cudaHostRegister (mapped, portable), so the pages are where the
// device's DMA and copy threads are.  node < 0 falls back to cudaMallocHost.
// Returns 0 or a cudaError_t value.
int host_alloc_on_node(std::size_t bytes, const NumaNode& n, void** out, bool* registered);
void host_free_on_node(void* p, std::size_t bytes, bool registered);

// A fixed set of threads that split one memcpy at a time between them.
// start() hands out a job and returns; wait() blocks until it is done.
class CopyPool {
public:
    // threads are bound to `node`'s CPUs when it is known; `streaming`: copy
    // with non-temporal stores (the destination is not read again soon)
    explicit CopyPool(int nthreads, NumaNode node = {}, bool streaming = true);
    ~CopyPool();
    CopyPool(const CopyPool&) = delete;
    CopyPool& operator=(const CopyPool&) = delete;
    // copies of at most kInlineBytes run on the calling thread
    static constexpr std::size_t kInlineBytes = std::size_t(64) << 10;
    // streaming: 1 / 0 = this job with / without streaming stores, -1 = the
    // pool's default
    void start(void* dst, const void* src, std::size_t bytes, int streaming = -1);
    void wait();
    int threads() const { return n_; }

private:
    void run(int i);
    const int n_;
    const NumaNode node_;
    const bool nt_allowed_;  // T3DES_HOST_NT_COPY (experiments) can switch streaming stores off
    const bool nt_;          // the default for jobs
    bool job_nt_ = false;
    std::mutex m_;
    std::condition_variable cv_, done_cv_;
    std::uint64_t gen_ = 0;
    int left_ = 0;
    bool stop_ = false;
    char* dst_ = nullptr;
    const char* src_ = nullptr;
    std::size_t bytes_ = 0;
    std::vector<std::thread> th_;
};

// n persistent threads that run one data-parallel job at a time: run(fn)
// calls fn(part, n) for part = 0..n-1 (part 0 on the calling thread) and
// returns when all parts are done.  The stream path's parallel pread/pwrite
// of regular files uses it.
class PartPool {
public:
    explicit PartPool(int n);
    ~PartPool();
    PartPool(const PartPool&) = delete;
    PartPool& operator=(const PartPool&) = delete;
    void run(const std::function<void(int, int)>& fn);
    int size() const { return n_; }

private:
    void loop(int part);
    const int n_;
    std::mutex m_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(int, int)>* fn_ = nullptr;
    std::uint64_t gen_ = 0;
    int left_ = 0;
    bool stop_ = false;
    std::vector<std::thread> th_;
};

// One persistent thread that runs one job at a time: run() hands it a job
// and returns; wait() blocks until the job has finished.  The pageable
// staging path's drain side (copies out of the ring) runs on it, decoupled
// from the fill side on the calling thread.
class Worker {
public:
    Worker();
    ~Worker();
    Worker(const Worker&) = delete;
    Worker& operator=(const Worker&) = delete;
    void run(std::function<void()> job);
    void wait();

private:
    std::mutex m_;
    std::condition_variable cv_, done_cv_;
    std::function<void()> job_;
    bool busy_ = false, stop_ = false;
    std::thread th_;
};

}  // namespace t3b
