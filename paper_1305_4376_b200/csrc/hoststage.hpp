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
#include <mutex>
#include <thread>
#include <vector>

namespace t3b {

// A fixed set of threads that split one memcpy at a time between them.
// start() hands out a job and returns; wait() blocks until it is done.
class CopyPool {
public:
    explicit CopyPool(int nthreads);
    ~CopyPool();
    CopyPool(const CopyPool&) = delete;
    CopyPool& operator=(const CopyPool&) = delete;
    // copies of at most kInlineBytes run on the calling thread
    static constexpr std::size_t kInlineBytes = std::size_t(64) << 10;
    void start(void* dst, const void* src, std::size_t bytes);
    void wait();
    int threads() const { return n_; }

private:
    void run(int i);
    const int n_;
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

}  // namespace t3b
