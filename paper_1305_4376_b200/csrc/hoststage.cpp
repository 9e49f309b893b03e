// Host copy pool for the pageable staging path (hoststage.hpp).
#include "hoststage.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#if defined(__x86_64__)
#include <emmintrin.h>
#endif

namespace t3b {

namespace {

// memcpy with non-temporal (streaming) stores: the staged bytes are not read
// again by this thread, and skipping the read-for-ownership of each
// destination line saves a quarter of the host memory traffic of a copy.
void stream_copy(char* d, const char* s, std::size_t n) {
#if defined(__x86_64__)
    static const bool enabled = [] {
        const char* e = std::getenv("T3DES_HOST_NT_COPY");
        return !e || std::atoi(e) != 0;
    }();
    if (enabled && n >= 4096) {
        const std::size_t head = (16 - (reinterpret_cast<std::uintptr_t>(d) & 15)) & 15;
        std::memcpy(d, s, head);
        d += head;
        s += head;
        n -= head;
        const std::size_t body = n & ~std::size_t(63);
        for (std::size_t i = 0; i < body; i += 64) {
            const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i));
            const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 16));
            const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 32));
            const __m128i e = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 48));
            _mm_stream_si128(reinterpret_cast<__m128i*>(d + i), a);
            _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 16), b);
            _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 32), c);
            _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 48), e);
        }
        std::memcpy(d + body, s + body, n - body);
        _mm_sfence();  // streaming stores are weakly ordered: publish before signalling
        return;
    }
#endif
    std::memcpy(d, s, n);
}

}  // namespace

CopyPool::CopyPool(int nthreads) : n_(std::max(1, nthreads)) {
    th_.reserve(n_);
    for (int i = 0; i < n_; ++i) th_.emplace_back([this, i] { run(i); });
}

CopyPool::~CopyPool() {
    {
        std::lock_guard<std::mutex> l(m_);
        stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
}

void CopyPool::start(void* dst, const void* src, std::size_t bytes) {
    if (bytes <= kInlineBytes) {  // waking the pool costs more than the copy
        std::memcpy(dst, src, bytes);
        std::lock_guard<std::mutex> l(m_);
        left_ = 0;
        return;
    }
    {
        std::lock_guard<std::mutex> l(m_);
        dst_ = static_cast<char*>(dst);
        src_ = static_cast<const char*>(src);
        bytes_ = bytes;
        left_ = n_;
        ++gen_;
    }
    cv_.notify_all();
}

void CopyPool::wait() {
    std::unique_lock<std::mutex> l(m_);
    done_cv_.wait(l, [&] { return left_ == 0; });
}

void CopyPool::run(int i) {
    std::uint64_t seen = 0;
    for (;;) {
        char* d;
        const char* s;
        std::size_t b;
        {
            std::unique_lock<std::mutex> l(m_);
            cv_.wait(l, [&] { return stop_ || gen_ != seen; });
            if (stop_) return;
            seen = gen_;
            d = dst_;
            s = src_;
            b = bytes_;
        }
        // piece i of n_, page-aligned so that threads never share a page
        const std::size_t per = ((b + n_ - 1) / n_ + 4095) & ~std::size_t(4095);
        const std::size_t lo = std::min(b, per * std::size_t(i)), hi = std::min(b, lo + per);
        if (hi > lo) stream_copy(d + lo, s + lo, hi - lo);
        {
            std::lock_guard<std::mutex> l(m_);
            if (--left_ == 0) done_cv_.notify_all();
        }
    }
}

}  // namespace t3b
