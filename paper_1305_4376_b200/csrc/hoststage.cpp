// Host copy pool for the pageable staging path (hoststage.hpp).
#include "hoststage.hpp"

#include <cuda_runtime.h>
#include <pthread.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <cctype>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#if defined(__x86_64__)
#include <emmintrin.h>
#endif

namespace t3b {

namespace {

// memcpy with non-temporal (streaming) stores: the staged bytes are not read
// again by this thread, and skipping the read-for-ownership of each
// destination line saves a quarter of the host memory traffic of a copy.
void stream_copy(char* d, const char* s, std::size_t n, bool nt) {
#if defined(__x86_64__)
    if (nt && n >= 4096) {
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
    (void)nt;
    std::memcpy(d, s, n);
}

bool env_flag(const char* name, bool dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) != 0 : dflt;
}

constexpr int kMpolDefault = 0, kMpolPreferred = 1;  // linux/mempolicy.h
constexpr unsigned long kMaxNode = 1024;                            // bits in the masks below

std::string sysfs_root() {
    const char* e = std::getenv("T3DES_SYSFS_ROOT");
    return e ? e : "/sys";
}

bool read_line(const std::string& path, std::string& out) {
    std::FILE* f = std::fopen(path.c_str(), "r");
    if (!f) return false;
    char buf[4096];
    const bool ok = std::fgets(buf, sizeof buf, f) != nullptr;
    std::fclose(f);
    if (!ok) return false;
    out = buf;
    while (!out.empty() && std::isspace(static_cast<unsigned char>(out.back()))) out.pop_back();
    return true;
}

int count_nodes(const std::string& root) {
    int n = 0;
    for (int k = 0; k < 1024; ++k) {
        std::string tmp;
        if (read_line(root + "/devices/system/node/node" + std::to_string(k) + "/cpulist", tmp)) ++n;
        else if (k > 64 && n) break;
    }
    return n;
}

}  // namespace

int available_cpus() {
    cpu_set_t set;
    CPU_ZERO(&set);
    if (sched_getaffinity(0, sizeof set, &set) == 0) return std::max(1, CPU_COUNT(&set));
    return std::max(1, int(std::thread::hardware_concurrency()));
}

std::vector<int> parse_cpulist(const char* s) {
    std::vector<int> cpus;
    if (!s) return cpus;
    const char* p = s;
    while (*p) {
        char* end = nullptr;
        const long a = std::strtol(p, &end, 10);
        if (end == p || a < 0) return {};
        long b = a;
        p = end;
        if (*p == '-') {
            ++p;
            b = std::strtol(p, &end, 10);
            if (end == p || b < a) return {};
            p = end;
        }
        for (long c = a; c <= b && c < 65536; ++c) cpus.push_back(int(c));
        if (*p == ',') ++p;
        else if (*p && !std::isspace(static_cast<unsigned char>(*p))) return {};
        else if (*p) break;
    }
    return cpus;
}

NumaNode numa_node_of_pci(const char* bus_id) {
    NumaNode n;
    if (const char* e = std::getenv("T3DES_NUMA"); e && std::atoi(e) == 0) return n;
    if (!bus_id) return n;
    std::string id(bus_id);
    for (auto& ch : id) ch = char(std::tolower(static_cast<unsigned char>(ch)));
    const std::string root = sysfs_root();
    std::string v;
    if (!read_line(root + "/bus/pci/devices/" + id + "/numa_node", v)) return n;
    const int node = std::atoi(v.c_str());
    if (node < 0 || count_nodes(root) < 2) return n;
    if (!read_line(root + "/devices/system/node/node" + std::to_string(node) + "/cpulist", v)) return n;
    cpu_set_t allowed;
    CPU_ZERO(&allowed);
    const bool have_mask = sched_getaffinity(0, sizeof allowed, &allowed) == 0;
    for (int c : parse_cpulist(v.c_str()))
        if (!have_mask || (c < CPU_SETSIZE && CPU_ISSET(c, &allowed))) n.cpus.push_back(c);
    if (!n.cpus.empty()) n.node = node;
    return n;
}

NumaBind::NumaBind(const NumaNode& n) {
    if (n.node < 0 || n.cpus.empty()) return;
    static_assert(sizeof(cpu_set_t) <= sizeof old_cpus_, "cpu_set_t storage");
    auto* old = reinterpret_cast<cpu_set_t*>(old_cpus_);
    if (pthread_getaffinity_np(pthread_self(), sizeof(cpu_set_t), old) == 0) {
        cpu_set_t set;
        CPU_ZERO(&set);
        for (int c : n.cpus)
            if (c < CPU_SETSIZE) CPU_SET(c, &set);
        cpus_bound_ = pthread_setaffinity_np(pthread_self(), sizeof set, &set) == 0;
    }
    unsigned long mask[kMaxNode / (8 * sizeof(unsigned long))] = {};
    if (n.node < int(kMaxNode)) {
        mask[n.node / (8 * sizeof(unsigned long))] |= 1ul << (n.node % (8 * sizeof(unsigned long)));
        if (syscall(SYS_get_mempolicy, &old_mode_, old_mask_, kMaxNode, nullptr, 0ul) == 0)
            policy_set_ = syscall(SYS_set_mempolicy, kMpolPreferred, mask, kMaxNode) == 0;
    }
}

NumaBind::~NumaBind() {
    if (cpus_bound_) pthread_setaffinity_np(pthread_self(), sizeof(cpu_set_t), reinterpret_cast<cpu_set_t*>(old_cpus_));
    if (policy_set_) {
        if (old_mode_ == kMpolDefault) syscall(SYS_set_mempolicy, kMpolDefault, nullptr, 0ul);
        else syscall(SYS_set_mempolicy, old_mode_, old_mask_, kMaxNode);
    }
}

int host_alloc_on_node(std::size_t bytes, const NumaNode& n, void** out, bool* registered) {
    *out = nullptr;
    *registered = false;
    if (n.node < 0 || n.node >= int(kMaxNode)) {
        const cudaError_t e = cudaMallocHost(out, bytes);
        return int(e);
    }
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p == MAP_FAILED) return int(cudaErrorMemoryAllocation);
    unsigned long mask[kMaxNode / (8 * sizeof(unsigned long))] = {};
    mask[n.node / (8 * sizeof(unsigned long))] |= 1ul << (n.node % (8 * sizeof(unsigned long)));
    // preferred, not bound: a full node falls back to another instead of failing
    (void)syscall(SYS_mbind, p, bytes, kMpolPreferred, mask, kMaxNode, 0u);
    std::memset(p, 0, bytes);                                         // fault the pages in on that node
    const cudaError_t e = cudaHostRegister(p, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        munmap(p, bytes);
        return int(e);
    }
    *out = p;
    *registered = true;
    return 0;
}

void host_free_on_node(void* p, std::size_t bytes, bool registered) {
    if (!p) return;
    if (registered) {
        cudaHostUnregister(p);
        munmap(p, bytes);
    } else {
        cudaFreeHost(p);
    }
}

CopyPool::CopyPool(int nthreads, NumaNode node, bool streaming)
    : n_(std::max(1, nthreads)),
      node_(std::move(node)),
      nt_allowed_(env_flag("T3DES_HOST_NT_COPY", true)),
      nt_(streaming && nt_allowed_) {
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

void CopyPool::start(void* dst, const void* src, std::size_t bytes, int streaming) {
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
        job_nt_ = streaming < 0 ? nt_ : (streaming > 0 && nt_allowed_);
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
    NumaBind bind(node_);  // for the thread's lifetime
    std::uint64_t seen = 0;
    for (;;) {
        char* d;
        const char* s;
        std::size_t b;
        bool nt;
        {
            std::unique_lock<std::mutex> l(m_);
            cv_.wait(l, [&] { return stop_ || gen_ != seen; });
            if (stop_) return;
            seen = gen_;
            d = dst_;
            s = src_;
            b = bytes_;
            nt = job_nt_;
        }
        // piece i of n_, page-aligned so that threads never share a page
        const std::size_t per = ((b + n_ - 1) / n_ + 4095) & ~std::size_t(4095);
        const std::size_t lo = std::min(b, per * std::size_t(i)), hi = std::min(b, lo + per);
        if (hi > lo) stream_copy(d + lo, s + lo, hi - lo, nt);
        {
            std::lock_guard<std::mutex> l(m_);
            if (--left_ == 0) done_cv_.notify_all();
        }
    }
}

Worker::Worker() {
    th_ = std::thread([this] {
        std::unique_lock<std::mutex> l(m_);
        for (;;) {
            cv_.wait(l, [&] { return stop_ || static_cast<bool>(job_); });
            if (stop_) return;
            auto job = std::move(job_);
            job_ = nullptr;
            l.unlock();
            job();
            l.lock();
            busy_ = false;
            done_cv_.notify_all();
        }
    });
}

Worker::~Worker() {
    {
        std::lock_guard<std::mutex> l(m_);
        stop_ = true;
    }
    cv_.notify_all();
    th_.join();
}

void Worker::run(std::function<void()> job) {
    {
        std::lock_guard<std::mutex> l(m_);
        job_ = std::move(job);
        busy_ = true;
    }
    cv_.notify_all();
}

void Worker::wait() {
    std::unique_lock<std::mutex> l(m_);
    done_cv_.wait(l, [&] { return !busy_; });
}

PartPool::PartPool(int n) : n_(std::max(1, n)) {
    th_.reserve(n_ - 1);
    for (int i = 1; i < n_; ++i) th_.emplace_back([this, i] { loop(i); });
}

PartPool::~PartPool() {
    {
        std::lock_guard<std::mutex> l(m_);
        stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
}

void PartPool::loop(int part) {
    std::uint64_t seen = 0;
    for (;;) {
        const std::function<void(int, int)>* fn;
        {
            std::unique_lock<std::mutex> l(m_);
            cv_.wait(l, [&] { return stop_ || gen_ != seen; });
            if (stop_) return;
            seen = gen_;
            fn = fn_;
        }
        (*fn)(part, n_);
        std::lock_guard<std::mutex> l(m_);
        if (--left_ == 0) done_cv_.notify_all();
    }
}

void PartPool::run(const std::function<void(int, int)>& fn) {
    {
        std::lock_guard<std::mutex> l(m_);
        fn_ = &fn;
        left_ = n_ - 1;
        ++gen_;
    }
    cv_.notify_all();
    fn(0, n_);
    std::unique_lock<std::mutex> l(m_);
    done_cv_.wait(l, [&] { return left_ == 0; });
}

}  // namespace t3b
