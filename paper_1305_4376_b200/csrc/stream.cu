// Pipelined chunked streams over the CUDA engine (see stream.hpp), and the
// file-descriptor C-ABI entry t3des_cu_stream_fd.
#include <cuda_runtime.h>
#include <errno.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>

#include <chrono>
#include <cstring>
#include <deque>
#include <vector>

#include "ctx.hpp"
#include "stream.hpp"
#include "t3des_cu.h"

namespace t3b {
namespace {

using Clock = std::chrono::steady_clock;

double since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

constexpr int kSlots = 3;

// Pinned host ring for the stream pipeline.
struct PinnedRing {
    std::uint8_t* p[kSlots] = {};
    explicit PinnedRing(std::size_t bytes) {
        for (auto& x : p)
            if (cudaHostAlloc(reinterpret_cast<void**>(&x), bytes, cudaHostAllocDefault) != cudaSuccess) {
                (void)cudaGetLastError();
                x = nullptr;
            }
    }
    ~PinnedRing() {
        for (auto* x : p)
            if (x) cudaFreeHost(x);
    }
    bool ok() const { return p[0] && p[1] && p[2]; }
};

struct Slot {
    int idx;
    std::size_t n;  // bytes in the slot (after padding)
    bool last;
};

// Fill dst with up to n bytes (short only at end of stream).
std::size_t read_full(ByteSource& src, std::uint8_t* dst, std::size_t n) {
    std::size_t got = 0;
    while (got < n) {
        const std::size_t r = src.read(dst + got, n - got);
        if (r == 0) break;
        got += r;
    }
    return got;
}

}  // namespace

void pkcs7_pad_bytes(std::uint8_t* data, std::size_t len, std::size_t* out_len) {
    const std::uint8_t pad = static_cast<std::uint8_t>(8 - len % 8);
    std::memset(data + len, pad, pad);
    *out_len = len + pad;
}

std::size_t pkcs7_unpad_len(const std::uint8_t* data, std::size_t len) {
    if (len == 0 || len % 8)
        throw StreamFailure(StreamFailure::Padding, "PKCS#7 data length must be a positive multiple of 8");
    const std::uint8_t pad = data[len - 1];
    if (pad < 1 || pad > 8) throw StreamFailure(StreamFailure::Padding, "bad PKCS#7 pad value");
    for (std::size_t i = len - pad; i < len; ++i)
        if (data[i] != pad) throw StreamFailure(StreamFailure::Padding, "inconsistent PKCS#7 padding");
    return len - pad;
}

StreamStats run_stream(t3des_cu_ctx* c, int dir, ByteSource& src, ByteSink& dst, std::size_t chunk_blocks,
                       bool pkcs7, std::size_t io_blocks, bool copy_only) {
    DeviceScope scope(c->device);  // the ring, staging and streams live on the context's device
    StreamStats st;
    const std::size_t logical = chunk_blocks * 8;  // the reference's chunk
    if (io_blocks < chunk_blocks || io_blocks % chunk_blocks) io_blocks = chunk_blocks;
    const std::size_t chunk = io_blocks * 8;  // I/O + transform granularity
    const bool enc = dir == T3DES_CU_ENCRYPT;
    PinnedRing ring(chunk + 8);
    if (!ring.ok()) throw StreamFailure(StreamFailure::Cuda, "pinned staging allocation failed", 0, T3DES_CU_ERR_CUDA);
    if (int rc = copy_only ? T3DES_CU_OK : ensure_staging(c, chunk + 8, kSlots))
        throw StreamFailure(StreamFailure::Cuda, t3des_cu_strerror(rc), 0, rc);

    std::deque<Slot> inflight;
    auto complete = [&](const Slot& s) {
        auto t0 = Clock::now();
        if (cudaStreamSynchronize(c->st[s.idx]) != cudaSuccess) {
            (void)cudaGetLastError();
            throw StreamFailure(StreamFailure::Cuda, "CUDA error in stream chunk", 0, T3DES_CU_ERR_CUDA);
        }
        st.compute_seconds += since(t0);
        std::size_t n = s.n;
        if (!enc && pkcs7 && s.last) {
            try {
                n = pkcs7_unpad_len(ring.p[s.idx], s.n);
            } catch (const StreamFailure&) {
                // the reference writes every chunk before the last one, whose
                // padding is bad: with I/O coarser than its chunks, write the
                // leading logical chunks of this slot first
                const std::size_t head = s.n ? (s.n - 1) / logical * logical : 0;
                if (head) dst.write(ring.p[s.idx], head);
                st.bytes_out += head;
                throw;
            }
        }
        if (n) {
            t0 = Clock::now();
            try {
                dst.write(ring.p[s.idx], n);
            } catch (const StreamFailure&) {
                throw;
            } catch (const std::exception&) {
                throw StreamFailure(StreamFailure::Io, "write failure", st.bytes_out);
            }
            st.io_seconds += since(t0);
            st.bytes_out += n;
        }
    };
    auto drain = [&](std::size_t keep) {
        while (inflight.size() > keep) {
            Slot s = inflight.front();
            inflight.pop_front();
            complete(s);
        }
    };
    auto fail_after_drain = [&](const StreamFailure& f) {
        drain(0);  // the reference has written every earlier chunk when it throws
        throw f;
    };
    auto timed_read = [&](int slot) -> std::size_t {
        auto t0 = Clock::now();
        std::size_t got;
        try {
            got = read_full(src, ring.p[slot], chunk);
        } catch (const StreamFailure&) {
            throw;
        } catch (const std::exception&) {
            throw StreamFailure(StreamFailure::Io, "read failure", st.bytes_in);
        }
        st.io_seconds += since(t0);
        st.bytes_in += got;
        return got;
    };

    int k = 0;
    std::size_t got = 0;
    try {
        got = timed_read(0);
    } catch (const StreamFailure& f) {
        fail_after_drain(f);
    }
    for (;;) {
        const int slot = k % kSlots;
        const bool first = k == 0;
        if (got == 0 && !(first && enc && pkcs7)) break;
        // read ahead into the next slot (once it is free) to learn whether
        // this chunk is the last one
        std::size_t next_got = 0;
        const int nslot = (k + 1) % kSlots;
        if (got == chunk) {
            drain(kSlots - 2);
            try {
                next_got = timed_read(nslot);
            } catch (const StreamFailure& f) {
                fail_after_drain(f);
            }
        }
        const bool last = got < chunk || next_got == 0;
        std::size_t n = got;
        if (enc) {
            if (pkcs7 && last) {
                pkcs7_pad_bytes(ring.p[slot], got, &n);
            } else if (n % 8) {
                fail_after_drain(StreamFailure(StreamFailure::Length,
                                               "input length is not a multiple of 8 bytes (use PKCS#7 padding "
                                               "for arbitrary lengths)"));
            }
        } else if (n % 8) {
            const StreamFailure f(StreamFailure::Length, "ciphertext length not a multiple of 8");
            if (!pkcs7) fail_after_drain(f);
            // PKCS#7: the reference holds each decrypted chunk back until the
            // next one is read, so the chunk before this one is never written
            drain(1);
            if (!inflight.empty()) {
                (void)cudaStreamSynchronize(c->st[inflight.front().idx]);
                (void)cudaGetLastError();
                inflight.clear();
            }
            throw f;
        }
        if (n && copy_only) {  // NoOpCopy: the slot is written out as read
            inflight.push_back(Slot{slot, n, last});
            ++st.chunks;
        } else if (n) {
            auto t0 = Clock::now();
            cudaStream_t s = c->st[slot];
            std::uint8_t* d = c->buf[slot];
            int rc = cudaMemcpyAsync(d, ring.p[slot], n, cudaMemcpyHostToDevice, s) == cudaSuccess ? 0
                                                                                                  : T3DES_CU_ERR_CUDA;
            if (!rc) rc = fault_at(std::size_t(k)) ? T3DES_CU_ERR_CUDA : run_device(c, dir, d, d, n / 8, s);
            if (!rc && cudaMemcpyAsync(ring.p[slot], d, n, cudaMemcpyDeviceToHost, s) != cudaSuccess)
                rc = T3DES_CU_ERR_CUDA;
            if (rc) {
                (void)cudaGetLastError();
                fail_after_drain(StreamFailure(StreamFailure::Cuda, t3des_cu_strerror(rc), 0, rc));
            }
            st.compute_seconds += since(t0);
            inflight.push_back(Slot{slot, n, last});
            ++st.chunks;
        }
        if (last) break;
        got = next_got;
        ++k;
    }
    drain(0);
    if (!enc && pkcs7 && st.bytes_in == 0)
        throw StreamFailure(StreamFailure::Padding, "empty ciphertext cannot carry PKCS#7 padding");
    if (chunk != logical)  // report the reference's chunk count
        st.chunks = st.bytes_in ? (st.bytes_in + logical - 1) / logical : (enc && pkcs7 ? 1 : 0);
    auto t0 = Clock::now();
    dst.flush();
    st.io_seconds += since(t0);
    return st;
}

}  // namespace t3b

namespace {

// Regular files are read and written with pread/pwrite split over a
// PartPool (page-cache copies are per-thread memcpy-bound: one thread
// read()+write()s a tmpfs file at ~2.7 GB/s); pipes, sockets and O_APPEND
// descriptors keep plain sequential read()/write().  The descriptor offsets
// are advanced as sequential I/O would leave them.
bool regular_fd(int fd, bool for_write, std::uint64_t* size, std::uint64_t* pos) {
    struct stat sb;
    if (fstat(fd, &sb) != 0 || !S_ISREG(sb.st_mode)) return false;
    if (for_write && (fcntl(fd, F_GETFL) & O_APPEND)) return false;
    const off_t p = lseek(fd, 0, SEEK_CUR);
    if (p < 0) return false;
    *size = static_cast<std::uint64_t>(sb.st_size);
    *pos = static_cast<std::uint64_t>(p);
    return true;
}

// [lo, hi) of part `i` of `n` over `bytes`, page-aligned cuts
void part_range(std::size_t bytes, int i, int n, std::size_t* lo, std::size_t* hi) {
    const std::size_t per = ((bytes + n - 1) / n + 4095) & ~std::size_t(4095);
    *lo = std::min(bytes, per * std::size_t(i));
    *hi = std::min(bytes, *lo + per);
}

struct FdSource : t3b::ByteSource {
    int fd;
    t3b::PartPool* pool;
    bool par = false;
    std::uint64_t size = 0, pos = 0;
    FdSource(int f, t3b::PartPool* p) : fd(f), pool(p) { par = pool && regular_fd(fd, false, &size, &pos); }
    ~FdSource() override {
        if (par) (void)lseek(fd, static_cast<off_t>(pos), SEEK_SET);
    }
    std::size_t read(std::uint8_t* dst, std::size_t n) override {
        if (!par || pos >= size || n < (std::size_t(1) << 20)) {
            for (;;) {
                const ssize_t r = par ? ::pread(fd, dst, n, static_cast<off_t>(pos)) : ::read(fd, dst, n);
                if (r >= 0) {
                    if (par) pos += static_cast<std::uint64_t>(r);
                    return static_cast<std::size_t>(r);
                }
                if (errno != EINTR) throw std::runtime_error("read");
            }
        }
        const std::size_t want = static_cast<std::size_t>(std::min<std::uint64_t>(n, size - pos));
        std::atomic<bool> bad{false};
        pool->run([&](int i, int parts) {
            std::size_t lo, hi;
            part_range(want, i, parts, &lo, &hi);
            while (lo < hi && !bad) {
                const ssize_t r = ::pread(fd, dst + lo, hi - lo, static_cast<off_t>(pos + lo));
                if (r > 0) lo += static_cast<std::size_t>(r);
                else if (r < 0 && errno == EINTR) continue;
                else bad = true;  // error, or the file shrank under us
            }
        });
        if (bad) throw std::runtime_error("read");
        pos += want;
        return want;
    }
};

struct FdSink : t3b::ByteSink {
    int fd;
    t3b::PartPool* pool;
    bool par = false;
    std::uint64_t size = 0, pos = 0;
    FdSink(int f, t3b::PartPool* p) : fd(f), pool(p) { par = pool && regular_fd(fd, true, &size, &pos); }
    ~FdSink() override {
        if (par) (void)lseek(fd, static_cast<off_t>(pos), SEEK_SET);
    }
    void write(const std::uint8_t* src, std::size_t n) override {
        if (par && n >= (std::size_t(1) << 20)) {
            std::atomic<bool> bad{false};
            pool->run([&](int i, int parts) {
                std::size_t lo, hi;
                part_range(n, i, parts, &lo, &hi);
                while (lo < hi && !bad) {
                    const ssize_t w = ::pwrite(fd, src + lo, hi - lo, static_cast<off_t>(pos + lo));
                    if (w > 0) lo += static_cast<std::size_t>(w);
                    else if (w < 0 && errno == EINTR) continue;
                    else bad = true;
                }
            });
            if (bad) throw std::runtime_error("write");
            pos += n;
            return;
        }
        while (n) {
            const ssize_t w = par ? ::pwrite(fd, src, n, static_cast<off_t>(pos)) : ::write(fd, src, n);
            if (w < 0) {
                if (errno == EINTR) continue;
                throw std::runtime_error("write");
            }
            if (par) pos += static_cast<std::uint64_t>(w);
            src += w;
            n -= static_cast<std::size_t>(w);
        }
    }
};

}  // namespace

extern "C" int t3des_cu_stream_fd(t3des_cu_ctx* c, int dir, int in_fd, int out_fd, size_t chunk_blocks, int pkcs7,
                                  t3des_cu_stream_report* report) {
    if (!c || (dir != T3DES_CU_ENCRYPT && dir != T3DES_CU_DECRYPT) || chunk_blocks == 0 || in_fd < 0 ||
        out_fd < 0)
        return T3DES_CU_ERR_ARG;
    if (!c->have_schedule) return T3DES_CU_ERR_NO_SCHEDULE;
    if (report) std::memset(report, 0, sizeof *report);
    // Regular files: parallel pread/pwrite, and I/O in >= 16 MiB pieces
    // (whole reference chunks) when the input's length is known to be valid
    // — a length error must surface after exactly the chunks the reference
    // writes first, which the chunk-by-chunk loop reproduces.
    if (!c->io_pool) c->io_pool = new t3b::PartPool(std::clamp(t3b::available_cpus() / 2, 1, 8));
    FdSource src(in_fd, c->io_pool);
    FdSink dst(out_fd, c->io_pool);
    std::size_t io_blocks = chunk_blocks;
    const bool len_ok = src.par && (src.size - src.pos) % 8 == 0;
    if (src.par && (len_ok || (dir == T3DES_CU_ENCRYPT && pkcs7))) {
        constexpr std::size_t kIoBlocks = (std::size_t(16) << 20) / 8;
        io_blocks = (kIoBlocks + chunk_blocks - 1) / chunk_blocks * chunk_blocks;
    }
    if (const char* e = std::getenv("T3DES_STREAM_IO_MIB"))  // experiments
        io_blocks = std::max<std::size_t>(1, (std::size_t(std::atoi(e)) << 17) / chunk_blocks) * chunk_blocks;
    try {
        const t3b::StreamStats s = t3b::run_stream(c, dir, src, dst, chunk_blocks, pkcs7 != 0, io_blocks);
        if (report) {
            report->bytes_in = s.bytes_in;
            report->bytes_out = s.bytes_out;
            report->chunks = s.chunks;
            report->compute_seconds = s.compute_seconds;
            report->io_seconds = s.io_seconds;
        }
        return T3DES_CU_OK;
    } catch (const t3b::StreamFailure& f) {
        if (report) report->error_offset = f.byte_offset;
        switch (f.kind) {
            case t3b::StreamFailure::Length: return T3DES_CU_ERR_LENGTH;
            case t3b::StreamFailure::Padding: return T3DES_CU_ERR_PADDING;
            case t3b::StreamFailure::Io: return T3DES_CU_ERR_IO;
            default: return f.status ? f.status : T3DES_CU_ERR_CUDA;
        }
    } catch (const std::exception&) {
        return T3DES_CU_ERR_CUDA;
    }
}
