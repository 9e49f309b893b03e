// Chunked stream encryption over the CUDA engine: the
// reference's run_stream (/root/reference/proj/src/dispatch.cpp:111-206)
// with the same chunking, PKCS#7 and error semantics, but pipelined: chunk
// k+1 is read while chunk k is in flight (pinned H2D -> kernel -> D2H on
// its own stream), which also tells the loop whether chunk k is the last
// one (the reference peeks the istream for that).
#pragma once
#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>

struct t3des_cu_ctx;

namespace t3b {

struct ByteSource {
    virtual ~ByteSource() = default;
    // Read up to n bytes; returns the count (0 at end of stream).  Throws
    // StreamFailure{kind = Io} on a read error.
    virtual std::size_t read(std::uint8_t* dst, std::size_t n) = 0;
};

struct ByteSink {
    virtual ~ByteSink() = default;
    virtual void write(const std::uint8_t* src, std::size_t n) = 0;  // throws on failure
    virtual void flush() {}
};

struct StreamStats {
    std::uint64_t bytes_in = 0;
    std::uint64_t bytes_out = 0;
    std::uint64_t chunks = 0;
    double compute_seconds = 0.0;  // engine time not overlapped with I/O
    double io_seconds = 0.0;       // reads and writes
};

// Failure kinds map to the reference's exception types: Length ->
// InputLengthError, Padding -> PaddingError, Io -> IoError{byte_offset},
// Cuda -> engine status.
struct StreamFailure : std::runtime_error {
    enum Kind { Length, Padding, Io, Cuda } kind;
    std::uint64_t byte_offset;
    int status;
    StreamFailure(Kind k, const std::string& what, std::uint64_t off = 0, int st = 0)
        : std::runtime_error(what), kind(k), byte_offset(off), status(st) {}
};

// PKCS#7 over 8-byte blocks (dispatch.cpp:245-261).
void pkcs7_pad_bytes(std::uint8_t* data, std::size_t len, std::size_t* out_len);  // needs len%8 + 8 room
// Returns the unpadded length; throws StreamFailure{Padding}.
std::size_t pkcs7_unpad_len(const std::uint8_t* data, std::size_t len);

// The context must hold a schedule.  chunk_blocks >= 1.  io_blocks (a
// multiple of chunk_blocks; 0 = chunk_blocks) is the granularity the source
// is read, transformed and written in: the output bytes, the padding and the
// reported chunk count are those of chunk_blocks (the reference's chunks),
// larger I/O only amortises per-call costs (the fd entry uses it for regular
// files of known length).  copy_only: Backend::NoOpCopy (the reference's
// timing instrument, dispatch.cpp:63-72) — the same chunking, padding, errors
// and counters, with the chunks written out untransformed (no device work).
StreamStats run_stream(t3des_cu_ctx* ctx, int direction, ByteSource& src, ByteSink& dst,
                       std::size_t chunk_blocks, bool pkcs7, std::size_t io_blocks = 0, bool copy_only = false);

}  // namespace t3b
