/*
 * t3des_cu.h — C ABI of the B200-native 3DES-ECB engine
 * (libt3des_b200.so, built from paper_1305_4376_b200/csrc).
 *
 * This is the drop-in boundary for the reference's hot path.  The
 * reference (/root/reference/proj, "t3des") exposes a C++ API; its batch
 * entry points are
 *     void encrypt_batch(std::span<const uint8_t> in, std::span<uint8_t> out,
 *                        const TripleSchedule&, const DispatchConfig&);
 *     void decrypt_batch(...);                  (include/t3des/dispatch.hpp:64-69)
 * dispatched per chunk to a Backend in run_chunk (src/dispatch.cpp:60-86).
 * The engine plugs in as a new Backend::Cuda routed from run_batch
 * (src/dispatch.cpp:105) to t3des_cu_ecb_host — see INTEGRATION.md.
 *
 * Conventions
 *   - plain pointers and sizes, no C++ or torch types;
 *   - every function returns an int status (T3DES_CU_OK = 0); nothing
 *     throws across the ABI; t3des_cu_strerror() maps codes to text;
 *   - no CPU fallback: without a usable sm_100 device the device-facing
 *     calls fail with T3DES_CU_ERR_NO_DEVICE / T3DES_CU_ERR_CUDA;
 *   - a context is used from one submitting thread at a time
 *     (reference SPEC.md:233: "safe to use from one submitting context").
 */
#ifndef T3DES_CU_H
#define T3DES_CU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  The C++ layer maps 1-2 to InputLengthError
 * (dispatch.hpp:44-47), 3 to KeyFormatError (tdes.hpp:25-28), 8 to
 * PaddingError and 9 to IoError (dispatch.hpp:49-59). */
#define T3DES_CU_OK 0
#define T3DES_CU_ERR_LENGTH 1      /* byte length not a multiple of 8       */
#define T3DES_CU_ERR_OVERLAP 2     /* in/out partially overlap              */
#define T3DES_CU_ERR_KEY 3         /* hex key: bad length or character      */
#define T3DES_CU_ERR_ARG 4         /* null pointer, bad enum, bad size      */
#define T3DES_CU_ERR_NO_DEVICE 5   /* no CUDA device / not sm_100           */
#define T3DES_CU_ERR_CUDA 6        /* a CUDA runtime call failed            */
#define T3DES_CU_ERR_NO_SCHEDULE 7 /* t3des_cu_set_schedule not called yet  */
#define T3DES_CU_ERR_PADDING 8     /* malformed PKCS#7 padding (PaddingError) */
#define T3DES_CU_ERR_IO 9          /* stream read/write failure (IoError)    */
#define T3DES_CU_ERR_JIT 10        /* NVRTC missing or the keyed compile failed */

#define T3DES_CU_ENCRYPT 0
#define T3DES_CU_DECRYPT 1

#define T3DES_CU_VARIANT_BITSLICE 0     /* bitsliced lop3 kernel, TMA tile prefetch           */
#define T3DES_CU_VARIANT_SPTABLE 1      /* shared-memory SP-table kernel                      */
#define T3DES_CU_VARIANT_BITSLICE_LDG 2 /* bitsliced, direct LDG loads (kept for measurement) */
/* Tuning variants of the bitsliced + TMA kernel (A/B measurement only):   */
#define T3DES_CU_VARIANT_BITSLICE_ALU 3    /* all key/shift work on the ALU pipe    */
#define T3DES_CU_VARIANT_BITSLICE_DFMA 4   /* E-duplicate key XORs as IMAD          */
#define T3DES_CU_VARIANT_BITSLICE_SHRFMA 5 /* transpose right shifts as IMAD.HI     */
/* Default: bitsliced, except launches of <= T3DES_CU_AUTO_SMALL_BLOCKS blocks,
 * which go to the SP-table kernel (lower latency: one thread per block instead
 * of one warp per 1024 blocks; measured crossover ~1 MiB). */
#define T3DES_CU_VARIANT_AUTO 6
#define T3DES_CU_AUTO_SMALL_BLOCKS 131072
/* Key-specialised bitsliced kernel: the installed schedule's
 * round keys folded into the LOP3 immediates of a cipher that NVRTC compiles
 * at run time, one module per (key sequence, direction), kept for the
 * process lifetime.  Opt-in: AUTO never compiles it — it executes about the
 * same ALU operations per block as the table-driven kernel (whitening
 * already keeps the key XORs off the ALU pipe) and the first use
 * of a key pays the compile (t3des_cu_keyed_prepare; seconds) — but once
 * t3des_cu_keyed_prepare has built it for the installed schedule and a
 * direction, AUTO's bitsliced launches (> T3DES_CU_AUTO_SMALL_BLOCKS) in that
 * direction run it, and small launches stay on the SP-table kernel.  Full 1024-block tiles
 * of 16-byte aligned spans run keyed; a partial tile and unaligned spans run
 * the table-driven kernels.  The compiled code embeds the key: it is held in
 * process and device memory only, never written to disk. */
#define T3DES_CU_VARIANT_KEYED 7

typedef struct t3des_cu_ctx t3des_cu_ctx;

/* Library version (major*10000 + minor*100 + patch). */
int t3des_cu_version(void);
const char* t3des_cu_strerror(int code);

/* ---- keying (host only, no device needed) ------------------------------ */

/* Replaces parse_hex_key (tdes.hpp:32; tdes.cpp:32-59): 48/32/16 hex chars
 * -> keying option 1/2/3 (written to *option) and keys k1,k2,k3 (k3 = k1
 * for option 2; all equal for option 3).  T3DES_CU_ERR_KEY on bad input. */
int t3des_cu_parse_hex_key(const char* hex, size_t len, uint64_t keys[3], int* option);

/* Replaces triple_schedule (tdes.hpp:42; tdes.cpp:84-87): 48 subkeys,
 * pass-major (16 for k1, then k2, then k3) — exactly the memory of the
 * reference's TripleSchedule {pass1, pass2, pass3} (tdes.hpp:38-40). */
int t3des_cu_triple_schedule(const uint64_t keys[3], uint64_t sub48[48]);

/* Key hygiene, replacing has_odd_parity / is_weak_key / is_semiweak_key
 * (des.hpp:41-48; des.cpp:159-207): a bit mask of the T3DES_CU_KEY_* flags
 * below for one 64-bit DES key.  Weak and semi-weak keys are compared with
 * the parity bits (the LSB of every byte) masked off, as in the reference. */
#define T3DES_CU_KEY_ODD_PARITY 1 /* every byte has odd parity        */
#define T3DES_CU_KEY_WEAK 2       /* one of the 4 weak keys           */
#define T3DES_CU_KEY_SEMIWEAK 4   /* one of the 12 semi-weak keys     */
int t3des_cu_des_key_flags(uint64_t key);

/* Replaces normalize_parity (des.hpp:42; des.cpp:167-175): flips the LSB of
 * every byte whose parity is even. */
uint64_t t3des_cu_normalize_parity(uint64_t key);

/* Replaces run_verification (verify.hpp:37; verify.cpp:65-124) for C and
 * ctypes callers: the walkthrough schedule, DES/3DES known answers, round
 * trips, complementation and the EDE collapse, on `device`.  The report
 * (one line per group, then "verification PASSED"/"FAILED") is copied into
 * `report` (NUL-terminated, truncated to `capacity`) when non-null.  Returns
 * T3DES_CU_OK if every group passed, T3DES_CU_ERR_ARG if one failed, or the
 * error of a failing call. */
int t3des_cu_run_verification(int device, char* report, size_t capacity);

/* ---- contexts ------------------------------------------------------------ */

int t3des_cu_device_count(int* count);

/* One context per device; owns its streams and staging buffers. */
int t3des_cu_create(int device, t3des_cu_ctx** out);
int t3des_cu_destroy(t3des_cu_ctx* ctx);

/* Install the 48-subkey schedule (pass-major, as above).  The host
 * flattens it once into the encrypt and decrypt execution sequences
 * (tdes.cpp:177-185) and the kernels' constant tables; no device traffic. */
int t3des_cu_set_schedule(t3des_cu_ctx* ctx, const uint64_t sub48[48]);

/* T3DES_CU_VARIANT_*; default AUTO. */
int t3des_cu_set_variant(t3des_cu_ctx* ctx, int variant);

/* T3DES_CU_VARIANT_KEYED: compile (or find in the process cache) the keyed
 * kernel for the installed schedule and `direction` and load it on the
 * context's device, so that no later launch pays for it (call it before
 * capturing a CUDA graph).  *compile_seconds (may be NULL) = the time spent
 * here, 0 on a cache hit.  T3DES_CU_ERR_JIT when NVRTC is unavailable
 * (libnvrtc.so.12; T3DES_NVRTC names another path) or fails. */
int t3des_cu_keyed_prepare(t3des_cu_ctx* ctx, int direction, double* compile_seconds);

/* Context-free and device-free: the keyed kernel's CUBIN (sm_100a) for a
 * schedule and direction, as t3des_cu_keyed_prepare builds it — for
 * inspection and tests (no GPU needed).  *size = the CUBIN's size; the bytes
 * are written when capacity >= *size (cubin may be NULL to query). */
int t3des_cu_keyed_compile(const uint64_t sub48[48], int direction, void* cubin, size_t capacity, size_t* size,
                           double* compile_seconds);

/* Launch shaping, the GPU reading of DispatchConfig (dispatch.hpp:25-30):
 * chunk_blocks = blocks per kernel launch (0 = whole batch in one launch,
 * the default), work_group = threads per CTA (0 = kernel default).  Only
 * for Table I/II-style sweeps; results never depend on them. */
int t3des_cu_set_launch(t3des_cu_ctx* ctx, size_t chunk_blocks, int work_group);

/* ---- ECB batch ------------------------------------------------------------ */

/* Device-resident batch: din/dout are device pointers on the context's
 * device, len is in bytes.  Asynchronous on `stream` (a cudaStream_t; NULL
 * = legacy default stream).  in == out (in place) is allowed, partial
 * overlap is rejected, len == 0 is a no-op (dispatch.cpp:91-104,215). */
int t3des_cu_ecb_device(t3des_cu_ctx* ctx, int direction, const void* din, void* dout,
                        size_t len, void* stream);
/* (Spans that are not 8-byte aligned are bounced through an aligned device
 * buffer, and the call then returns only when the work is done.) */

/* Host buffers, end to end: chunked H2D -> kernel -> D2H pipelined over
 * several streams (t3des_cu_set_pipeline); returns when `out` holds the result.  This is the entry
 * a Backend::Cuda branch of run_batch calls (same contract as
 * encrypt_batch/decrypt_batch).  Pinned buffers (t3des_cu_host_alloc)
 * give full PCIe overlap; pageable spans are staged through a pinned ring
 * by host copy threads (T3DES_HOST_COPY_THREADS, default 3/4 of the host's
 * threads, at most 12).  Device memory is rejected (T3DES_CU_ERR_ARG): use
 * t3des_cu_ecb_device. */
int t3des_cu_ecb_host(t3des_cu_ctx* ctx, int direction, const uint8_t* in, uint8_t* out,
                      size_t len);

/* Host-path pipeline shape: bytes per stage (multiple of 8) and number of
 * streams/staging buffers (1..8).  Default: 3 streams, stage size adapted
 * to each batch (about len/8, clamped to 8..32 MiB). */
int t3des_cu_set_pipeline(t3des_cu_ctx* ctx, size_t chunk_bytes, int streams);

/* Host buffers sharded by contiguous block ranges (multiples of 1024
 * blocks) over `ndev` devices, one host thread and (pooled) context per
 * device; no collective.  Blocks are independent, so the result
 * equals the single-device result.  Where the host has several NUMA nodes,
 * each shard's submitting thread, host copy threads and pinned staging ring
 * are placed on its GPU's node (sysfs; T3DES_NUMA=0 disables). */
int t3des_cu_ecb_multi(const int* devices, int ndev, const uint64_t sub48[48], int direction,
                       const uint8_t* in, uint8_t* out, size_t len);

/* The GPU reading of the reference's DispatchConfig.workers
 * (dispatch.hpp:28, the worker count its run_chunk hands to OpenMP,
 * dispatch.cpp:73-84): min(workers, visible devices) shards (workers 0 = 1)
 * of the host batch on consecutive devices from first_device (wrapping) —
 * workers = 8 on an 8-GPU node uses every GPU once; on one GPU any workers
 * value runs one shard (a CPU-sized thread count would only put several
 * contexts on one device; t3des_cu_ecb_multi with a repeated device does
 * that on purpose).  One shard runs on a pooled context of first_device;
 * more go through t3des_cu_ecb_multi over that device list.  Synchronous.
 * This is what the patched reference's Backend::Cuda calls. */
int t3des_cu_ecb_workers(unsigned workers, int first_device, const uint64_t sub48[48], int direction,
                         const uint8_t* in, uint8_t* out, size_t len);

/* Device-resident multi-GPU (NVLink 5 / NVSwitch): din/dout
 * live on `home_device`; shard g (t3des_cu_shard_range) is copied to
 * devices[g] with cudaMemcpyPeerAsync, transformed there and copied back.
 * A shard whose device is the home device is transformed in place of
 * din -> dout without copies unless flags & T3DES_CU_MULTI_STAGE_ALL; the
 * shard sizes are t3des_cu_multi_device_shards (the home shard weighted).
 * A remote shard whose device can map the home GPU's memory runs
 * peer-direct: its kernel loads and stores the home buffers over NVLink, so
 * transfer and compute overlap inside the kernel with no staging.  Otherwise
 * (or with T3DES_CU_MULTI_COPY) it is pipelined in chunks over three streams
 * of its device (peer copy in, kernel, peer copy out overlap chunk by chunk).
 * Synchronous.  Peer access is enabled where the topology allows it. */
#define T3DES_CU_MULTI_STAGE_ALL 1 /* every shard, the home one too, through the copy pipeline */
#define T3DES_CU_MULTI_COPY 2      /* remote shards through the copy pipeline even with peer access */
int t3des_cu_ecb_multi_device(const int* devices, int ndev, const uint64_t sub48[48], int direction,
                              int home_device, const void* din, void* dout, size_t len, int flags);

/* The block ranges t3des_cu_ecb_multi_device gives each of its `ndev`
 * devices for a payload resident on `home` (first[g], count[g]): the home
 * GPU's shard, which needs no NVLink copy, is weighted against the remote
 * shards' peer-copy bound (about a third of the blocks at 3+ GPUs); equal
 * tile-rounded ranges when the home GPU is not among the devices exactly once
 * or with T3DES_CU_MULTI_STAGE_ALL. */
int t3des_cu_multi_device_shards(const int* devices, int ndev, int home, uint64_t nblocks, int flags,
                                 uint64_t* first, uint64_t* count);

/* The block range device `g` of `ndev` owns in t3des_cu_ecb_multi (and in
 * bench.py's torchrun ranks): [first, first + count), boundaries at
 * floor(g*N/ndev) rounded down to 1024-block tiles; the last shard ends at N. */
int t3des_cu_shard_range(uint64_t nblocks, int ndev, int g, uint64_t* first, uint64_t* count);

/* ---- streams ------------------------------------------------------------- */

/* Mirrors the reference's StreamReport (dispatch.hpp:71-77). */
typedef struct t3des_cu_stream_report {
    uint64_t bytes_in;
    uint64_t bytes_out;
    uint64_t chunks;
    double compute_seconds; /* engine time not overlapped with I/O */
    double io_seconds;      /* reads and writes                    */
    uint64_t error_offset;  /* byte offset of an IO error          */
} t3des_cu_stream_report;

/* Replaces encrypt_stream/decrypt_stream (dispatch.hpp:79-91,
 * dispatch.cpp:111-206) on file descriptors: reads chunk_blocks*8-byte
 * chunks from in_fd, writes the transformed bytes to out_fd in order.
 * pkcs7 = 1: encrypt pads the last chunk, decrypt strips and checks the
 * padding of the last chunk (T3DES_CU_ERR_PADDING).  Without padding the
 * input length must be a multiple of 8 (T3DES_CU_ERR_LENGTH).  Read/write
 * failures return T3DES_CU_ERR_IO with report->error_offset set.  Chunk k+1
 * is read while chunk k runs on the device; output equals the reference's
 * byte for byte. */
int t3des_cu_stream_fd(t3des_cu_ctx* ctx, int direction, int in_fd, int out_fd, size_t chunk_blocks,
                       int pkcs7, t3des_cu_stream_report* report);

/* ---- utilities --------------------------------------------------------- */

/* Pinned host memory for t3des_cu_ecb_host. */
int t3des_cu_host_alloc(size_t bytes, void** out);
int t3des_cu_host_free(void* p);

/* Opt-in page-locking of a caller's existing (pageable) buffer, for callers
 * that pass the same std::vector / array to many batch calls: once
 * registered, t3des_cu_ecb_host DMAs straight from/to it (the pinned path,
 * PCIe-bound) instead of staging it through the engine's pinned ring (host-
 * DRAM-bound, about half the rate).  Registration itself costs about as much
 * as one staged transform of the buffer, so it pays from the second call on.
 * The caller must unregister before freeing the memory.  Never done
 * implicitly: a freed-and-reused address would keep stale pages pinned. */
int t3des_cu_host_register(void* p, size_t bytes);
int t3des_cu_host_unregister(void* p);

/* Device payload generator for inputs larger than host RAM: block
 * (first_block + i) = splitmix64(seed ^ (first_block + i)), big-endian. */
int t3des_cu_fill_splitmix(t3des_cu_ctx* ctx, void* dptr, uint64_t first_block, size_t nblocks,
                           uint64_t seed, void* stream);

/* Shard-additive, order-sensitive checksum of nblocks device blocks whose
 * global index starts at first_block.  Runs on `stream` (ordered after the
 * work that produced dptr) and synchronises it; result in *out. */
int t3des_cu_checksum(t3des_cu_ctx* ctx, const void* dptr, uint64_t first_block, size_t nblocks,
                      uint64_t* out, void* stream);

/* Number of cipher kernels this context has launched (for bench.py's
 * gpu_launches count). */
int t3des_cu_launch_count(t3des_cu_ctx* ctx, uint64_t* out);

#ifdef __cplusplus
}
#endif

#endif /* T3DES_CU_H */
