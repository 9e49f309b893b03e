// Key-specialised kernels compiled at run time:
// T3DES_CU_VARIANT_KEYED.
//
// The reference computes the schedule once per run, before any block work
// (SPEC.md:118-120), so a kernel can be built for one key: keyed_kernel.cuh
// instantiates t3_keyed_round<K> (generated/keyed_rounds.cuh) for the 48 (or
// 16) round keys of one execution sequence, which puts every key bit into a
// LOP3 immediate.  NVRTC compiles that source to an sm_100a CUBIN here;
// cudaLibraryLoadData loads it (context-independent, so one module serves
// every device).  Modules are cached per (sequence, rounds) for the process
// lifetime.  The headers NVRTC reads are embedded at build time
// (embed_sources.py -> build/keyed_sources.inc), and libnvrtc is opened
// with dlopen on first use, so the engine has no link-time NVRTC dependency
// and the other variants never touch it.
//
// Secrets: the source text and the CUBIN encode the key.  Both are wiped
// after use; nothing is written to disk (no on-disk kernel cache).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "ctx.hpp"
#include "schedule.hpp"
#include "t3des_cu.h"

#include "build/keyed_sources.inc"

namespace {

constexpr int kKeyedWarps = 16;  // T3_KEYED_WARPS of keyed_kernel.cuh
constexpr int kKeyedSmem = kKeyedWarps * T3_TILE_BLOCKS * 8;

void wipe(void* p, std::size_t n) {
    volatile unsigned char* v = static_cast<volatile unsigned char*>(p);
    while (n--) *v++ = 0;
}

// libnvrtc, resolved once
struct Nvrtc {
    decltype(&nvrtcCreateProgram) create = nullptr;
    decltype(&nvrtcCompileProgram) compile = nullptr;
    decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
    decltype(&nvrtcGetCUBIN) cubin = nullptr;
    decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
    decltype(&nvrtcGetProgramLog) log = nullptr;
    decltype(&nvrtcDestroyProgram) destroy = nullptr;
    bool ok = false;

    static const Nvrtc& get() {
        static const Nvrtc n = [] {
            Nvrtc r;
            const char* env = std::getenv("T3DES_NVRTC");
            const char* cands[] = {env, "/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so.12", "libnvrtc.so"};
            void* h = nullptr;
            for (const char* p : cands)
                if (p && (h = dlopen(p, RTLD_NOW | RTLD_LOCAL))) break;
            if (!h) return r;
            r.create = reinterpret_cast<decltype(r.create)>(dlsym(h, "nvrtcCreateProgram"));
            r.compile = reinterpret_cast<decltype(r.compile)>(dlsym(h, "nvrtcCompileProgram"));
            r.cubin_size = reinterpret_cast<decltype(r.cubin_size)>(dlsym(h, "nvrtcGetCUBINSize"));
            r.cubin = reinterpret_cast<decltype(r.cubin)>(dlsym(h, "nvrtcGetCUBIN"));
            r.log_size = reinterpret_cast<decltype(r.log_size)>(dlsym(h, "nvrtcGetProgramLogSize"));
            r.log = reinterpret_cast<decltype(r.log)>(dlsym(h, "nvrtcGetProgramLog"));
            r.destroy = reinterpret_cast<decltype(r.destroy)>(dlsym(h, "nvrtcDestroyProgram"));
            r.ok = r.create && r.compile && r.cubin_size && r.cubin && r.log_size && r.log && r.destroy;
            return r;
        }();
        return n;
    }
};

// The execution sequence the kernels run for `dir`: 48 keys, or the 16 of
// a schedule whose EDE collapses to single DES (as t3des_cu_set_schedule).
int keyed_sequence(const std::uint64_t sub48[48], int dir, std::uint64_t seq[48]) {
    std::fill(seq, seq + 48, 0);
    if (t3b::collapsed_sequence(sub48, dir == T3DES_CU_DECRYPT, seq) == 16) return 16;
    t3b::key_sequence(sub48, dir == T3DES_CU_DECRYPT, seq);
    return 48;
}

// NVRTC: the keyed kernel for one sequence -> CUBIN.  T3DES_CU_OK or
// T3DES_CU_ERR_JIT (the log goes to stderr with T3DES_JIT_VERBOSE=1).
int compile_cubin(const std::uint64_t* seq, int rounds, std::vector<char>& cubin) {
    const Nvrtc& nv = Nvrtc::get();
    if (!nv.ok) return T3DES_CU_ERR_JIT;
    std::string src = "#include <stdint.h>\nconstexpr uint64_t T3_KSEQ[] = {";
    char num[32];
    for (int t = 0; t < rounds; ++t) {
        std::snprintf(num, sizeof num, "%s0x%012llxull", t ? ", " : "", static_cast<unsigned long long>(seq[t]));
        src += num;
    }
    wipe(num, sizeof num);
    src += "};\nconstexpr int T3_KROUNDS = " + std::to_string(rounds) + ";\n#include \"keyed_kernel.cuh\"\n";
    nvrtcProgram prog = nullptr;
    int rc = T3DES_CU_OK;
    if (nv.create(&prog, src.c_str(), "t3des_keyed.cu", kKeyedHeaderCount, kKeyedHeaders, kKeyedHeaderNames) !=
        NVRTC_SUCCESS)
        rc = T3DES_CU_ERR_JIT;
    if (!rc) {
        std::vector<const char*> opts = {"-arch=sm_100a", "-std=c++17", "-lineinfo", "-DT3_NVRTC=1"};
        // experiments: extra NVRTC options, e.g. "-DT3_KEYED_SYNC_EVERY=8"
        std::vector<std::string> extra;
        if (const char* e = std::getenv("T3DES_KEYED_NVRTC_OPTS")) {
            std::string all(e);
            for (std::size_t p = 0; p < all.size();) {
                const std::size_t q = std::min(all.find(' ', p), all.size());
                if (q > p) extra.push_back(all.substr(p, q - p));
                p = q + 1;
            }
        }
        for (const auto& x : extra) opts.push_back(x.c_str());
        const nvrtcResult cr = nv.compile(prog, int(opts.size()), opts.data());
        if (cr != NVRTC_SUCCESS || std::getenv("T3DES_JIT_VERBOSE")) {
            std::size_t n = 0;
            if (nv.log_size(prog, &n) == NVRTC_SUCCESS && n > 1) {
                std::string log(n, '\0');
                if (nv.log(prog, &log[0]) == NVRTC_SUCCESS) std::fprintf(stderr, "t3des keyed JIT: %s\n", log.c_str());
            }
        }
        if (cr != NVRTC_SUCCESS) rc = T3DES_CU_ERR_JIT;
    }
    std::size_t n = 0;
    if (!rc && (nv.cubin_size(prog, &n) != NVRTC_SUCCESS || n == 0)) rc = T3DES_CU_ERR_JIT;
    if (!rc) {
        cubin.assign(n, 0);
        if (nv.cubin(prog, cubin.data()) != NVRTC_SUCCESS) rc = T3DES_CU_ERR_JIT;
    }
    if (prog) nv.destroy(&prog);
    wipe(&src[0], src.size());
    return rc;
}

struct KeyedModule {
    std::uint64_t seq[48];
    int rounds;
    cudaLibrary_t lib;
    cudaKernel_t kern;
    std::uint64_t smem_set;  // devices (bit d) on which the dynamic shared memory limit is raised
};

std::mutex g_mu;
std::vector<std::unique_ptr<KeyedModule>> g_modules;  // never unloaded: contexts hold pointers

KeyedModule* find_module(const std::uint64_t* seq, int rounds) {
    for (auto& m : g_modules)
        if (m->rounds == rounds && std::memcmp(m->seq, seq, sizeof m->seq) == 0) return m.get();
    return nullptr;
}

double seconds_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

namespace t3b {

int keyed_prepare(t3des_cu_ctx* c, int dir, double* seconds) {
    const auto t0 = std::chrono::steady_clock::now();
    if (seconds) *seconds = 0.0;
    if (!c->have_schedule) return T3DES_CU_ERR_NO_SCHEDULE;
    std::uint64_t seq[48];
    const int rounds = keyed_sequence(c->sub48, dir, seq);
    KeyedModule* m = nullptr;
    {
        std::lock_guard<std::mutex> l(g_mu);
        m = find_module(seq, rounds);
    }
    if (!m) {  // compile outside the lock: other keys' launches go on meanwhile
        std::vector<char> cubin;
        int rc = compile_cubin(seq, rounds, cubin);
        auto fresh = std::make_unique<KeyedModule>();
        std::memcpy(fresh->seq, seq, sizeof seq);
        fresh->rounds = rounds;
        fresh->smem_set = 0;
        if (!rc && cudaLibraryLoadData(&fresh->lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) != cudaSuccess)
            rc = T3DES_CU_ERR_CUDA;
        wipe(cubin.data(), cubin.size());
        if (!rc && cudaLibraryGetKernel(&fresh->kern, fresh->lib, "t3_keyed_kernel") != cudaSuccess) {
            cudaLibraryUnload(fresh->lib);
            rc = T3DES_CU_ERR_CUDA;
        }
        wipe(seq, sizeof seq);
        if (rc) {
            (void)cudaGetLastError();
            return rc;
        }
        std::lock_guard<std::mutex> l(g_mu);
        if ((m = find_module(fresh->seq, rounds)) != nullptr) {
            cudaLibraryUnload(fresh->lib);  // another thread loaded the same key first
        } else {
            g_modules.push_back(std::move(fresh));
            m = g_modules.back().get();
        }
    }
    wipe(seq, sizeof seq);
    {
        std::lock_guard<std::mutex> l(g_mu);
        const std::uint64_t bit = c->device < 64 ? (std::uint64_t(1) << c->device) : 0;
        if (!(m->smem_set & bit)) {
            if (cudaKernelSetAttributeForDevice(m->kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kKeyedSmem,
                                                c->device) != cudaSuccess) {
                (void)cudaGetLastError();
                return T3DES_CU_ERR_CUDA;
            }
            m->smem_set |= bit;
        }
    }
    c->keyed[dir] = m;
    if (seconds) *seconds = seconds_since(t0);
    return T3DES_CU_OK;
}

int keyed_launch(t3des_cu_ctx* c, int dir, const std::uint8_t* in, std::uint8_t* out, std::uint64_t ntiles,
                 cudaStream_t s) {
    if (!c->keyed[dir])
        if (int rc = keyed_prepare(c, dir, nullptr)) return rc;
    const auto* m = static_cast<const KeyedModule*>(c->keyed[dir]);
    // one 16-warp CTA per SM (launch bounds 512 x 1), every warp the same
    // number of tiles (keyed_kernel.cuh)
    const std::uint64_t grid =
        std::min<std::uint64_t>(std::uint64_t(c->sms), (ntiles + kKeyedWarps - 1) / kKeyedWarps);
    std::uint32_t zero = 0;  // an operand the compiler cannot fold (T3_KEYED_PIN experiments)
    void* args[] = {&in, &out, &ntiles, &zero};
    if (cudaLaunchKernel(reinterpret_cast<const void*>(m->kern), dim3(unsigned(std::max<std::uint64_t>(grid, 1))),
                         dim3(kKeyedWarps * 32), args, kKeyedSmem, s) != cudaSuccess) {
        (void)cudaGetLastError();
        return T3DES_CU_ERR_CUDA;
    }
    return T3DES_CU_OK;
}

}  // namespace t3b

extern "C" {

int t3des_cu_keyed_prepare(t3des_cu_ctx* c, int dir, double* compile_seconds) {
    if (!c || (dir != T3DES_CU_ENCRYPT && dir != T3DES_CU_DECRYPT)) return T3DES_CU_ERR_ARG;
    t3b::DeviceScope scope(c->device);
    return t3b::keyed_prepare(c, dir, compile_seconds);
}

int t3des_cu_keyed_compile(const std::uint64_t sub48[48], int dir, void* cubin, std::size_t capacity,
                           std::size_t* size, double* compile_seconds) {
    if (!sub48 || !size || (dir != T3DES_CU_ENCRYPT && dir != T3DES_CU_DECRYPT)) return T3DES_CU_ERR_ARG;
    const auto t0 = std::chrono::steady_clock::now();
    std::uint64_t seq[48];
    const int rounds = keyed_sequence(sub48, dir, seq);
    std::vector<char> bin;
    const int rc = compile_cubin(seq, rounds, bin);
    wipe(seq, sizeof seq);
    if (compile_seconds) *compile_seconds = seconds_since(t0);
    if (rc) return rc;
    *size = bin.size();
    if (cubin && capacity >= bin.size()) std::memcpy(cubin, bin.data(), bin.size());
    wipe(bin.data(), bin.size());
    return T3DES_CU_OK;
}

}  // extern "C"
