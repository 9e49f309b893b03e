// t3des_b200 — command-line front end of the B200 engine, mirroring the
// reference CLI (/root/reference/proj/tools/t3des_cli.cpp): subcommands
// encrypt | decrypt | verify | bench, the same flags and the same exit codes
// (0 ok, 1 I/O, 2 usage, 3 key format, 4 input length, 5 padding, 6 parity,
// 7 verification failed).  Differences: the backend is "cuda" (the engine
// has no CPU cipher; the reference's names scalar/threaded run on the
// engine, noop copies through), --workers counts GPUs, bench sweeps GPU
// launch shapes.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <string>
#include <vector>

#include "t3des_b200/bench.hpp"
#include "t3des_b200/t3des.hpp"
#include "t3des_cu.h"

namespace {

constexpr int kExitIo = 1, kExitUsage = 2, kExitKeyFormat = 3, kExitInputLength = 4, kExitPadding = 5,
              kExitParity = 6, kExitVerifyFailed = 7;

using t3des::ParityError;
struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct Opts {
    std::string cmd;
    std::string key_hex, key_file, input = "-", output = "-";
    bool pkcs7 = false, check_parity = false, strict_keys = false;
    std::size_t chunk_blocks = 131072, work_group = 0;  // work_group: CTA threads, 0 = kernel default
    unsigned workers = 0;
    std::string backend = "cuda", variant = "auto";
    int device = 0;
    // bench
    std::string sweep = "chunk", format = "csv", out, mode = "device";
    std::vector<std::size_t> values;
    std::uint64_t payload_mb = 64, seed = 0x3DE5C0DE;
    unsigned reps = 3;
};

std::size_t to_size(const std::string& v, const char* flag) {
    char* end = nullptr;
    const unsigned long long x = std::strtoull(v.c_str(), &end, 0);
    if (v.empty() || *end) throw UsageError(std::string("bad value for ") + flag + ": " + v);
    return static_cast<std::size_t>(x);
}

Opts parse(int argc, char** argv) {
    if (argc < 2) throw UsageError("a subcommand is required: encrypt | decrypt | verify | bench");
    Opts o;
    o.cmd = argv[1];
    if (o.cmd == "-h" || o.cmd == "--help") throw UsageError("");
    if (o.cmd != "encrypt" && o.cmd != "decrypt" && o.cmd != "verify" && o.cmd != "bench")
        throw UsageError("unknown subcommand: " + o.cmd);
    const bool crypt = o.cmd == "encrypt" || o.cmd == "decrypt";
    std::vector<std::string> pos;
    for (int i = 2; i < argc; ++i) {
        std::string a = argv[i];
        auto val = [&](const char* flag) -> std::string {
            const std::string f(flag);
            if (a.size() > f.size() && a.compare(0, f.size() + 1, f + "=") == 0) return a.substr(f.size() + 1);
            if (i + 1 >= argc) throw UsageError(std::string(flag) + " needs a value");
            return argv[++i];
        };
        auto is = [&](const char* flag) { return a == flag || a.rfind(std::string(flag) + "=", 0) == 0; };
        if (crypt && is("--key")) o.key_hex = val("--key");
        else if (crypt && is("--key-file")) o.key_file = val("--key-file");
        else if (crypt && a == "--pkcs7") o.pkcs7 = true;
        else if (crypt && a == "--check-parity") o.check_parity = true;
        else if (crypt && a == "--strict-keys") o.strict_keys = true;
        else if (is("--chunk-blocks")) o.chunk_blocks = to_size(val("--chunk-blocks"), "--chunk-blocks");
        else if (is("--work-group")) o.work_group = to_size(val("--work-group"), "--work-group");
        else if (is("--workers")) o.workers = static_cast<unsigned>(to_size(val("--workers"), "--workers"));
        else if (is("--backend")) o.backend = val("--backend");
        else if (is("--variant")) o.variant = val("--variant");
        else if (is("--device")) o.device = static_cast<int>(to_size(val("--device"), "--device"));
        else if (o.cmd == "bench" && is("--sweep")) o.sweep = val("--sweep");
        else if (o.cmd == "bench" && is("--values")) {
            std::string v = val("--values");
            std::size_t p = 0;
            while (p <= v.size()) {
                const std::size_t q = std::min(v.find(',', p), v.size());
                o.values.push_back(to_size(v.substr(p, q - p), "--values"));
                p = q + 1;
            }
        } else if (o.cmd == "bench" && is("--payload-mb")) o.payload_mb = to_size(val("--payload-mb"), "--payload-mb");
        else if (o.cmd == "bench" && is("--seed")) o.seed = to_size(val("--seed"), "--seed");
        else if (o.cmd == "bench" && is("--reps")) o.reps = static_cast<unsigned>(to_size(val("--reps"), "--reps"));
        else if (o.cmd == "bench" && is("--format")) o.format = val("--format");
        else if (o.cmd == "bench" && is("--out")) o.out = val("--out");
        else if (o.cmd == "bench" && is("--mode")) o.mode = val("--mode");
        else if (!a.empty() && a[0] == '-' && a != "-") throw UsageError("unknown option: " + a);
        else pos.push_back(a);
    }
    if (crypt) {
        if (pos.size() > 2) throw UsageError("too many positional arguments");
        if (!pos.empty()) o.input = pos[0];
        if (pos.size() > 1) o.output = pos[1];
    } else if (!pos.empty()) {
        throw UsageError("unexpected argument: " + pos[0]);
    }
    // the reference's names are accepted so its scripts run unchanged:
    // scalar/threaded (its two CPU routes of the same function) run on the
    // engine, noop copies through as in the reference
    if (o.backend != "cuda" && o.backend != "scalar" && o.backend != "threaded" && o.backend != "noop")
        throw UsageError("--backend must be cuda|scalar|threaded|noop");
    if ((o.backend == "scalar" || o.backend == "threaded") && crypt)
        std::cerr << "note: --backend " << o.backend << " runs on the B200 engine (this build has no CPU cipher)\n";
    if (o.variant != "auto" && o.variant != "bitslice" && o.variant != "sptable")
        throw UsageError("--variant must be auto|bitslice|sptable");
    if (o.cmd == "bench") {
        if (o.sweep != "workers" && o.sweep != "chunk" && o.sweep != "workgroup")
            throw UsageError("--sweep must be workers|chunk|workgroup");
        if (o.format != "csv" && o.format != "markdown") throw UsageError("--format must be csv|markdown");
        if (o.mode != "device" && o.mode != "host") throw UsageError("--mode must be device|host");
        if (o.reps < 1) throw UsageError("--reps must be >= 1");
    }
    if (o.chunk_blocks == 0) throw UsageError("--chunk-blocks must be positive");
    return o;
}

t3des::TripleKey load_key(const Opts& o) {
    std::string hex = o.key_hex;
    if (hex.empty() && !o.key_file.empty()) {
        std::ifstream in(o.key_file);
        if (!in) throw t3des::IoError("cannot open key file: " + o.key_file, 0);
        std::getline(in, hex);
        while (!hex.empty() && (hex.back() == '\r' || hex.back() == ' ')) hex.pop_back();
    }
    if (hex.empty()) throw t3des::KeyFormatError("a key is required (--key or --key-file)");
    t3des::TripleKey key = t3des::parse_hex_key(hex);
    for (const t3des::DesKey& k : {key.k1, key.k2, key.k3}) {
        if (o.check_parity && !t3des::has_odd_parity(k))
            throw ParityError("key byte fails odd-parity check (--check-parity)");
        if (t3des::is_weak_key(k) || t3des::is_semiweak_key(k)) {
            if (o.strict_keys) throw t3des::KeyFormatError("weak or semi-weak DES key rejected (--strict-keys)");
            std::cerr << "warning: key component is a weak or semi-weak DES key\n";
        }
    }
    return key;
}

t3des::DispatchConfig make_config(const Opts& o) {
    t3des::DispatchConfig cfg;
    cfg.chunk_blocks = o.chunk_blocks;
    cfg.work_group = o.work_group;
    cfg.workers = o.workers;
    if (cfg.workers == 0)
        if (const char* env = std::getenv("T3DES_WORKERS")) cfg.workers = static_cast<unsigned>(std::strtoul(env, nullptr, 10));
    cfg.backend = o.backend == "noop" ? t3des::Backend::NoOpCopy : t3des::Backend::Cuda;
    cfg.device = o.device;
    cfg.variant = o.variant == "sptable"    ? T3DES_CU_VARIANT_SPTABLE
                  : o.variant == "bitslice" ? T3DES_CU_VARIANT_BITSLICE
                                            : T3DES_CU_VARIANT_AUTO;
    return cfg;
}

int run_crypt(const Opts& o, bool encrypt) {
    const t3des::TripleSchedule ts = t3des::triple_schedule(load_key(o));
    const t3des::DispatchConfig cfg = make_config(o);
    const t3des::PaddingMode pad = o.pkcs7 ? t3des::PaddingMode::Pkcs7 : t3des::PaddingMode::None;
    std::ifstream fin;
    std::ofstream fout;
    std::istream* in = &std::cin;
    std::ostream* out = &std::cout;
    if (o.input != "-") {
        fin.open(o.input, std::ios::binary);
        if (!fin) {
            std::cerr << "error: cannot open input file: " << o.input << '\n';
            return kExitIo;
        }
        in = &fin;
    }
    if (o.output != "-") {
        fout.open(o.output, std::ios::binary);
        if (!fout) {
            std::cerr << "error: cannot open output file: " << o.output << '\n';
            return kExitIo;
        }
        out = &fout;
    }
    const t3des::StreamReport r = encrypt ? t3des::encrypt_stream(*in, *out, ts, cfg, pad)
                                          : t3des::decrypt_stream(*in, *out, ts, cfg, pad);
    std::cerr << (encrypt ? "encrypted " : "decrypted ") << r.bytes_in << " -> " << r.bytes_out << " bytes, "
              << r.chunks << " chunks, compute " << r.compute_seconds << " s, io " << r.io_seconds << " s\n";
    return 0;
}

// ---- verify: known answers and structural properties, on the GPU --------
// (the library's t3des::run_verification, verify_api.cpp)
int run_verify(const Opts& o) {
    return t3des::run_verification(std::cout, make_config(o)) ? 0 : kExitVerifyFailed;
}

// ---- bench: GPU sweeps shaped like the reference's Tables I/II/IV ---------
// Records, payload and reports are the library's t3des::bench (the reference
// harness's interface and formats); the device mode times the kernels alone.
using t3des::bench::BenchRecord;

int run_bench(const Opts& o) {
    std::vector<std::size_t> values = o.values;
    if (values.empty()) {
        if (o.sweep == "workers") values = {1};
        else if (o.sweep == "chunk") values = {128, 1024, 16384, 131072, 1048576};
        else values = {32, 64, 128};
    }
    for (std::size_t i = 1; i < values.size(); ++i)
        if (values[i] <= values[i - 1]) throw UsageError("--values must be strictly increasing");
    const std::uint64_t bytes = o.payload_mb << 20;
    const std::vector<std::uint8_t> payload = t3des::bench::make_payload(bytes, o.seed);
    const auto ts = t3des::triple_schedule(t3des::parse_hex_key("133457799BBCDFF10E329232EA6D0D737CA110454A1A6E57"));
    std::uint64_t sub48[48];
    std::memcpy(sub48, ts.pass1.data(), 128);
    std::memcpy(sub48 + 16, ts.pass2.data(), 128);
    std::memcpy(sub48 + 32, ts.pass3.data(), 128);
    std::vector<std::uint8_t> first_ct, out(bytes), back(bytes);
    std::vector<BenchRecord> recs;
    for (std::size_t v : values) {
        BenchRecord r;
        r.backend = t3des::Backend::Cuda;
        r.workers = o.workers ? o.workers : 1;
        r.chunk_blocks = o.chunk_blocks;
        r.work_group = o.work_group;
        r.payload_bytes = bytes;
        if (o.sweep == "workers") r.workers = static_cast<unsigned>(v);
        if (o.sweep == "chunk") r.chunk_blocks = v;
        if (o.sweep == "workgroup") r.work_group = v;
        const std::size_t wg_arg = r.work_group;  // 0 = the kernels' own CTA-size rule
        if (r.work_group == 0) {  // report the size that rule picks (capi.cu launch_sptable / launch_bitslice)
            const std::uint64_t launch_blocks =
                r.chunk_blocks ? std::min<std::uint64_t>(r.chunk_blocks, bytes / 8) : bytes / 8;
            int sms = 148;
            if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, o.device) != cudaSuccess) sms = 148;
            const std::uint64_t per_sm = (launch_blocks + sms - 1) / std::uint64_t(sms);
            r.work_group = o.variant == "sptable" ? (per_sm >= 1024 ? 1024 : std::max<std::uint64_t>(128, (per_sm + 31) / 32 * 32))
                                          : 128;
        }
        try {
            double best = 0;
            if (o.mode == "device" && r.workers == 1) {
                t3des_cu_ctx* c = nullptr;
                int rc = t3des_cu_create(o.device, &c);
                if (rc) throw std::runtime_error(t3des_cu_strerror(rc));
                // buffers and timing events on the context's device (not the
                // current one): the kernels run there
                int prev_dev = 0;
                cudaGetDevice(&prev_dev);
                void *din = nullptr, *dout = nullptr;
                cudaEvent_t e0 = nullptr, e1 = nullptr;
                auto ck = [&](cudaError_t e) {
                    if (e != cudaSuccess && !rc) rc = T3DES_CU_ERR_CUDA;
                    return rc == 0;
                };
                if (ck(cudaSetDevice(o.device)) && ck(cudaMalloc(&din, bytes)) && ck(cudaMalloc(&dout, bytes)) &&
                    ck(cudaMemcpy(din, payload.data(), bytes, cudaMemcpyHostToDevice)) && ck(cudaEventCreate(&e0)) &&
                    ck(cudaEventCreate(&e1))) {
                    rc = t3des_cu_set_schedule(c, sub48);
                    if (!rc) rc = t3des_cu_set_variant(c, make_config(o).variant);
                    if (!rc) rc = t3des_cu_set_launch(c, r.chunk_blocks, static_cast<int>(wg_arg));
                }
                for (unsigned rep = 0; rep <= o.reps && !rc; ++rep) {  // rep 0 = warm-up
                    ck(cudaEventRecord(e0, nullptr));
                    if (!rc) rc = t3des_cu_ecb_device(c, T3DES_CU_ENCRYPT, din, dout, bytes, nullptr);
                    ck(cudaEventRecord(e1, nullptr));
                    ck(cudaEventSynchronize(e1));
                    float ms = 0;
                    ck(cudaEventElapsedTime(&ms, e0, e1));
                    if (rep > 0 && (rep == 1 || ms * 1e-3 < best)) best = ms * 1e-3;
                }
                if (!rc) ck(cudaMemcpy(out.data(), dout, bytes, cudaMemcpyDeviceToHost));
                if (e0) cudaEventDestroy(e0);
                if (e1) cudaEventDestroy(e1);
                if (din) cudaFree(din);
                if (dout) cudaFree(dout);
                (void)cudaGetLastError();
                cudaSetDevice(prev_dev);
                t3des_cu_destroy(c);
                if (rc) throw std::runtime_error(t3des_cu_strerror(rc));
            } else {
                t3des::DispatchConfig cfg = make_config(o);
                cfg.workers = r.workers;
                cfg.chunk_blocks = r.chunk_blocks;
                cfg.work_group = wg_arg;
                cfg.gpu_chunked = true;
                for (unsigned rep = 0; rep <= o.reps; ++rep) {
                    const auto t0 = std::chrono::steady_clock::now();
                    t3des::encrypt_batch(payload, out, ts, cfg);
                    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                    if (rep > 0 && (rep == 1 || s < best)) best = s;
                }
            }
            // every record must decrypt back and agree with the first record
            t3des::DispatchConfig chk;
            chk.device = o.device;
            t3des::decrypt_batch(out, back, ts, chk);
            if (back != payload) throw std::runtime_error("round trip mismatch");
            if (first_ct.empty()) first_ct = out;
            else if (out != first_ct) throw std::runtime_error("launch-shape dependence");
            r.compute_seconds = best;
            r.throughput_mb_s = static_cast<double>(bytes) / best / (1 << 20);
        } catch (const std::exception& e) {
            std::cerr << "record failed: " << e.what() << '\n';
            r.ok = false;
        }
        recs.push_back(r);
    }
    if (!recs.empty() && recs[0].ok)
        for (BenchRecord& r : recs)
            if (r.ok) r.speedup_vs_baseline = recs[0].compute_seconds / r.compute_seconds;
    const std::string rep = t3des::bench::emit_report(
        recs, o.format == "csv" ? t3des::bench::ReportFormat::Csv : t3des::bench::ReportFormat::Markdown);
    if (o.out.empty() || o.out == "-") {
        std::cout << rep;
    } else {
        std::ofstream f(o.out);
        if (!f) {
            std::cerr << "error: cannot open report file: " << o.out << '\n';
            return kExitIo;
        }
        f << rep;
    }
    for (const BenchRecord& r : recs)
        if (!r.ok) return kExitVerifyFailed;
    return 0;
}

const char* kUsage =
    "usage: t3des_b200 <encrypt|decrypt> [--key HEX | --key-file F] [input|-] [output|-] [--pkcs7]\n"
    "                  [--check-parity] [--strict-keys] [--chunk-blocks N] [--work-group N]\n"
    "                  [--workers N] [--backend cuda|scalar|threaded|noop] [--variant auto|bitslice|sptable]\n"
    "                  [--device D]\n"
    "       t3des_b200 verify [--device D]\n"
    "       t3des_b200 bench [--sweep workers|chunk|workgroup] [--values a,b,...] [--payload-mb M]\n"
    "                  [--seed S] [--reps R] [--format csv|markdown] [--out F] [--mode device|host]\n";

}  // namespace

int main(int argc, char** argv) {
    Opts o;
    try {
        o = parse(argc, argv);
    } catch (const UsageError& e) {
        if (*e.what()) std::cerr << "error: " << e.what() << '\n';
        std::cerr << kUsage;
        return (argc >= 2 && (std::strcmp(argv[1], "-h") == 0 || std::strcmp(argv[1], "--help") == 0)) ? 0
                                                                                                        : kExitUsage;
    }
    try {
        if (o.cmd == "encrypt") return run_crypt(o, true);
        if (o.cmd == "decrypt") return run_crypt(o, false);
        if (o.cmd == "verify") return run_verify(o);
        return run_bench(o);
    } catch (const t3des::KeyFormatError& e) {
        std::cerr << "error: " << e.what() << '\n';
        return kExitKeyFormat;
    } catch (const t3des::PaddingError& e) {
        std::cerr << "error: " << e.what() << '\n';
        return kExitPadding;
    } catch (const t3des::InputLengthError& e) {
        std::cerr << "error: " << e.what() << '\n';
        return kExitInputLength;
    } catch (const t3des::IoError& e) {
        std::cerr << "error: " << e.what() << " at byte offset " << e.byte_offset << '\n';
        return kExitIo;
    } catch (const ParityError& e) {
        std::cerr << "error: " << e.what() << '\n';
        return kExitParity;
    } catch (const UsageError& e) {
        std::cerr << "error: " << e.what() << '\n';
        return kExitUsage;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return kExitUsage;
    }
}
