// polar_api.cu -- the C ABI of libpolar.so (include/polar.h).
//
// Hot path: polar_decode_f32 / polar_decode_i8 launch the decoder specialised at build time
// for the handle's code (registry.hpp) on the caller's stream.  Everything else here is
// non-hot: handle creation, GA construction, the systematic encoder, the BPSK-AWGN frame
// generator, error counting and the host-buffer end-to-end path.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <chrono>
#include <mutex>
#include <string>
#include <vector>

#include <dlfcn.h>
#include <unistd.h>
#include <sys/stat.h>

#include <fstream>
#include <map>
#include <memory>
#include <sstream>

#include "../../include/polar.h"
#include "jit.hpp"
#include "registry.hpp"
#include "tree.hpp"

namespace polar {
void construct_ga(int N, int K, double design_ebn0_db, uint8_t* frozen);
}
// generic.cu: the program-interpreted decoder for frozen sets without a specialised kernel
const void* polar_generic_kernel(bool i8);
int polar_generic_smem(bool i8, int N, int K);
// ... and its long-code form (N > 32768): one CTA per frame, large stages in a global slot
const void* polar_generic_big_kernel(bool i8);
int polar_generic_big_smem(bool i8, int N);
long long polar_generic_big_gslot_bytes(bool i8, int N);
int polar_generic_big_threads();
constexpr uint32_t kMaxUnrolledN = 32768;  // registry and run-time specialisation
constexpr uint32_t kMaxN = 1u << 20;       // program-interpreted decoder

using namespace polar;

// ------------------------------------------------------------------------- errors

static thread_local std::string g_last_error;

static polar_status fail(polar_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return s;
}

#define CUDA_TRY(expr)                                                                    \
    do {                                                                                  \
        cudaError_t e_ = (expr);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return fail(e_ == cudaErrorMemoryAllocation ? POLAR_ERR_OUT_OF_MEMORY : POLAR_ERR_CUDA, \
                        "%s: %s", #expr, cudaGetErrorString(e_));                         \
    } while (0)

// ------------------------------------------------------------- run-time specialisation
// An unregistered frozen set gets its unrolled decoder at create time, as the paper generates
// one per code: codegen.cpp emits the source it would have written at build time,
// NVRTC compiles the four k_frame variants for sm_100a, and the cubin is cached on disk under a
// hash of the source (POLAR_JIT_CACHE, default ~/.cache/polar_jit) and in the process.  NVRTC is
// opened at run time; without it, with POLAR_JIT=0 or on a compile error the code keeps the
// generic program-interpreted decoder (same results, lower throughput).

namespace {

struct Nvrtc {
    typedef int (*CreateFn)(void**, const char*, const char*, int, const char* const*, const char* const*);
    typedef int (*CompileFn)(void*, int, const char* const*);
    typedef int (*SizeFn)(void*, size_t*);
    typedef int (*GetFn)(void*, char*);
    typedef int (*NameFn)(void*, const char*);
    typedef int (*LoweredFn)(void*, const char*, const char**);
    typedef int (*DestroyFn)(void**);
    void* so = nullptr;
    CreateFn create = nullptr;
    CompileFn compile = nullptr;
    SizeFn log_size = nullptr, cubin_size = nullptr;
    GetFn log = nullptr, cubin = nullptr;
    NameFn add_name = nullptr;
    LoweredFn lowered = nullptr;
    DestroyFn destroy = nullptr;
    bool ok() const { return create && compile && log_size && cubin_size && log && cubin && add_name && lowered && destroy; }
};

const Nvrtc& nvrtc() {
    static Nvrtc n = [] {
        Nvrtc r;
        const char* names[] = {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"};
        for (const char* nm : names)
            if ((r.so = dlopen(nm, RTLD_NOW | RTLD_LOCAL))) break;
        if (!r.so) return r;
        r.create = (Nvrtc::CreateFn)dlsym(r.so, "nvrtcCreateProgram");
        r.compile = (Nvrtc::CompileFn)dlsym(r.so, "nvrtcCompileProgram");
        r.log_size = (Nvrtc::SizeFn)dlsym(r.so, "nvrtcGetProgramLogSize");
        r.cubin_size = (Nvrtc::SizeFn)dlsym(r.so, "nvrtcGetCUBINSize");
        r.log = (Nvrtc::GetFn)dlsym(r.so, "nvrtcGetProgramLog");
        r.cubin = (Nvrtc::GetFn)dlsym(r.so, "nvrtcGetCUBIN");
        r.add_name = (Nvrtc::NameFn)dlsym(r.so, "nvrtcAddNameExpression");
        r.lowered = (Nvrtc::LoweredFn)dlsym(r.so, "nvrtcGetLoweredName");
        r.destroy = (Nvrtc::DestroyFn)dlsym(r.so, "nvrtcDestroyProgram");
        return r;
    }();
    return n;
}

uint64_t fnv1a(const std::string& s, uint64_t h = 1469598103934665603ull) {
    for (unsigned char c : s) h = (h ^ c) * 1099511628211ull;
    return h;
}

struct JitModule {
    cudaLibrary_t lib = nullptr;
    const void* kern[4] = {nullptr, nullptr, nullptr, nullptr};
    unsigned smem[4] = {0, 0, 0, 0};
    const void* none = nullptr;
    unsigned zero = 0;
    std::vector<uint8_t> mask;
    std::string schedule;
    RegistryEntry entry{};
    ~JitModule() {
        if (lib) cudaLibraryUnload(lib);
    }
};

std::mutex g_jit_mu;
std::map<std::pair<uint64_t, std::vector<uint8_t>>, std::weak_ptr<JitModule>> g_jit_cache;

std::string jit_cache_dir() {
    if (const char* d = std::getenv("POLAR_JIT_CACHE")) return d;
    const char* home = std::getenv("HOME");
    return std::string(home ? home : "/tmp") + "/.cache/polar_jit";
}

// Compile (or load from the disk cache) the unrolled decoder of an unregistered code.
std::shared_ptr<JitModule> jit_build(uint32_t N, uint32_t K, const std::vector<uint8_t>& mask, std::string* why,
                                     bool load = true) {
    std::lock_guard<std::mutex> lock(g_jit_mu);
    const auto key = std::make_pair(code_hash((int)N, (int)K, mask.data()), mask);
    if (auto m = g_jit_cache[key].lock()) return m;
    JitCode jc;
    if (!codegen_jit((int)N, (int)K, mask.data(), &jc, why)) return nullptr;
    std::string cuda_inc = "-I/usr/local/cuda/include";
    if (const char* ch = std::getenv("CUDA_HOME")) cuda_inc = std::string("-I") + ch + "/include";
    const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo", cuda_inc.c_str()};
    uint64_t h = fnv1a(jc.source);
    for (int i = 0; i < kJitHeaderCount; ++i) h = fnv1a(kJitHeaderText[i], h);
    for (const char* o : opts) h = fnv1a(o, h);
    char tag[64];
    snprintf(tag, sizeof tag, "polar_%u_%u_%016llx", N, K, (unsigned long long)h);
    const std::string dir = jit_cache_dir(), base = dir + "/" + tag;
    std::string cubin;
    std::vector<std::string> lowered(4);
    if (std::getenv("POLAR_JIT_NO_CACHE")) {
    } else {  // disk cache: <base>.cubin + <base>.names (the four lowered kernel names)
        std::ifstream fc(base + ".cubin", std::ios::binary), fn(base + ".names");
        if (fc && fn) {
            cubin.assign(std::istreambuf_iterator<char>(fc), std::istreambuf_iterator<char>());
            for (auto& l : lowered) std::getline(fn, l);
            if (lowered[3].empty()) cubin.clear();
        }
    }
    if (cubin.empty()) {
        const Nvrtc& nv = nvrtc();
        if (!nv.ok()) {
            if (why) *why = "NVRTC (libnvrtc.so.12) not found";
            return nullptr;
        }
        void* prog = nullptr;
        if (nv.create(&prog, jc.source.c_str(), "polar_jit.cu", kJitHeaderCount, kJitHeaderText, kJitHeaderNames) != 0) {
            if (why) *why = "nvrtcCreateProgram failed";
            return nullptr;
        }
        for (auto& v : jc.vars) nv.add_name(prog, v.kernel.c_str());
        const int rc = nv.compile(prog, 4, opts);
        if (rc != 0) {
            size_t n = 0;
            nv.log_size(prog, &n);
            std::string log(n, '\0');
            nv.log(prog, &log[0]);
            if (why) *why = "NVRTC compile failed: " + log.substr(0, 2000);
            nv.destroy(&prog);
            return nullptr;
        }
        for (int i = 0; i < 4; ++i) {
            const char* ln = nullptr;
            nv.lowered(prog, jc.vars[i].kernel.c_str(), &ln);
            lowered[i] = ln ? ln : "";
        }
        size_t n = 0;
        nv.cubin_size(prog, &n);
        cubin.assign(n, '\0');
        nv.cubin(prog, &cubin[0]);
        nv.destroy(&prog);
        mkdir((dir.substr(0, dir.rfind('/'))).c_str(), 0755);
        mkdir(dir.c_str(), 0755);
        const std::string tmp = base + ".tmp" + std::to_string((long long)getpid());
        {
            std::ofstream fc(tmp + ".cubin", std::ios::binary), fn(tmp + ".names");
            fc.write(cubin.data(), (std::streamsize)cubin.size());
            for (auto& l : lowered) fn << l << "\n";
        }
        std::rename((tmp + ".names").c_str(), (base + ".names").c_str());
        std::rename((tmp + ".cubin").c_str(), (base + ".cubin").c_str());
    }
    if (why && why->empty()) *why = "compiled " + std::string(tag);
    if (!load) return nullptr;
    auto m = std::make_shared<JitModule>();
    if (cudaLibraryLoadData(&m->lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) != cudaSuccess) {
        cudaGetLastError();
        if (why) *why = "cudaLibraryLoadData failed";
        return nullptr;
    }
    for (int i = 0; i < 4; ++i) {
        cudaKernel_t k = nullptr;
        if (cudaLibraryGetKernel(&k, m->lib, lowered[i].c_str()) != cudaSuccess) {
            cudaGetLastError();
            if (why) *why = "kernel " + lowered[i] + " not in the JIT library";
            return nullptr;
        }
        m->kern[i] = (const void*)k;
    }
    void* dsm = nullptr;
    size_t bytes = 0;
    if (cudaLibraryGetGlobal(&dsm, &bytes, m->lib, "polar_jit_smem") != cudaSuccess || bytes != sizeof m->smem ||
        cudaMemcpy(m->smem, dsm, sizeof m->smem, cudaMemcpyDeviceToHost) != cudaSuccess) {
        cudaGetLastError();
        if (why) *why = "polar_jit_smem not readable";
        return nullptr;
    }
    m->mask = mask;
    m->schedule = jc.schedule;
    RegistryEntry& e = m->entry;
    e.name = "jit";
    e.N = N;
    e.K = K;
    e.mask = m->mask.data();
    e.hash = key.first;
    e.n_ops = jc.n_ops;
    e.warp_root = jc.warp_root;
    Variant* vs[4] = {&e.tp_f32, &e.tp_i8, &e.lat_f32, &e.lat_i8};
    for (int i = 0; i < 4; ++i)
        *vs[i] = Variant{&m->kern[i], &m->smem[i], jc.vars[i].threads, jc.vars[i].frames, jc.vars[i].gscratch, jc.vars[i].extra};
    e.xf_i8 = Variant{&m->none, &m->zero, 32, 1, 0, 0};  // no frame-interleaved kernel
    e.xf_gslot = &m->zero;
    e.mbox_i8 = Variant{nullptr, nullptr, 0, 0, 0, 0};
    e.schedule = m->schedule.c_str();
    g_jit_cache[key] = m;
    return m;
}

}  // namespace

// ------------------------------------------------------------------------- handle

struct polar_code {
    uint32_t N = 0, K = 0;
    std::vector<uint8_t> mask;
    const RegistryEntry* entry = nullptr;  // specialised decoder, or nullptr: generic
    std::shared_ptr<JitModule> jit;         // run-time specialised decoder (entry points into it)
    std::string jit_note;                   // why an unregistered code kept the generic decoder
    std::vector<uint32_t> prog;             // generic decoder: the op program (tree.hpp)
    std::string sched;                      // Listing-1 op list
    uint32_t* d_prog = nullptr;
    int occ_generic[2] = {0, 0};  // resident CTAs per SM of the generic decoder (f32, int8)
    uint32_t n_ops = 0;
    bool systematic_ok = false;  // information set closed under bit-superset (reading C4)
    // device side (absent when no usable device at create time)
    bool dev_ready = false;
    int device = -1;
    int n_sm = 0;
    int occ[5] = {0, 0, 0, 0, 0};  // resident CTAs per SM: tp_f32, tp_i8, lat_f32, lat_i8, xf_i8
    int variant = 0;              // 0 auto, 1 throughput, 2 latency, 3 generic, 4 frame-interleaved
    unsigned flags = 0;           // kernel flags: bit 0 = non-systematic output (polar_code_set_output)
    uint32_t* d_pos = nullptr;    // K information positions, ascending (encoder / generator)
    uint32_t* d_gtab = nullptr;   // gather table: info mask words, then info-bit prefix per word
    // per variant global stage scratch: tp_f32, tp_i8, lat_f32, lat_i8, xf_i8, long-code generic
    void* d_gscratch[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    size_t sc_bytes[6] = {0, 0, 0, 0, 0, 0};  // its size (0: the variant needs none)
    // Launches of one variant share its scratch slots: a launch on another stream waits for the
    // previous one (event), so concurrent decode calls on one handle stay correct.
    std::mutex sc_mu;
    cudaEvent_t sc_ev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    cudaStream_t sc_last[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    bool sc_used[6] = {false, false, false, false, false, false};
    unsigned long long* d_trace = nullptr;  // POLAR_TRACE builds: per-op clock64 of the latency variant
    float* d_dump = nullptr;                // POLAR_DEBUG_DUMP builds: alpha stages of up to kDumpFrames frames
    uint32_t* d_info_mask = nullptr;  // N/32 words (>= 1), bit set = information position
    // host-buffer path (lazily allocated, guarded by mu)
    std::mutex mu;
    cudaStream_t streams[2] = {nullptr, nullptr};
    void* d_stage_llr[2] = {nullptr, nullptr};
    uint32_t* d_stage_out[2] = {nullptr, nullptr};
    int64_t stage_frames = 0;
    size_t stage_elem = 0;
    // batch-1 mailbox (polar_mailbox_*): host-mapped control word, frame and output
    struct {
        bool open = false;
        void* ctl = nullptr;       // pd::MailboxCtl, host-mapped pinned
        int8_t* hframe = nullptr;  // N bytes, host-mapped pinned
        uint32_t* hout = nullptr;  // ceil(K/32) words, host-mapped pinned
        int8_t* dbuf = nullptr;    // N bytes of device memory
        cudaStream_t s = nullptr;
        unsigned int seq = 0;
    } mb;
};

static inline uint32_t words_of(uint32_t bits) { return (bits + 31) / 32; }

// Must match kernels.cuh: SCRATCH_HDR bytes at the start of a throughput variant's global
// scratch hold its frame-group counter (POLAR_DYN scheduling).
#ifndef POLAR_DYN
#define POLAR_DYN 1
#endif
constexpr size_t kScratchHdr = 256;
// POLAR_DEBUG_DUMP: frames per dumped decode and floats per frame (decoder.cuh dump_stride)
constexpr int64_t kDumpFrames = 8;
static uint64_t dump_stride(uint32_t N) {
    uint32_t l = 0;
    while ((1u << l) < N) ++l;
    return (uint64_t)N * (l > 0 ? l : 1);
}

extern "C" const char* polar_status_string(polar_status s) {
    switch (s) {
        case POLAR_OK: return "ok";
        case POLAR_ERR_INVALID_ARGUMENT: return "invalid argument";
        case POLAR_ERR_UNSUPPORTED_CODE: return "unsupported code (no specialised decoder)";
        case POLAR_ERR_CUDA: return "CUDA error";
        case POLAR_ERR_OUT_OF_MEMORY: return "out of memory";
    }
    return "unknown status";
}

extern "C" const char* polar_last_error(void) { return g_last_error.c_str(); }

static polar_status init_device(polar_code* h) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        return POLAR_OK;  // host-only handle; decode calls will report POLAR_ERR_CUDA
    }
    CUDA_TRY(cudaGetDevice(&h->device));
    CUDA_TRY(cudaDeviceGetAttribute(&h->n_sm, cudaDevAttrMultiProcessorCount, h->device));
    const RegistryEntry* e = h->entry;
    {  // generic decoder (any code): one warp per frame, all stages in shared memory; for
       // N > 32768 one CTA per frame with the large stages in a global slot (allocated lazily)
        const bool big = h->N > kMaxUnrolledN;
        for (int i = 0; i < 2; ++i) {
            const void* k = big ? polar_generic_big_kernel(i == 1) : polar_generic_kernel(i == 1);
            const int sm = big ? polar_generic_big_smem(i == 1, (int)h->N) : polar_generic_smem(i == 1, (int)h->N, (int)h->K);
            CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
            CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&h->occ_generic[i], k, big ? polar_generic_big_threads() : 32, sm));
            if (h->occ_generic[i] < 1) return fail(POLAR_ERR_CUDA, "generic decoder cannot be resident");
        }
        if (big) {
            h->sc_bytes[5] = (size_t)std::max(h->occ_generic[0], h->occ_generic[1]) * h->n_sm *
                             (size_t)polar_generic_big_gslot_bytes(false, (int)h->N);
            CUDA_TRY(cudaEventCreateWithFlags(&h->sc_ev[5], cudaEventDisableTiming));
        }
        CUDA_TRY(cudaMalloc(&h->d_prog, std::max<size_t>(1, h->prog.size()) * sizeof(uint32_t)));
        CUDA_TRY(cudaMemcpy(h->d_prog, h->prog.data(), h->prog.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
    }
    const Variant* vs[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    if (e) {
        vs[0] = &e->tp_f32;
        vs[1] = &e->tp_i8;
        vs[2] = &e->lat_f32;
        vs[3] = &e->lat_i8;
        vs[4] = &e->xf_i8;
    }
    for (int i = 0; i < (e ? 5 : 0); ++i) {
        const void* k = *vs[i]->kern;
        if (!k) continue;  // a run-time specialised code has no frame-interleaved kernel
        CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)*vs[i]->smem));
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &h->occ[i], k, (int)(vs[i]->threads * vs[i]->frames + vs[i]->extra), *vs[i]->smem));
        if (h->occ[i] < 1) return fail(POLAR_ERR_CUDA, "decoder kernel variant %d cannot be resident", i);
        // one slot per resident frame group (xf: per warp) of the persistent grid, after the
        // counter header (always present for the xf variant).  The frame-interleaved scratch
        // (~1.2 GB at N = 32768, where auto never selects it) is allocated on its first launch.
        h->sc_bytes[i] = 0;
        const size_t slot = i == 4 ? *e->xf_gslot : vs[i]->gscratch;
        if (slot || i == 4)
            h->sc_bytes[i] = (size_t)h->occ[i] * h->n_sm * vs[i]->frames * slot + (i < 2 || i == 4 ? kScratchHdr : 0);
        if (h->sc_bytes[i] && i != 4) CUDA_TRY(cudaMalloc(&h->d_gscratch[i], h->sc_bytes[i]));
        if (h->sc_bytes[i]) CUDA_TRY(cudaEventCreateWithFlags(&h->sc_ev[i], cudaEventDisableTiming));
    }
    std::vector<uint32_t> pos;
    std::vector<uint32_t> im(std::max<uint32_t>(1, h->N / 32), 0);
    for (uint32_t i = 0; i < h->N; ++i)
        if (!h->mask[i]) {
            pos.push_back(i);
            im[i / 32] |= 1u << (i % 32);
        }
    CUDA_TRY(cudaMalloc(&h->d_pos, pos.size() * sizeof(uint32_t)));
    CUDA_TRY(cudaMemcpy(h->d_pos, pos.data(), pos.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
    std::vector<uint32_t> gt(im);
    uint32_t acc = 0;
    for (uint32_t w : im) {
        gt.push_back(acc);
        acc += (uint32_t)__builtin_popcount(w);
    }
    // Piece table of the gather (decoder.cuh gather_info, generic.cu): output word q of x_hat[A]
    // is the OR of its pieces -- maximal runs of consecutive information positions inside one
    // output word -- each a uint2 {lo << 16 | (hi - lo) << 5 | s, destination mask}: the run's
    // source bits are bits s.. of the pair (beta[hi] : beta[lo]) (a run starting at bit a of word
    // lo lands at output bit d: s = (a - d) mod 32; hi = lo + 1 when it crosses into the next
    // word, which implies a > d).  Output words go in groups of 32 (one per lane); group g owns
    // rows hdr[g] .. hdr[g+1]-1, as many as its longest word rounded up to even, and piece j of
    // word 32g + l is element l of row hdr[g] + j (padding: {0, 0}).  Layout after the two
    // tables above: hdr[NG + 1] padded to 4 words (gather_hdr_words), then the rows.
    {
        const uint32_t nwk = words_of(h->K), ng = (nwk + 31) / 32;
        std::vector<std::vector<std::pair<uint32_t, uint32_t>>> pw(nwk);
        for (uint32_t j = 0; j < (uint32_t)pos.size();) {
            const uint32_t q = j / 32, src = pos[j];
            uint32_t len = 1;
            while (j + len < (uint32_t)pos.size() && (j + len) / 32 == q && pos[j + len] == src + len) ++len;
            const uint32_t d = j % 32, a = src % 32, lo = src / 32, cross = a + len > 32 ? 1u : 0u;
            const uint32_t m = (len >= 32 ? 0xffffffffu : ((1u << len) - 1u)) << d;
            pw[q].push_back({(lo << 16) | (cross << 5) | ((a - d) & 31u), m});
            j += len;
        }
        std::vector<uint32_t> hdr(ng + 1, 0);
        for (uint32_t g = 0; g < ng; ++g) {
            size_t mx = 0;
            for (uint32_t q = 32 * g; q < std::min(nwk, 32 * g + 32); ++q) mx = std::max(mx, pw[q].size());
            hdr[g + 1] = hdr[g] + (uint32_t)((mx + 1) & ~(size_t)1);
        }
        while (hdr.size() % 4) hdr.push_back(0);
        while (gt.size() % 4) gt.push_back(0);
        gt.insert(gt.end(), hdr.begin(), hdr.end());
        const size_t base = gt.size();
        gt.resize(base + 2 * 32 * (size_t)hdr[ng], 0u);
        for (uint32_t q = 0; q < nwk; ++q)
            for (size_t jj = 0; jj < pw[q].size(); ++jj) {
                const size_t at = base + 2 * ((size_t)(hdr[q / 32] + jj) * 32 + q % 32);
                gt[at] = pw[q][jj].first;
                gt[at + 1] = pw[q][jj].second;
            }
    }
    CUDA_TRY(cudaMalloc(&h->d_gtab, gt.size() * sizeof(uint32_t)));
    CUDA_TRY(cudaMemcpy(h->d_gtab, gt.data(), gt.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMalloc(&h->d_info_mask, im.size() * sizeof(uint32_t)));
    CUDA_TRY(cudaMemcpy(h->d_info_mask, im.data(), im.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
#ifdef POLAR_DEBUG_DUMP
    CUDA_TRY(cudaMalloc(&h->d_dump, kDumpFrames * dump_stride(h->N) * sizeof(float)));
#endif
#ifdef POLAR_TRACE
    CUDA_TRY(cudaMalloc(&h->d_trace, 65536 * sizeof(unsigned long long)));
    CUDA_TRY(cudaMemset(h->d_trace, 0, 65536 * sizeof(unsigned long long)));
#endif
    h->dev_ready = true;
    return POLAR_OK;
}

extern "C" polar_status polar_code_create(uint32_t N, uint32_t K, const uint8_t* frozen_mask, polar_code** out) {
    if (!out || !frozen_mask) return fail(POLAR_ERR_INVALID_ARGUMENT, "null pointer");
    *out = nullptr;
    if (N < 2 || N > kMaxN || (N & (N - 1))) return fail(POLAR_ERR_INVALID_ARGUMENT, "N=%u is not a power of two in [2, 2^20]", N);
    if (K < 1 || K > N) return fail(POLAR_ERR_INVALID_ARGUMENT, "K=%u not in [1, N]", K);
    std::vector<uint8_t> m(frozen_mask, frozen_mask + N);
    uint32_t nf = 0;
    for (auto& b : m) {
        b = b ? 1 : 0;
        nf += b;
    }
    if (nf != N - K) return fail(POLAR_ERR_INVALID_ARGUMENT, "mask has %u frozen bits, expected N-K=%u", nf, N - K);
    const uint64_t hsh = code_hash((int)N, (int)K, m.data());
    const RegistryEntry* e = nullptr;
    for (uint32_t i = 0; i < (N <= kMaxUnrolledN ? kRegistrySize : 0); ++i)
        if (kRegistry[i].hash == hsh && kRegistry[i].N == N && kRegistry[i].K == K &&
            std::memcmp(kRegistry[i].mask, m.data(), N) == 0)
            e = &kRegistry[i];
    polar_code* h = new polar_code;
    h->N = N;
    h->K = K;
    // POLAR_JIT_FORCE=1: ignore the build-time decoder (measures the run-time path on a code
    // that has both)
    if (const char* f = std::getenv("POLAR_JIT_FORCE"); f && f[0] == '1') e = nullptr;
    if (!e) {  // no build-time decoder: specialise at run time (needs a device and NVRTC)
        const char* env = std::getenv("POLAR_JIT");
        const char* mx = std::getenv("POLAR_JIT_MAX_OPS");
        const uint32_t max_ops = mx ? (uint32_t)std::strtoul(mx, nullptr, 10) : 4096u;
        const uint32_t ops_fast = (uint32_t)schedule(build_tree((int)N, m.data())).size();
        int count = 0;
        if (env && env[0] == '0') h->jit_note = "POLAR_JIT=0";
        else if (N > kMaxUnrolledN) h->jit_note = "N > 32768: program-interpreted (P:1277)";
        else if (ops_fast > max_ops)  // compile time grows with the unrolled length
            h->jit_note = std::to_string(ops_fast) + " Fast-SSC ops > POLAR_JIT_MAX_OPS=" + std::to_string(max_ops);
        else if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
            cudaGetLastError();
            h->jit_note = "no CUDA device";
        } else if ((h->jit = jit_build(N, K, m, &h->jit_note))) {
            e = &h->jit->entry;
        }
    }
    h->mask = std::move(m);
    h->entry = e;  // nullptr: no specialised decoder, the generic (interpreted) one is used
    const Tree tree = build_tree((int)N, h->mask.data());
    const std::vector<std::string> ops = schedule(tree);
    h->n_ops = (uint32_t)ops.size();
    for (auto& o : ops) h->sched += o + ";";
    if (e) {  // the specialised decoder's own op list (a build may use another node set, tree.hpp NodeSet)
        h->n_ops = e->n_ops;
        h->sched = e->schedule;
    }
    h->prog = program(tree);  // the generic decoder serves unregistered codes and variant 3
    h->systematic_ok = superset_closed((int)N, h->mask.data());
    polar_status s = init_device(h);
    if (s != POLAR_OK) {
        polar_code_destroy(h);
        return s;
    }
    *out = h;
    return POLAR_OK;
}

extern "C" void polar_code_destroy(polar_code* h) {
    if (!h) return;
    if (h->mb.open) polar_mailbox_close(h);
    // every resource that exists is released, also after a partial init_device (cudaFree(nullptr)
    // is a no-op; the pointers start null)
    if (h->d_trace) cudaFree(h->d_trace);
    if (h->d_dump) cudaFree(h->d_dump);
    if (h->d_prog) cudaFree(h->d_prog);
    if (h->d_pos) cudaFree(h->d_pos);
    if (h->d_info_mask) cudaFree(h->d_info_mask);
    if (h->d_gtab) cudaFree(h->d_gtab);
    for (int i = 0; i < 6; ++i) {
        if (h->d_gscratch[i]) cudaFree(h->d_gscratch[i]);
        if (h->sc_ev[i]) cudaEventDestroy(h->sc_ev[i]);
    }
    for (int i = 0; i < 2; ++i) {
        if (h->d_stage_llr[i]) cudaFree(h->d_stage_llr[i]);
        if (h->d_stage_out[i]) cudaFree(h->d_stage_out[i]);
        if (h->streams[i]) cudaStreamDestroy(h->streams[i]);
    }
    delete h;
}

extern "C" polar_status polar_jit_compile(uint32_t N, uint32_t K, const uint8_t* frozen_mask, char* log, uint32_t cap) {
    if (!frozen_mask) return fail(POLAR_ERR_INVALID_ARGUMENT, "null mask");
    if (N < 2 || N > 32768 || (N & (N - 1)) || K < 1 || K > N) return fail(POLAR_ERR_INVALID_ARGUMENT, "bad (N, K)");
    std::vector<uint8_t> m(frozen_mask, frozen_mask + N);
    for (auto& b : m) b = b ? 1 : 0;
    std::string why;
    jit_build(N, K, m, &why, false);
    if (log && cap) {
        std::strncpy(log, why.c_str(), cap - 1);
        log[cap - 1] = 0;
    }
    return why.rfind("compiled ", 0) == 0 ? POLAR_OK : fail(POLAR_ERR_UNSUPPORTED_CODE, "%s", why.substr(0, 400).c_str());
}

extern "C" polar_status polar_code_query(const polar_code* h, uint32_t* N, uint32_t* K, uint32_t* n_ops,
                                         uint32_t* smem_bytes, uint32_t* warp_root) {
    if (!h) return fail(POLAR_ERR_INVALID_ARGUMENT, "null handle");
    if (N) *N = h->N;
    if (K) *K = h->K;
    if (n_ops) *n_ops = h->n_ops;
    if (smem_bytes) *smem_bytes = h->entry ? *h->entry->tp_i8.smem : (uint32_t)polar_generic_smem(true, (int)h->N, (int)h->K);
    if (warp_root) *warp_root = h->entry ? h->entry->warp_root : 0;
    return POLAR_OK;
}

extern "C" polar_status polar_code_is_specialised(const polar_code* h, int* specialised) {
    if (!h || !specialised) return fail(POLAR_ERR_INVALID_ARGUMENT, "null pointer");
    *specialised = h->jit ? 2 : h->entry != nullptr ? 1 : 0;
    if (!h->entry && !h->jit_note.empty()) g_last_error = "generic decoder: " + h->jit_note;
    return POLAR_OK;
}

extern "C" polar_status polar_code_set_variant(polar_code* h, int variant) {
    if (!h || variant < 0 || variant > 4) return fail(POLAR_ERR_INVALID_ARGUMENT, "variant must be 0, 1, 2, 3 or 4");
    h->variant = variant;
    return POLAR_OK;
}

extern "C" polar_status polar_code_set_output(polar_code* h, int mode) {
    if (!h || (mode != POLAR_OUTPUT_SYSTEMATIC && mode != POLAR_OUTPUT_NONSYSTEMATIC))
        return fail(POLAR_ERR_INVALID_ARGUMENT, "output mode must be POLAR_OUTPUT_SYSTEMATIC or POLAR_OUTPUT_NONSYSTEMATIC");
    h->flags = mode == POLAR_OUTPUT_NONSYSTEMATIC ? 1u : 0u;
    return POLAR_OK;
}

extern "C" polar_status polar_code_mask(const polar_code* h, uint8_t* mask_out) {
    if (!h || !mask_out) return fail(POLAR_ERR_INVALID_ARGUMENT, "null pointer");
    std::memcpy(mask_out, h->mask.data(), h->N);
    return POLAR_OK;
}

extern "C" polar_status polar_code_schedule(const polar_code* h, char* buf, uint32_t cap, uint32_t* needed) {
    if (!h) return fail(POLAR_ERR_INVALID_ARGUMENT, "null handle");
    const char* s = h->sched.c_str();
    const uint32_t len = (uint32_t)std::strlen(s);
    if (needed) *needed = len + 1;
    if (buf && cap) {
        const uint32_t n = std::min(len, cap - 1);
        std::memcpy(buf, s, n);
        buf[n] = 0;
    }
    return POLAR_OK;
}

extern "C" polar_status polar_trace_fetch(const polar_code* h, uint64_t* host, uint32_t n) {
    if (!h || !host) return fail(POLAR_ERR_INVALID_ARGUMENT, "null pointer");
#ifdef POLAR_TRACE
    if (!h->dev_ready) return fail(POLAR_ERR_CUDA, "no CUDA device");
    CUDA_TRY(cudaMemcpy(host, h->d_trace, std::min<uint32_t>(n, 65536) * 8, cudaMemcpyDeviceToHost));
    return POLAR_OK;
#else
    (void)n;
    return fail(POLAR_ERR_UNSUPPORTED_CODE, "not a POLAR_TRACE build");
#endif
}

extern "C" polar_status polar_debug_dump_stride(const polar_code* h, uint64_t* stride) {
    if (!h || !stride) return fail(POLAR_ERR_INVALID_ARGUMENT, "null pointer");
#ifdef POLAR_DEBUG_DUMP
    *stride = dump_stride(h->N);
    return POLAR_OK;
#else
    return fail(POLAR_ERR_UNSUPPORTED_CODE, "not a POLAR_DEBUG_DUMP build");
#endif
}

extern "C" polar_status polar_debug_dump_fetch(const polar_code* h, float* host, uint64_t n) {
    if (!h || !host) return fail(POLAR_ERR_INVALID_ARGUMENT, "null pointer");
#ifdef POLAR_DEBUG_DUMP
    if (!h->dev_ready) return fail(POLAR_ERR_CUDA, "no CUDA device");
    if (n > (uint64_t)kDumpFrames * dump_stride(h->N)) return fail(POLAR_ERR_INVALID_ARGUMENT, "n exceeds the dump");
    CUDA_TRY(cudaMemcpy(host, h->d_dump, n * sizeof(float), cudaMemcpyDeviceToHost));
    return POLAR_OK;
#else
    (void)n;
    return fail(POLAR_ERR_UNSUPPORTED_CODE, "not a POLAR_DEBUG_DUMP build");
#endif
}

extern "C" uint32_t polar_registry_size(void) { return kRegistrySize; }

extern "C" polar_status polar_registry_entry(uint32_t i, uint32_t* N, uint32_t* K, uint8_t* mask_out) {
    if (i >= kRegistrySize) return fail(POLAR_ERR_INVALID_ARGUMENT, "registry index %u out of range", i);
    if (N) *N = kRegistry[i].N;
    if (K) *K = kRegistry[i].K;
    if (mask_out) std::memcpy(mask_out, kRegistry[i].mask, kRegistry[i].N);
    return POLAR_OK;
}

// ------------------------------------------------------------------------- decode (hot)

// Launch a kernel that uses the global scratch of variant vi, ordered after the previous
// launch of that variant when it was on another stream.  Under stream capture the ordering is
// the caller's (an event recorded outside the capture cannot be waited on inside it).
static polar_status launch_with_scratch(const polar_code* hc, int vi, const void* kern, dim3 grid, dim3 block,
                                        void** args, unsigned smem, cudaStream_t s, int scratch_arg = 4) {
    polar_code* h = const_cast<polar_code*>(hc);
    if (!h->sc_bytes[vi]) {
        CUDA_TRY(cudaLaunchKernel(kern, grid, block, args, smem, s));
        return POLAR_OK;
    }
    if (!h->d_gscratch[vi]) {  // lazily allocated scratch (frame-interleaved variant)
        std::lock_guard<std::mutex> lock(h->sc_mu);
        if (!h->d_gscratch[vi]) CUDA_TRY(cudaMalloc(&h->d_gscratch[vi], h->sc_bytes[vi]));
    }
    args[scratch_arg] = (void*)&h->d_gscratch[vi];
    // throughput variants with global stages: zero the frame-group counter (kernels.cuh DYN)
    const bool ctr = (POLAR_DYN && vi < 2) || vi == 4;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CUDA_TRY(cudaStreamIsCapturing(s, &cs));
    if (cs != cudaStreamCaptureStatusNone) {
        if (ctr) CUDA_TRY(cudaMemsetAsync(h->d_gscratch[vi], 0, sizeof(unsigned long long), s));
        CUDA_TRY(cudaLaunchKernel(kern, grid, block, args, smem, s));
        return POLAR_OK;
    }
    std::lock_guard<std::mutex> lock(h->sc_mu);
    if (h->sc_used[vi] && h->sc_last[vi] != s) CUDA_TRY(cudaStreamWaitEvent(s, h->sc_ev[vi], 0));
    if (ctr) CUDA_TRY(cudaMemsetAsync(h->d_gscratch[vi], 0, sizeof(unsigned long long), s));
    CUDA_TRY(cudaLaunchKernel(kern, grid, block, args, smem, s));
    CUDA_TRY(cudaEventRecord(h->sc_ev[vi], s));
    h->sc_last[vi] = s;
    h->sc_used[vi] = true;
    return POLAR_OK;
}

static polar_status launch_decode(const polar_code* h, bool i8, const void* llr, int64_t n, uint32_t* out,
                                  cudaStream_t s) {
    if (!h) return fail(POLAR_ERR_INVALID_ARGUMENT, "null handle");
    if (n < 0) return fail(POLAR_ERR_INVALID_ARGUMENT, "n_frames < 0");
    if (n == 0) return POLAR_OK;
    if (!llr || !out) return fail(POLAR_ERR_INVALID_ARGUMENT, "null buffer");
    if (((uintptr_t)llr & 15) != 0) return fail(POLAR_ERR_INVALID_ARGUMENT, "llr must be 16-byte aligned");
    if (((uintptr_t)out & 3) != 0) return fail(POLAR_ERR_INVALID_ARGUMENT, "info_bits must be 4-byte aligned");
    if (!h->dev_ready) return fail(POLAR_ERR_CUDA, "no CUDA device was available when the handle was created");
    const RegistryEntry* e = h->entry;
    if (!e || h->variant == 3) {  // generic decoder
        const bool big = h->N > kMaxUnrolledN;
        const void* kern = big ? polar_generic_big_kernel(i8) : polar_generic_kernel(i8);
        const int sm = big ? polar_generic_big_smem(i8, (int)h->N) : polar_generic_smem(i8, (int)h->N, (int)h->K);
        const unsigned grid = (unsigned)std::min<int64_t>(n, (int64_t)h->occ_generic[i8 ? 1 : 0] * h->n_sm);
        long long nn = (long long)n;
        const uint32_t* gtab = h->d_gtab;
        const uint32_t* prog = h->d_prog;
        int nops = (int)h->prog.size(), N = (int)h->N, K = (int)h->K;
        unsigned fl = h->flags;
        void* gslot = nullptr;
        void* args[] = {(void*)&llr, (void*)&nn, (void*)&out, (void*)&gtab, (void*)&prog, (void*)&nops, (void*)&N, (void*)&K,
                        (void*)&fl, (void*)&gslot};
        if (big) return launch_with_scratch(h, 5, kern, dim3(grid), dim3(polar_generic_big_threads()), args, sm, s, 9);
        CUDA_TRY(cudaLaunchKernel(kern, dim3(grid), dim3(32), args, sm, s));
        return POLAR_OK;
    }
    // Latency variant (a CTA per frame) for batches that cannot fill the GPU with one frame
    // per warp; otherwise the throughput variant (a warp per frame).
    // (measured crossover, profiles/r1_sweeps.md: at N >= 16384 one latency wave of #SMs
    // frames takes ~1/4 of a throughput wave)
    const int64_t lat_max = (int64_t)h->n_sm * (h->N >= 16384 ? 4 : 1);
    // Frame-interleaved variant (a lane per frame): forced by variant 4; automatic for int8
    // codes with N <= 1024 once the batch fills every SM with several 32-frame warps
    // (measured faster there only: (1024,512) 172 vs 146 Gbps; (2048,1723) 262 vs 316).
    if (h->variant == 4 && h->flags) return fail(POLAR_ERR_UNSUPPORTED_CODE, "the frame-interleaved variant has systematic output only");
    const bool has_xf = *e->xf_i8.kern != nullptr;
    if (h->variant == 4 && i8 && !has_xf) return fail(POLAR_ERR_UNSUPPORTED_CODE, "no frame-interleaved kernel for this code");
    const bool xf = i8 && has_xf && !h->flags && (h->variant == 4 || (h->variant == 0 && h->N <= 1024 && n >= (int64_t)h->n_sm * 32 * 4));
    if (xf) {  // 32 frames per warp, frames = warps per CTA
        const Variant& v = e->xf_i8;
        const int64_t groups = (n + 31) / 32;
        const int64_t resident = (int64_t)h->occ[4] * h->n_sm;
        const unsigned grid = (unsigned)std::min<int64_t>((groups + v.frames - 1) / v.frames, resident);
        long long nn = (long long)n;
        const uint32_t* gtab = h->d_gtab;
        void* gs = h->d_gscratch[4];
        void* args[] = {(void*)&llr, (void*)&nn, (void*)&out, (void*)&gtab, (void*)&gs};
        return launch_with_scratch(h, 4, *v.kern, dim3(grid), dim3(32 * v.frames), args, *v.smem, s);
    }
    const bool lat = h->variant == 2 || (h->variant == 0 && n <= lat_max);
    const int vi = (lat ? 2 : 0) + (i8 ? 1 : 0);
    const Variant& v = vi == 0 ? e->tp_f32 : vi == 1 ? e->tp_i8 : vi == 2 ? e->lat_f32 : e->lat_i8;
    const void* kern = *v.kern;
    const unsigned smem = *v.smem;
    const int64_t resident = (int64_t)h->occ[vi] * h->n_sm;
    const unsigned grid = (unsigned)std::min<int64_t>((n + v.frames - 1) / v.frames, resident);
    long long nn = (long long)n;
    const uint32_t* gtab = h->d_gtab;
    void* gs = h->d_gscratch[vi];
#ifdef POLAR_TRACE
    if (lat) gs = h->d_trace;
#endif
#ifdef POLAR_DEBUG_DUMP
    if (n > kDumpFrames) return fail(POLAR_ERR_INVALID_ARGUMENT, "POLAR_DEBUG_DUMP build: at most %d frames", (int)kDumpFrames);
    CUDA_TRY(cudaMemsetAsync(h->d_dump, 0xff, kDumpFrames * dump_stride(h->N) * sizeof(float), s));  // NaN
    float* dump = h->d_dump;
    unsigned fl = h->flags;
    void* args[] = {(void*)&llr, (void*)&nn, (void*)&out, (void*)&gtab, (void*)&gs, (void*)&fl, (void*)&dump};
#else
    unsigned fl = h->flags;
    void* args[] = {(void*)&llr, (void*)&nn, (void*)&out, (void*)&gtab, (void*)&gs, (void*)&fl};
#endif
    return launch_with_scratch(h, vi, kern, dim3(grid), dim3(v.threads * v.frames + v.extra), args, smem, s);
}

extern "C" polar_status polar_decode_f32(const polar_code* h, const float* llr, int64_t n, uint32_t* info,
                                         polar_stream stream) {
    return launch_decode(h, false, llr, n, info, (cudaStream_t)stream);
}

extern "C" polar_status polar_decode_i8(const polar_code* h, const int8_t* llr, int64_t n, uint32_t* info,
                                        polar_stream stream) {
    return launch_decode(h, true, llr, n, info, (cudaStream_t)stream);
}

// Host-buffer end-to-end path: chunks alternate over two streams so that the H2D copy of
// one chunk, the decode of another and the D2H copy of a third overlap (P:1187-1189 idea).
static polar_status decode_host(polar_code* h, bool i8, const void* host_llr, int64_t n, uint32_t* host_info) {
    if (!h) return fail(POLAR_ERR_INVALID_ARGUMENT, "null handle");
    if (n < 0) return fail(POLAR_ERR_INVALID_ARGUMENT, "n_frames < 0");
    if (n == 0) return POLAR_OK;
    if (!host_llr || !host_info) return fail(POLAR_ERR_INVALID_ARGUMENT, "null buffer");
    if (!h->dev_ready) return fail(POLAR_ERR_CUDA, "no CUDA device was available when the handle was created");
    std::lock_guard<std::mutex> lock(h->mu);
    const size_t elem = i8 ? 1 : 4;
    const size_t frame_bytes = (size_t)h->N * elem;
    const uint32_t wk = words_of(h->K);
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(n, (int64_t)((64u << 20) / frame_bytes)));
    if (h->stage_frames < chunk || h->stage_elem < elem) {
        for (int i = 0; i < 2; ++i) {
            if (h->d_stage_llr[i]) cudaFree(h->d_stage_llr[i]);
            if (h->d_stage_out[i]) cudaFree(h->d_stage_out[i]);
            h->d_stage_llr[i] = nullptr;
            h->d_stage_out[i] = nullptr;
        }
        h->stage_frames = 0;
        for (int i = 0; i < 2; ++i) {
            if (!h->streams[i]) CUDA_TRY(cudaStreamCreateWithFlags(&h->streams[i], cudaStreamNonBlocking));
            CUDA_TRY(cudaMalloc(&h->d_stage_llr[i], chunk * (size_t)h->N * 4));
            CUDA_TRY(cudaMalloc(&h->d_stage_out[i], chunk * (size_t)wk * 4));
        }
        h->stage_frames = chunk;
        h->stage_elem = 4;
    }
    for (int64_t f0 = 0, c = 0; f0 < n; f0 += chunk, ++c) {
        const int64_t m = std::min(chunk, n - f0);
        const int b = (int)(c & 1);
        cudaStream_t s = h->streams[b];
        CUDA_TRY(cudaMemcpyAsync(h->d_stage_llr[b], (const char*)host_llr + f0 * frame_bytes, m * frame_bytes,
                                 cudaMemcpyHostToDevice, s));
        polar_status st = launch_decode(h, i8, h->d_stage_llr[b], m, h->d_stage_out[b], s);
        if (st != POLAR_OK) return st;
        CUDA_TRY(cudaMemcpyAsync(host_info + f0 * wk, h->d_stage_out[b], m * (size_t)wk * 4, cudaMemcpyDeviceToHost, s));
    }
    CUDA_TRY(cudaStreamSynchronize(h->streams[0]));
    CUDA_TRY(cudaStreamSynchronize(h->streams[1]));
    return POLAR_OK;
}

extern "C" polar_status polar_decode_f32_host(polar_code* h, const float* host_llr, int64_t n, uint32_t* host_info) {
    return decode_host(h, false, host_llr, n, host_info);
}

extern "C" polar_status polar_decode_i8_host(polar_code* h, const int8_t* host_llr, int64_t n, uint32_t* host_info) {
    return decode_host(h, true, host_llr, n, host_info);
}

// ------------------------------------------------------------- batch-1 mailbox (NEXT N3)
struct MailboxCtlHost {  // layout of pd::MailboxCtl (kernels.cuh)
    unsigned int req;
    unsigned int pad0[31];
    unsigned int done;
    unsigned int pad1[31];
};

static void mailbox_free(polar_code* h) {
    if (h->mb.s) cudaStreamDestroy(h->mb.s);
    if (h->mb.ctl) cudaFreeHost(h->mb.ctl);
    if (h->mb.hframe) cudaFreeHost(h->mb.hframe);
    if (h->mb.hout) cudaFreeHost(h->mb.hout);
    if (h->mb.dbuf) cudaFree(h->mb.dbuf);
    h->mb.s = nullptr;
    h->mb.ctl = nullptr;
    h->mb.hframe = nullptr;
    h->mb.hout = nullptr;
    h->mb.dbuf = nullptr;
    h->mb.open = false;
}

extern "C" polar_status polar_mailbox_open(polar_code* h, double idle_seconds) {
    if (!h) return fail(POLAR_ERR_INVALID_ARGUMENT, "null handle");
    if (!(idle_seconds > 0.0) || idle_seconds > 3600.0) return fail(POLAR_ERR_INVALID_ARGUMENT, "idle_seconds not in (0, 3600]");
    if (!h->dev_ready) return fail(POLAR_ERR_CUDA, "no CUDA device was available when the handle was created");
    if (!h->entry || !h->entry->mbox_i8.kern) return fail(POLAR_ERR_UNSUPPORTED_CODE, "no mailbox kernel was built for this code (MAILBOX=1)");
    std::lock_guard<std::mutex> lock(h->mu);
    if (h->mb.open) return fail(POLAR_ERR_INVALID_ARGUMENT, "mailbox already open");
    const Variant& v = h->entry->mbox_i8;
    auto bail = [&](const char* what, cudaError_t e) {
        mailbox_free(h);
        cudaGetLastError();
        return fail(e == cudaErrorMemoryAllocation ? POLAR_ERR_OUT_OF_MEMORY : POLAR_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    };
    cudaError_t e;
    if ((e = cudaHostAlloc(&h->mb.ctl, sizeof(MailboxCtlHost), cudaHostAllocMapped)) != cudaSuccess) return bail("ctl", e);
    if ((e = cudaHostAlloc((void**)&h->mb.hframe, h->N, cudaHostAllocMapped)) != cudaSuccess) return bail("frame", e);
    if ((e = cudaHostAlloc((void**)&h->mb.hout, words_of(h->K) * 4, cudaHostAllocMapped)) != cudaSuccess) return bail("out", e);
    if ((e = cudaMalloc((void**)&h->mb.dbuf, h->N)) != cudaSuccess) return bail("dbuf", e);
    std::memset(h->mb.ctl, 0, sizeof(MailboxCtlHost));
    h->mb.seq = 0;
    if ((e = cudaStreamCreateWithFlags(&h->mb.s, cudaStreamNonBlocking)) != cudaSuccess) return bail("stream", e);
    if ((e = cudaFuncSetAttribute(*v.kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)*v.smem)) != cudaSuccess)
        return bail("smem attribute", e);
    void *dctl, *dframe, *dout;
    if ((e = cudaHostGetDevicePointer(&dctl, h->mb.ctl, 0)) != cudaSuccess) return bail("map ctl", e);
    if ((e = cudaHostGetDevicePointer(&dframe, h->mb.hframe, 0)) != cudaSuccess) return bail("map frame", e);
    if ((e = cudaHostGetDevicePointer(&dout, h->mb.hout, 0)) != cudaSuccess) return bail("map out", e);
    unsigned long long idle_ns = (unsigned long long)(idle_seconds * 1e9);
    const uint32_t* gtab = h->d_gtab;
    int8_t* dbuf = h->mb.dbuf;
    unsigned fl = h->flags;
    void* args[] = {&dframe, &dout, &dctl, &dbuf, (void*)&gtab, &idle_ns, &fl};
    if ((e = cudaLaunchKernel(*v.kern, dim3(1), dim3(v.threads), args, *v.smem, h->mb.s)) != cudaSuccess) return bail("launch", e);
    h->mb.open = true;
    return POLAR_OK;
}

extern "C" polar_status polar_mailbox_decode_i8(polar_code* h, const int8_t* host_llr, uint32_t* host_info, double timeout_seconds) {
    if (!h || !host_llr || !host_info) return fail(POLAR_ERR_INVALID_ARGUMENT, "null pointer");
    if (!h->mb.open) return fail(POLAR_ERR_INVALID_ARGUMENT, "mailbox not open");
    std::memcpy(h->mb.hframe, host_llr, h->N);
    volatile MailboxCtlHost* ctl = (volatile MailboxCtlHost*)h->mb.ctl;
    // 0 is the initial value of done and 0xffffffff the stop request: the sequence skips both
    if (++h->mb.seq == 0xffffffffu) h->mb.seq = 1;
    const unsigned int seq = h->mb.seq;
    __atomic_store_n(&((MailboxCtlHost*)h->mb.ctl)->req, seq, __ATOMIC_RELEASE);
    const auto t0 = std::chrono::steady_clock::now();
    for (uint32_t spin = 0;; ++spin) {
        if (__atomic_load_n(&((MailboxCtlHost*)h->mb.ctl)->done, __ATOMIC_ACQUIRE) == seq) break;
        if ((spin & 1023u) == 0 &&
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_seconds) {
            (void)ctl;
            return fail(POLAR_ERR_CUDA, "mailbox kernel did not answer within %.3f s (idle timeout or fault)", timeout_seconds);
        }
    }
    std::memcpy(host_info, h->mb.hout, words_of(h->K) * 4);
    return POLAR_OK;
}

extern "C" polar_status polar_mailbox_close(polar_code* h) {
    if (!h) return fail(POLAR_ERR_INVALID_ARGUMENT, "null handle");
    std::lock_guard<std::mutex> lock(h->mu);
    if (!h->mb.open) return POLAR_OK;
    __atomic_store_n(&((MailboxCtlHost*)h->mb.ctl)->req, 0xffffffffu, __ATOMIC_RELEASE);
    const cudaError_t e = cudaStreamSynchronize(h->mb.s);
    mailbox_free(h);
    if (e != cudaSuccess) return fail(POLAR_ERR_CUDA, "mailbox kernel: %s", cudaGetErrorString(e));
    return POLAR_OK;
}

// ------------------------------------------------------------------------- construction

extern "C" polar_status polar_construct_ga(uint32_t N, uint32_t K, double design_ebn0_db, uint8_t* mask_out) {
    if (!mask_out) return fail(POLAR_ERR_INVALID_ARGUMENT, "null mask_out");
    if (N < 2 || N > (1u << 24) || (N & (N - 1))) return fail(POLAR_ERR_INVALID_ARGUMENT, "N=%u is not a power of two", N);
    if (K < 1 || K > N) return fail(POLAR_ERR_INVALID_ARGUMENT, "K=%u not in [1, N]", K);
    if (!std::isfinite(design_ebn0_db)) return fail(POLAR_ERR_INVALID_ARGUMENT, "design Eb/N0 not finite");
    construct_ga((int)N, (int)K, design_ebn0_db, mask_out);
    return POLAR_OK;
}

// ------------------------------------------------------------------------- encoder / generator

namespace {

// Philox4x32-10 (Salmon et al., SC'11), counter (c0..c3), key (k0, k1).
struct U4 {
    uint32_t x, y, z, w;
};
__device__ __forceinline__ U4 philox(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

// x <- x G_N on a packed codeword in shared memory (nw = N/32 words, or 1 word if N < 32):
// x[j] ^= x[j | d] for every bit d of the index (G_N[i][j] = [j subset of i]).
__device__ void transform_smem(uint32_t* x, int N, int nw) {
    const uint32_t in_word[5] = {0x55555555u, 0x33333333u, 0x0F0F0F0Fu, 0x00FF00FFu, 0x0000FFFFu};
    for (int b = 0; b < 5 && (1 << b) < N; ++b) {
        const int d = 1 << b;
        for (int k = threadIdx.x; k < nw; k += blockDim.x) x[k] ^= (x[k] >> d) & in_word[b];
        __syncthreads();
    }
    for (int D = 1; D < nw; D <<= 1) {
        for (int k = threadIdx.x; k < nw; k += blockDim.x)
            if (!(k & D)) x[k] ^= x[k | D];
        __syncthreads();
    }
}

// Systematic codeword in smem from packed info bits (reading C4): v[A] = d, x = mask_A(vG) G.
// info_word(q) yields information word q (32 bits, LSB-first); each thread places the set bits
// of its words at their positions pos[] (uint32: N up to 2^20).
template <class InfoWord>
__device__ void systematic_smem(uint32_t* x, InfoWord info_word, const uint32_t* pos, const uint32_t* info_mask,
                                int N, int K, int nw) {
    for (int k = threadIdx.x; k < nw; k += blockDim.x) x[k] = 0;
    __syncthreads();
    for (int q = threadIdx.x; q < (K + 31) / 32; q += blockDim.x)
        for (uint32_t w = info_word(q); w; w &= w - 1) {
            const uint32_t t = pos[32 * q + __ffs(w) - 1];
            atomicOr(&x[t >> 5], 1u << (t & 31));
        }
    __syncthreads();
    transform_smem(x, N, nw);
    for (int k = threadIdx.x; k < nw; k += blockDim.x) x[k] &= info_mask[k];
    __syncthreads();
    transform_smem(x, N, nw);
}

__global__ void k_encode(const uint32_t* info, long long n, uint32_t* cw, const uint32_t* pos,
                         const uint32_t* info_mask, int N, int K) {
    extern __shared__ uint32_t x[];
    const int nw = N >= 32 ? N / 32 : 1;
    const int wk = (K + 31) / 32;
    for (long long f = blockIdx.x; f < n; f += gridDim.x) {
        const uint32_t* d = info + f * wk;
        systematic_smem(x, [&](int q) { return d[q]; }, pos, info_mask, N, K, nw);
        for (int k = threadIdx.x; k < nw; k += blockDim.x) cw[f * nw + k] = x[k];
        __syncthreads();
    }
}

__global__ void k_gen(unsigned long long seed, unsigned long long first, long long n, float sigma, float llr_scale,
                      float q_scale, float* llr_f32, int8_t* llr_i8, uint32_t* info_out, const uint32_t* pos,
                      const uint32_t* info_mask, int N, int K) {
    extern __shared__ uint32_t sm[];
    const int nw = N >= 32 ? N / 32 : 1;
    const int wk = (K + 31) / 32;
    uint32_t* x = sm;
    const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    for (long long f = blockIdx.x; f < n; f += gridDim.x) {
        const unsigned long long g = first + (unsigned long long)f;
        // information word q of frame g: Philox keyed by the seed, counter (g, q) (reading C6)
        auto info_word = [&](int q) {
            uint32_t w = philox(U4{(uint32_t)g, (uint32_t)(g >> 32), (uint32_t)q, 0xB17u}, k0, k1).x;
            if (q == wk - 1 && (K & 31)) w &= (1u << (K & 31)) - 1u;
            return w;
        };
        if (info_out)
            for (int q = threadIdx.x; q < wk; q += blockDim.x) info_out[f * wk + q] = info_word(q);
        systematic_smem(x, info_word, pos, info_mask, N, K, nw);
        // BPSK 0 -> +1, 1 -> -1; y = s + sigma n; LLR = 2 y / sigma^2 (readings C6/C7).
        for (int q4 = threadIdx.x; q4 < (N + 3) / 4; q4 += blockDim.x) {
            const U4 r = philox(U4{(uint32_t)g, (uint32_t)(g >> 32), (uint32_t)q4, 0xA3Cu}, k0, k1);
            const uint32_t u[4] = {r.x, r.y, r.z, r.w};
            float nz[4];
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                const float u1 = ((float)u[2 * p] + 1.0f) * 2.3283064365386963e-10f;  // (0, 1]
                const float u2 = (float)u[2 * p + 1] * 2.3283064365386963e-10f;
                const float rad = sqrtf(-2.0f * logf(u1));
                float sn, cs;
                sincospif(2.0f * u2, &sn, &cs);
                nz[2 * p] = rad * cs;
                nz[2 * p + 1] = rad * sn;
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int i = 4 * q4 + e;
                if (i >= N) break;
                const float s = ((x[i >> 5] >> (i & 31)) & 1u) ? -1.0f : 1.0f;
                const float llr = llr_scale * (s + sigma * nz[e]);
                if (llr_f32) llr_f32[f * N + i] = llr;
                if (llr_i8) llr_i8[f * N + i] = (int8_t)fminf(fmaxf(rintf(q_scale * llr), -127.0f), 127.0f);
            }
        }
        __syncthreads();
    }
}

__global__ void k_count(const uint32_t* dec, const uint32_t* truth, long long n, int wk, unsigned long long* ctr) {
    const int lane = threadIdx.x & 31;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    unsigned long long bits = 0, frames_bad = 0;
    for (long long f = warp; f < n; f += nwarps) {
        uint32_t e = 0;
        for (int q = lane; q < wk; q += 32) {
            const uint32_t d = dec[f * wk + q] ^ truth[f * wk + q];
            e += __popc(d);
        }
        for (int o = 16; o; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
        bits += e;
        frames_bad += e != 0;
    }
    if (lane == 0) {
        atomicAdd(&ctr[1], bits);
        atomicAdd(&ctr[2], frames_bad);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&ctr[0], (unsigned long long)n);
}

}  // namespace

extern "C" polar_status polar_encode_systematic(const polar_code* h, const uint32_t* info, int64_t n, uint32_t* cw,
                                                polar_stream stream) {
    if (!h) return fail(POLAR_ERR_INVALID_ARGUMENT, "null handle");
    if (n < 0) return fail(POLAR_ERR_INVALID_ARGUMENT, "n_frames < 0");
    if (n == 0) return POLAR_OK;
    if (!info || !cw) return fail(POLAR_ERR_INVALID_ARGUMENT, "null buffer");
    if (!h->systematic_ok) return fail(POLAR_ERR_UNSUPPORTED_CODE, "information set not closed under bit-superset");
    if (!h->dev_ready) return fail(POLAR_ERR_CUDA, "no CUDA device");
    const int nw = h->N >= 32 ? h->N / 32 : 1;
    const unsigned grid = (unsigned)std::min<int64_t>(n, (int64_t)h->n_sm * 16);
    if (nw * 4 > 48 * 1024) CUDA_TRY(cudaFuncSetAttribute(k_encode, cudaFuncAttributeMaxDynamicSharedMemorySize, nw * 4));
    k_encode<<<grid, 256, nw * 4, (cudaStream_t)stream>>>(info, (long long)n, cw, h->d_pos, h->d_info_mask, (int)h->N,
                                                          (int)h->K);
    CUDA_TRY(cudaGetLastError());
    return POLAR_OK;
}

extern "C" polar_status polar_gen_bpsk_awgn(const polar_code* h, uint64_t seed, uint64_t first_frame, int64_t n,
                                            double ebn0_db, float q_scale, float* llr_f32, int8_t* llr_i8,
                                            uint32_t* info, polar_stream stream) {
    if (!h) return fail(POLAR_ERR_INVALID_ARGUMENT, "null handle");
    if (n < 0) return fail(POLAR_ERR_INVALID_ARGUMENT, "n_frames < 0");
    if (!std::isfinite(ebn0_db)) return fail(POLAR_ERR_INVALID_ARGUMENT, "Eb/N0 not finite");
    if (n == 0) return POLAR_OK;
    if (!h->systematic_ok) return fail(POLAR_ERR_UNSUPPORTED_CODE, "information set not closed under bit-superset");
    if (!h->dev_ready) return fail(POLAR_ERR_CUDA, "no CUDA device");
    const double rate = (double)h->K / (double)h->N;
    const double sigma2 = 1.0 / (2.0 * rate * std::pow(10.0, ebn0_db / 10.0));
    const int nw = h->N >= 32 ? h->N / 32 : 1;
    const unsigned grid = (unsigned)std::min<int64_t>(n, (int64_t)h->n_sm * 16);
    if (nw * 4 > 48 * 1024) CUDA_TRY(cudaFuncSetAttribute(k_gen, cudaFuncAttributeMaxDynamicSharedMemorySize, nw * 4));
    k_gen<<<grid, 256, nw * 4, (cudaStream_t)stream>>>(
        (unsigned long long)seed, (unsigned long long)first_frame, (long long)n, (float)std::sqrt(sigma2),
        (float)(2.0 / sigma2), q_scale, llr_f32, llr_i8, info, h->d_pos, h->d_info_mask, (int)h->N, (int)h->K);
    CUDA_TRY(cudaGetLastError());
    return POLAR_OK;
}

extern "C" polar_status polar_count_errors(const polar_code* h, const uint32_t* decoded, const uint32_t* truth,
                                           int64_t n, int64_t* counters, polar_stream stream) {
    if (!h || !decoded || !truth || !counters) return fail(POLAR_ERR_INVALID_ARGUMENT, "null pointer");
    if (n < 0) return fail(POLAR_ERR_INVALID_ARGUMENT, "n_frames < 0");
    if (n == 0) return POLAR_OK;
    if (!h->dev_ready) return fail(POLAR_ERR_CUDA, "no CUDA device");
    const unsigned grid = (unsigned)std::min<int64_t>((n + 7) / 8, (int64_t)h->n_sm * 8);
    k_count<<<grid, 256, 0, (cudaStream_t)stream>>>(decoded, truth, (long long)n, (int)words_of(h->K),
                                                    (unsigned long long*)counters);
    CUDA_TRY(cudaGetLastError());
    return POLAR_OK;
}
