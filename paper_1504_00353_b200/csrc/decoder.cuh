// decoder.cuh -- sm_100a device building blocks of the unrolled Fast-SSC decoders.
//
// Giard et al., arXiv:1504.00353.  The unrolled decoder is a straight list of operations
// with compile-time sizes (Listing 1; template specialisation P:792-795).  Here
// every operation is a force-inlined template instantiated by the code emitted per code
// (codegen.cpp), re-derived for SIMT:
//
//  * warp scope (node sizes N_v <= W, W <= 2048): one warp owns the subtree.  The LLRs of
//    the level-k stage (2^k values, the paper's alpha layout, one buffer per level,
//    P:789-790) live in registers r_k[] with element i = lane + 32*slot.  F/G at N_v >= 64
//    pair slot j with slot j + N_v/64 inside each lane; at N_v <= 32 the partner is
//    N_v/2 lanes away (one shuffle).  The hard decisions beta of nodes with N_v >= 32 live
//    as bits of a per-lane 64-bit word bw (bit s of lane l = beta[l + 32 s]); nodes with
//    N_v <= 32 keep beta as a warp-uniform mask (bit i = beta[i]).  Combine (eq:combine
//    P:318-325) is then a shift-and-xor on bw or on masks.
//  * CTA scope (N_v > W, only for N > 2048): all threads of the CTA run the op on shared
//    memory stages; beta is the codeword's natural bit array, packed in 32-bit words
//    (one N-bit array, combined in place).
//
// Profiles (the paper's float and 8-bit fixed point):
//  * PF32: f32 values; g is one IEEE add (__fadd_rn, no FMA contraction, reading C17);
//  * PI8 : int8 storage, int32 registers; g saturates to [-127, 127] (reading C8).
#pragma once

#ifdef __CUDACC_RTC__
// NVRTC (run-time specialisation of an unregistered code, polar_api.cu jit_code): no host
// standard headers; the fixed-width types the kernels use.
typedef signed char int8_t;
typedef unsigned char uint8_t;
typedef unsigned short uint16_t;
typedef unsigned int uint32_t;
typedef long long int64_t;
typedef unsigned long long uint64_t;
#include <cuda_fp16.h>
#else
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#endif

namespace pd {

#define PD_INLINE __device__ __forceinline__
constexpr unsigned FULL = 0xffffffffu;

// min(|a|, |b|) carrying the sign sign(a) xor sign(b): f32 and f16x2 (sm_86+ PTX min.xorsign.abs)
PD_INLINE float fminxs(float a, float b) {
    float d;
    asm("min.xorsign.abs.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
    return d;
}
PD_INLINE uint32_t h2minxs(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("min.xorsign.abs.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
PD_INLINE uint32_t h2add(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("add.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
PD_INLINE uint32_t h2max(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("max.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}

PD_INLINE unsigned lane_id() { return threadIdx.x & 31u; }

template <class A, class B>
struct same_t {
    static constexpr bool value = false;
};
template <class A>
struct same_t<A, A> {
    static constexpr bool value = true;
};
template <bool B, class T, class F>
struct cond_t {
    using type = T;
};
template <class T, class F>
struct cond_t<false, T, F> {
    using type = F;
};

// POLAR_TRACE builds: clock64() after every op of the latency variant's critical path, block 0
// thread 0 only, into the buffer the library passes (tools/trace_latency.py reads it back).
#ifdef POLAR_TRACE
static __device__ unsigned long long* g_ptrace;
#define PTRACE(k)                                                                  \
    do {                                                                           \
        if (threadIdx.x == 0 && blockIdx.x == 0 && g_ptrace) g_ptrace[(k)] = clock64(); \
    } while (0)
#else
#define PTRACE(k) \
    do {          \
    } while (0)
#endif
// POLAR_DEBUG_DUMP builds (libpolar_dump.so, test infrastructure): every F / G / G_0R output
// vector is appended, in the decoder's op order, to a per-frame float array (the alpha stages
// the north star's f32 bar compares with the oracle, 1e-5 relative).  The frame's array and
// its fill position live in shared memory per warp index: the warp of a throughput frame
// group, 0 for the latency CTA (only its warp 0 runs the register subtrees).
// floats per frame in the dump: every level of the tree holds at most N F/G outputs
__host__ __device__ constexpr int dump_stride(int N) {
    int l = 0;
    while ((1 << l) < N) ++l;
    return N * (l > 0 ? l : 1);
}
#ifdef POLAR_DEBUG_DUMP
__shared__ float* s_dbase[32];
__shared__ int s_dpos[32];
PD_INLINE unsigned dump_slot() { return threadIdx.x >> 5; }
// register outputs of a warp op: n/2 values, element i at (lane i mod 32, slot i / 32) when
// n >= 64, replicated (lane l holds element l mod n/2) when n <= 32
template <int n, class V>
PD_INLINE void dump_reg(const V* c) {
    const unsigned w = dump_slot();
    float* const d = s_dbase[w] + s_dpos[w];
    if constexpr (n >= 64) {
#pragma unroll
        for (int j = 0; j < n / 64; ++j) d[(threadIdx.x & 31u) + 32 * j] = (float)c[j];
    } else {
        if ((threadIdx.x & 31u) < (unsigned)(n / 2)) d[threadIdx.x & 31u] = (float)c[0];
    }
    __syncwarp();
    if ((threadIdx.x & 31u) == 0) s_dpos[w] += n / 2;
    __syncwarp();
}
PD_INLINE float dump_val(float x) { return x; }
PD_INLINE float dump_val(int8_t x) { return (float)x; }
PD_INLINE float dump_val(uint8_t x) { return (float)((int)x - 128); }  // biased int8 stage
PD_INLINE float dump_val(__half x) { return __half2float(x); }
// a stage written by a CTA-scope op: h elements at p (group of T threads)
template <int T, class S>
PD_INLINE void dump_stage(const S* p, int h) {
    const unsigned w = T == 32 ? dump_slot() : 0u;
    const int tid = T == 32 ? (int)(threadIdx.x & 31u) : (int)threadIdx.x;
    float* const d = s_dbase[w] + s_dpos[w];
    for (int i = tid; i < h; i += T) d[i] = dump_val(p[i]);
    if constexpr (T == 32) __syncwarp(); else asm volatile("bar.sync 1, %0;" ::"n"(T) : "memory");
    if (tid == 0) s_dpos[w] += h;
    if constexpr (T == 32) __syncwarp(); else asm volatile("bar.sync 1, %0;" ::"n"(T) : "memory");
}
#define PD_DUMPR(n, c) dump_reg<n>(c)
#define PD_DUMPS(p, h) dump_stage<T>(p, h)
#else
#define PD_DUMPR(n, c) \
    do {               \
    } while (0)
#define PD_DUMPS(p, h) \
    do {               \
    } while (0)
#endif

// Index of the thread in its frame group of T threads (T = 32: the lane).
template <int T>
PD_INLINE int gtid() { return T == 32 ? (int)(threadIdx.x & 31u) : (int)threadIdx.x; }

__host__ __device__ constexpr int slots(int n) { return n >= 32 ? n / 32 : 1; }
__host__ __device__ constexpr uint32_t low_mask(int n) { return n >= 32 ? 0xffffffffu : ((1u << n) - 1u); }

// ------------------------------------------------------------------------------ profiles

struct PF32 {
    using in_t = float;   // channel LLR storage
    using st_t = float;   // shared-memory stage storage (CTA scope)
    using v_t = float;    // register value
    using acc_t = float;  // repetition accumulator
    static constexpr bool kExactSum = false;    // repetition sums in halving order (C13)
    static constexpr bool kPackedKey = false;   // SPC argmin needs two reductions
    static constexpr bool kChanInSmem = false;  // N=32768 f32 channel does not fit with the tree
    static PD_INLINE v_t ld(float x) { return x; }
    static PD_INLINE float st(v_t x) { return x; }
    // eq:f: sgn(a) sgn(b) min(|a|, |b|) -- one FMNMX.XORSIGN |a|, |b| (the sign
    // is sign(a) xor sign(b); it differs from the comparison rule only on signed zeros,
    // which no decision reads, reading C9)
    static PD_INLINE v_t f(v_t a, v_t b) { return fminxs(a, b); }
    // eq:g: b + a if beta = 0 else b - a; beta flips the sign bit (P:817 idea)
    static PD_INLINE v_t g(v_t a, v_t b, uint32_t beta) {
        return __fadd_rn(b, __uint_as_float(__float_as_uint(a) ^ (beta << 31)));
    }
    static PD_INLINE v_t g0(v_t a, v_t b) { return __fadd_rn(b, a); }
    // g with beta given as the sign-bit mask (beta << 31)
    static PD_INLINE v_t gs(v_t a, v_t b, uint32_t sgn) { return __fadd_rn(b, __uint_as_float(__float_as_uint(a) ^ sgn)); }
    static PD_INLINE bool hd(v_t a) { return a < 0.0f; }  // eq:info P:444-449, -0 -> 0 (C9)
    static PD_INLINE uint32_t mag_key(v_t a) { return __float_as_uint(a) & 0x7fffffffu; }
    static PD_INLINE acc_t acc(v_t a) { return a; }
    static PD_INLINE acc_t add(acc_t a, acc_t b) { return __fadd_rn(a, b); }
    static PD_INLINE bool acc_neg(acc_t a) { return a < 0.0f; }
};

// int8 profile: 8-bit storage (channel and shared-memory stages); registers hold the same
// integers as f32, which is exact here (|values| <= 254 in any single g, sums < 2^24), so
// f is one FMNMX with |.| modifiers plus the sign, and g one FADD plus the clamp.
// Stages written by the decoder hold v + 128 as an unsigned byte ("biased"): the f16x2 unpack
// (0x64tt = 1024 + t) and pack then need no sign-bias XOR, one ALU-pipe instruction less per 4
// values each way (the ALU pipe is the kernel's busiest unit, profiles/r2k_tp32k.txt).  The
// channel stays signed int8 as the API defines it.
struct PI8 {
    using in_t = int8_t;
    using st_t = uint8_t;
    using v_t = float;
    using acc_t = float;
    static constexpr bool kExactSum = true;  // integer sums below 2^24: any order is exact (C12)
    static constexpr bool kPackedKey = true;
    static constexpr bool kChanInSmem = true;
    // -128 -> -127 (C8); int -> float by the exponent trick (integer ALU + one FADD)
    static PD_INLINE v_t ld(int8_t x) { return __int_as_float(0x4B400000 + max((int)x, -127)) - 12582912.0f; }
    static PD_INLINE uint8_t st(v_t x) { return (uint8_t)(__float2int_rn(x) + 128); }
    static PD_INLINE v_t ld(uint8_t t) { return __int_as_float(0x4B400000 + (int)t) - 12583040.0f; }  // biased stage
    static PD_INLINE v_t ld(float x) { return x; }  // the f32 subtree-input stage
    static PD_INLINE v_t ld(__half x) { return __half2float(x); }  // f16 stages (exact integers)
    static PD_INLINE v_t f(v_t a, v_t b) { return PF32::f(a, b); }
    // saturating adder (max(-127) P:848): clamp(x) = copysign(min(|x|, 127), x)
    static PD_INLINE v_t g(v_t a, v_t b, uint32_t beta) { return fminxs(PF32::g(a, b, beta), 127.0f); }
    static PD_INLINE v_t g0(v_t a, v_t b) { return fminxs(__fadd_rn(b, a), 127.0f); }
    static PD_INLINE v_t gs(v_t a, v_t b, uint32_t sgn) { return fminxs(PF32::gs(a, b, sgn), 127.0f); }
    static PD_INLINE bool hd(v_t a) { return a < 0.0f; }
    static PD_INLINE uint32_t mag_key(v_t a) { return __float_as_uint(a) & 0x7fffffffu; }
    static PD_INLINE acc_t acc(v_t a) { return a; }
    static PD_INLINE acc_t add(acc_t a, acc_t b) { return __fadd_rn(a, b); }
    static PD_INLINE bool acc_neg(acc_t a) { return a < 0.0f; }
};

// ------------------------------------------------------------- vector chunks (CTA scope)
// CTA-scope ops move CE consecutive elements per thread: float4 (f32) or 4/8/16 packed int8.

// Vector loads/stores with an explicit state space (SP_SHARED / SP_GLOBAL), so that the
// stage ops can be shared non-inlined functions without falling back to generic accesses.
enum : int { SP_GLOBAL = 0, SP_SHARED = 1 };

// L2 eviction priority for global accesses: the channel is streamed (evict_first), the stage
// scratch should stay resident (evict_last).  Measured at N = 32768: 200 -> 215 Gbps, DRAM
// writes per frame 35 KB -> 13 KB (profiles/r1_history.md); POLAR_NO_L2_HINTS disables.
enum : int { L2_NORMAL = 0, L2_FIRST = 1, L2_LAST = 2 };
template <int H>
PD_INLINE uint64_t l2_policy() {
    uint64_t pol;
    if constexpr (H == L2_FIRST) asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    else asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

template <int SP, int BYTES, int H = L2_NORMAL>
PD_INLINE void vld(const void* p, uint32_t* w) {
#ifdef POLAR_NO_L2_HINTS
    constexpr int HH = L2_NORMAL;
#else
    constexpr int HH = H;
#endif
    if constexpr (SP == SP_GLOBAL && HH != L2_NORMAL) {
        const uint64_t pol = l2_policy<HH>();
        if constexpr (BYTES == 16)
            asm volatile("ld.global.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                         : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]) : "l"(p), "l"(pol));
        else if constexpr (BYTES == 8)
            asm volatile("ld.global.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;" : "=r"(w[0]), "=r"(w[1]) : "l"(p), "l"(pol));
        else
            asm volatile("ld.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(w[0]) : "l"(p), "l"(pol));
        return;
    }
    if constexpr (SP == SP_SHARED) {
        const uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
        if constexpr (BYTES == 16)
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]) : "r"(a));
        else if constexpr (BYTES == 8)
            asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(w[0]), "=r"(w[1]) : "r"(a));
        else
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w[0]) : "r"(a));
    } else {
        if constexpr (BYTES == 16)
            asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]) : "l"(p));
        else if constexpr (BYTES == 8)
            asm volatile("ld.global.v2.u32 {%0,%1}, [%2];" : "=r"(w[0]), "=r"(w[1]) : "l"(p));
        else
            asm volatile("ld.global.u32 %0, [%1];" : "=r"(w[0]) : "l"(p));
    }
}
template <int SP, int BYTES, int H = L2_NORMAL>
PD_INLINE void vst(void* p, const uint32_t* w) {
#ifdef POLAR_NO_L2_HINTS
    constexpr int HH = L2_NORMAL;
#else
    constexpr int HH = H;
#endif
    if constexpr (SP == SP_GLOBAL && HH != L2_NORMAL) {
        const uint64_t pol = l2_policy<HH>();
        if constexpr (BYTES == 16)
            asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "r"(w[0]), "r"(w[1]),
                         "r"(w[2]), "r"(w[3]), "l"(pol) : "memory");
        else if constexpr (BYTES == 8)
            asm volatile("st.global.L2::cache_hint.v2.u32 [%0], {%1,%2}, %3;" ::"l"(p), "r"(w[0]), "r"(w[1]), "l"(pol)
                         : "memory");
        else
            asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p), "r"(w[0]), "l"(pol) : "memory");
        return;
    }
    if constexpr (SP == SP_SHARED) {
        const uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
        if constexpr (BYTES == 16)
            asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]) : "memory");
        else if constexpr (BYTES == 8)
            asm volatile("st.shared.v2.u32 [%0], {%1,%2};" ::"r"(a), "r"(w[0]), "r"(w[1]) : "memory");
        else
            asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(w[0]) : "memory");
    } else {
        if constexpr (BYTES == 16)
            asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]) : "memory");
        else if constexpr (BYTES == 8)
            asm volatile("st.global.v2.u32 [%0], {%1,%2};" ::"l"(p), "r"(w[0]), "r"(w[1]) : "memory");
        else
            asm volatile("st.global.u32 [%0], %1;" ::"l"(p), "r"(w[0]) : "memory");
    }
}

template <class P, int CE>
struct Chunk;

template <int CE>
struct Chunk<PF32, CE> {
    static_assert(CE == 4, "");
    float v[4];
    uint32_t w[4];
    template <int SP, int H, class S>
    PD_INLINE void load_raw(const S* p) { vld<SP, 16, H>(p, w); }
    template <class S>
    PD_INLINE void unpack_raw(bool = false) {
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = __uint_as_float(w[k]);
    }
    template <int SP, int H, class D>
    PD_INLINE void store(D* p) const {
        const uint32_t w[4] = {__float_as_uint(v[0]), __float_as_uint(v[1]), __float_as_uint(v[2]), __float_as_uint(v[3])};
        vst<SP, 16, H>(p, w);
    }
};

// int8 stages are processed as integer-valued f16x2 (exact: |values| <= 254 before the clamp).
// unpack: t = w ^ 0x80808080 (bias 128), halves 0x64tt = 1024 + t, minus 1152 -> the value.
// pack: + 1152 -> 0x64tt, gather the low bytes, remove the bias.
template <int CE>
struct Chunk<PI8, CE> {
    static_assert(CE == 4 || CE == 8 || CE == 16, "");
    uint32_t h[CE / 2];
    // biased: stage bytes already hold v + 128 (PI8); else the signed channel (bias by XOR)
    PD_INLINE void unpack(const uint32_t* w, bool clamp, bool biased = false) {
#pragma unroll
        for (int q = 0; q < CE / 4; ++q) {
            const uint32_t t = biased ? w[q] : w[q] ^ 0x80808080u;
            h[2 * q] = h2add(__byte_perm(t, 0x64646464u, 0x4140), 0xE480E480u);
            h[2 * q + 1] = h2add(__byte_perm(t, 0x64646464u, 0x4342), 0xE480E480u);
            if (clamp) {  // channel input: -128 -> -127 (reading C8)
                h[2 * q] = h2max(h[2 * q], 0xD7F0D7F0u);
                h[2 * q + 1] = h2max(h[2 * q + 1], 0xD7F0D7F0u);
            }
        }
    }
    uint32_t w[CE / 4];
    // Source S: int8 (channel or an int8 stage: CE bytes, unpacked after the load) or __half
    // (an f16 stage: the CE values load straight into h[], no conversion).
    template <int SP, int H, class S>
    PD_INLINE void load_raw(const S* p) {
        if constexpr (sizeof(S) == 1) {
            vld<SP, CE, H>(p, w);
        } else {
            static_assert(sizeof(S) == 2, "");
            if constexpr (CE == 16) {
                vld<SP, 16, H>(p, h);
                vld<SP, 16, H>((const S*)p + 8, h + 4);
            } else {
                vld<SP, 2 * CE, H>(p, h);
            }
        }
    }
    template <class S>
    PD_INLINE void unpack_raw(bool clamp) {
        if constexpr (sizeof(S) == 1) unpack(w, clamp, same_t<S, uint8_t>::value);
    }
    // D: float (the f32 stage feeding the register subtrees, latency variant), __half (an f16
    // stage: h[] stored as is) or int8
    template <int SP, int H, class D>
    PD_INLINE void store(D* p) const {
        if constexpr (sizeof(D) == 2) {
            if constexpr (CE == 16) {
                vst<SP, 16, H>(p, h);
                vst<SP, 16, H>(p + 8, h + 4);
            } else {
                vst<SP, 2 * CE, H>(p, h);
            }
        } else if constexpr (sizeof(D) == 4) {
#pragma unroll
            for (int q = 0; q < CE / 4; ++q) {
                const float2 lo = __half22float2(*reinterpret_cast<const __half2*>(&h[2 * q]));
                const float2 hi = __half22float2(*reinterpret_cast<const __half2*>(&h[2 * q + 1]));
                const uint32_t w[4] = {__float_as_uint(lo.x), __float_as_uint(lo.y), __float_as_uint(hi.x),
                                       __float_as_uint(hi.y)};
                vst<SP, 16>((float*)p + 4 * q, w);
            }
        } else {
            uint32_t w[CE / 4];
#pragma unroll
            for (int q = 0; q < CE / 4; ++q)
                w[q] = __byte_perm(h2add(h[2 * q], 0x64806480u), h2add(h[2 * q + 1], 0x64806480u), 0x6420) ^
                       (same_t<D, uint8_t>::value ? 0u : 0x80808080u);
            vst<SP, CE, H>(p, w);
        }
    }
    // F: h = f(h, b)
    PD_INLINE void f(const Chunk& b) {
#pragma unroll
        for (int q = 0; q < CE / 2; ++q) h[q] = h2minxs(h[q], b.h[q]);
    }
    // G: h = sat(b + (beta ? -h : h)); bit k of `bits` is beta of element k; the saturation
    // is min.xorsign.abs against 127.
    PD_INLINE void g(const Chunk& b, uint32_t bits) {
        // sign mask of the pair (2q, 2q+1) = bit 2q at 15 and bit 2q+1 at 31.  sp holds the even
        // bits in place and the odd bits moved up by 15 (bit 2j+1 at 2j+16), so one left shift by
        // 15 - 2q puts both of pair q's bits where they belong; the mask and the XOR into h are
        // one LOP3 -- two instructions per pair (was four: shift, and, multiply, and-xor).
        const uint32_t sp = (bits & 0x5555u) | ((bits & 0xAAAAu) << 15);
#pragma unroll
        for (int q = 0; q < CE / 2; ++q) {
            const uint32_t m = (sp << (15 - 2 * q)) & 0x80008000u;
            h[q] = h2minxs(h2add(b.h[q], h[q] ^ m), 0x57F057F0u);
        }
    }
    PD_INLINE void g0(const Chunk& b) {
#pragma unroll
        for (int q = 0; q < CE / 2; ++q) h[q] = h2minxs(h2add(b.h[q], h[q]), 0x57F057F0u);
    }
};

template <int CE>
PD_INLINE void chunk_f(Chunk<PF32, CE>& a, const Chunk<PF32, CE>& b) {
#pragma unroll
    for (int k = 0; k < CE; ++k) a.v[k] = PF32::f(a.v[k], b.v[k]);
}
template <int CE>
PD_INLINE void chunk_g(Chunk<PF32, CE>& a, const Chunk<PF32, CE>& b, uint32_t bits) {
#pragma unroll
    for (int k = 0; k < CE; ++k) a.v[k] = PF32::g(a.v[k], b.v[k], (bits >> k) & 1u);
}
template <int CE>
PD_INLINE void chunk_g0(Chunk<PF32, CE>& a, const Chunk<PF32, CE>& b) {
#pragma unroll
    for (int k = 0; k < CE; ++k) a.v[k] = PF32::g0(a.v[k], b.v[k]);
}
template <int CE>
PD_INLINE void chunk_f(Chunk<PI8, CE>& a, const Chunk<PI8, CE>& b) { a.f(b); }
template <int CE>
PD_INLINE void chunk_g(Chunk<PI8, CE>& a, const Chunk<PI8, CE>& b, uint32_t bits) { a.g(b, bits); }
template <int CE>
PD_INLINE void chunk_g0(Chunk<PI8, CE>& a, const Chunk<PI8, CE>& b) { a.g0(b); }

// Elements per chunk for a CTA op over `half` outputs with T threads.
template <class P, int half, int T>
__host__ __device__ constexpr int chunk_elems() {
    if constexpr (sizeof(typename P::st_t) == 4) return 4;
    else return (half / T >= 16) ? 16 : (half / T >= 8) ? 8 : 4;
}

// Barrier of a T-thread frame group (a lone warp needs only __syncwarp).  A CTA-wide group
// uses named barrier 1 over its T threads, so that an extra helper warp of the latency
// variant (kernels.cuh) never takes part.
template <int T>
PD_INLINE void group_sync() {
    if constexpr (T == 32) __syncwarp();
    else asm volatile("bar.sync 1, %0;" ::"n"(T) : "memory");
}

// ------------------------------------------------------------------- warp-scope sources
// A source of node LLRs: a register stage (RegSrc) or a shared-memory stage (MemSrc, the
// subtree root).  v(j): element lane + 32 j (N_v >= 64).  Nodes with N_v <= 32 are held
// replicated: lane l holds element l mod N_v, so every lane carries a valid value and every
// warp reduction below ends uniform without a broadcast.  one(n): element lane mod n.
// pair(h, x, y) (node of 2h elements): x = own element (lane mod 2h), y = the partner
// (lane mod 2h) xor h; lanes with (lane & h) hold the second element of their pair.

template <class P>
struct RegSrc {
    using V = typename P::v_t;
    V* a;
    PD_INLINE V v(int j) const { return a[j]; }
    PD_INLINE V one(int) const { return a[0]; }
    PD_INLINE void pair(int h, V& x, V& y) const {
        x = a[0];
        y = __shfl_xor_sync(FULL, a[0], h);
    }
};

// CHAN: the source is the channel (int8 input -128 is clamped, reading C8); stages written by
// the decoder never hold -128, so their loads skip the clamp.
template <class P, class T, bool CHAN = true>
struct MemSrc {
    using V = typename P::v_t;
    const T* p;
    PD_INLINE V ld(T x) const {
        if constexpr (same_t<T, uint8_t>::value) return __int_as_float(0x4B400000 + (int)x) - 12583040.0f;  // biased
        else if constexpr (!CHAN && sizeof(T) == 1) return __int_as_float(0x4B400000 + (int)x) - 12582912.0f;
        else return P::ld(x);
    }
    PD_INLINE V v(int j) const { return ld(p[lane_id() + 32 * j]); }
    PD_INLINE V one(int n) const { return ld(p[lane_id() & (n - 1)]); }
    PD_INLINE void pair(int h, V& x, V& y) const {
        const unsigned l = lane_id() & (2 * h - 1);
        x = ld(p[l]);
        y = ld(p[l ^ h]);
    }
};

// ----------------------------------------------------------------- warp-scope operations

// F<n>: child[i] = f(alpha[i], alpha[i + n/2]).  f is symmetric, so for n <= 32 both
// lanes of a pair compute child element lane mod n/2 (the child stays replicated).
template <class P, int n, class Src>
PD_INLINE void wF(const Src& s, typename P::v_t* c) {
    if constexpr (n >= 64) {
#pragma unroll
        for (int j = 0; j < n / 64; ++j) c[j] = P::f(s.v(j), s.v(j + n / 64));
    } else {
        typename P::v_t x, y;
        s.pair(n / 2, x, y);
        c[0] = P::f(x, y);
    }
    PD_DUMPR(n, c);
}

// G<n>: child[i] = g(alpha[i], alpha[i + n/2], beta_l[i]); beta_l from bw slots
// s0.. (n >= 64) or from the left child's mask ml (n <= 32).
template <class P, int n, int s0, class Src>
PD_INLINE void wG(const Src& s, typename P::v_t* c, uint64_t bw, uint32_t ml) {
    if constexpr (n >= 64) {
#pragma unroll
        for (int j = 0; j < n / 64; ++j)
            c[j] = P::g(s.v(j), s.v(j + n / 64), (uint32_t)(bw >> (s0 + j)) & 1u);
    } else {
        // b + (a ^ s) with (a, b) = (own, partner) in the first half of each pair and
        // (partner, own) in the second: flip the sign of own (first half) or of the partner
        // (second half), then add -- the masks depend only on ml and the lane, so the
        // critical path after the shuffle is xor, add, saturate.
#ifdef POLAR_SELECT_SMALL_G
        typename P::v_t x, y;
        s.pair(n / 2, x, y);
        const bool second = lane_id() & (n / 2);
        c[0] = P::g(second ? y : x, second ? x : y, (ml >> (lane_id() & (n / 2 - 1))) & 1u);
#else
        // sgn: beta of this lane's element at bit 31 only; sec: the lane's "second half" bit
        // (lane & n/2) shifted to bit 31 (the lower lane bits land below 31, masked by sgn), so
        // each flip is one three-input LOP3 (no predicate / select)
        constexpr int LH = n >= 4 ? (n == 4 ? 1 : n == 8 ? 2 : n == 16 ? 3 : n == 32 ? 4 : 0) : 0;
        const uint32_t sgn = (ml >> (lane_id() & (n / 2 - 1))) << 31;
        const uint32_t sec = lane_id() << (31 - LH);
        typename P::v_t x, y;
        s.pair(n / 2, x, y);
        const float xa = __uint_as_float(__float_as_uint(x) ^ (sgn & ~sec));
        const float ya = __uint_as_float(__float_as_uint(y) ^ (sgn & sec));
        c[0] = P::g0(xa, ya);
#endif
    }
    PD_DUMPR(n, c);
}

// G<n> (n <= 32) after a repetition left child: its mask ml is all ones or zero, so the sign
// is bit 0 of ml moved to bit 31 -- no per-lane bit extraction on the critical path.
template <class P, int n, class Src>
PD_INLINE void wGu(const Src& s, typename P::v_t* c, uint32_t ml) {
    static_assert(n <= 32, "");
    constexpr int LH = n == 2 ? 0 : n == 4 ? 1 : n == 8 ? 2 : n == 16 ? 3 : 4;
    const uint32_t sgn = ml << 31;
    const uint32_t sec = lane_id() << (31 - LH);
    typename P::v_t x, y;
    s.pair(n / 2, x, y);
    const float xa = __uint_as_float(__float_as_uint(x) ^ (sgn & ~sec));
    const float ya = __uint_as_float(__float_as_uint(y) ^ (sgn & sec));
    c[0] = P::g0(xa, ya);
    PD_DUMPR(n, c);
}

// G_0R<n>: G with beta_l = 0 (left child Rate-0); b + a is symmetric.
template <class P, int n, class Src>
PD_INLINE void wG0R(const Src& s, typename P::v_t* c) {
    if constexpr (n >= 64) {
#pragma unroll
        for (int j = 0; j < n / 64; ++j) c[j] = P::g0(s.v(j), s.v(j + n / 64));
    } else {
        typename P::v_t x, y;
        s.pair(n / 2, x, y);
        c[0] = P::g0(x, y);
    }
    PD_DUMPR(n, c);
}

// Rate-1 / Info<n> (eq:info P:444-449): beta = hard decisions.
template <class P, int n, int s0, class Src>
PD_INLINE void wR1(const Src& s, uint64_t& bw) {
    static_assert(n >= 64, "");
#pragma unroll
    for (int j = 0; j < n / 32; ++j) bw |= (uint64_t)P::hd(s.v(j)) << (s0 + j);
}
template <class P, int n, class Src>
PD_INLINE uint32_t wR1m(const Src& s) {
    static_assert(n <= 32, "");
    return __ballot_sync(FULL, P::hd(s.one(n))) & low_mask(n);
}

// Repetition<n>: all bits = [sum alpha < 0].  Sum in pairwise-halving order
// x[i] += x[i + m/2], m = n, n/2, ..., 2 (reading C13): lane-local slot halving first, then
// an xor butterfly over the lanes, which performs the same additions (each one commuted in
// half of the lanes) and leaves the sum in every lane.
template <class P, int n, class Src>
PD_INLINE bool wRepDecide(const Src& s) {
    using A = typename P::acc_t;
    A t0;
    constexpr int start = n >= 64 ? 16 : n / 2;
    if constexpr (n >= 64) {
        A t[n / 32];
#pragma unroll
        for (int j = 0; j < n / 32; ++j) t[j] = P::acc(s.v(j));
#pragma unroll
        for (int m = n / 32; m > 1; m /= 2)
#pragma unroll
            for (int j = 0; j < m / 2; ++j) t[j] = P::add(t[j], t[j + m / 2]);
        t0 = t[0];
    } else {
        t0 = P::acc(s.one(n));
    }
    if constexpr (P::kExactSum) {
        // int8 profile: the values are integers, so the lane's partial is converted exactly
        // (1.5 * 2^23 magic) and one redux.sync.add sums the warp: the node's sum (N_v >= 64) or
        // 32 / N_v copies of it (replicated N_v <= 32) -- the same sign, hence the same decision
        // (C9, C12) -- one 23-cycle collective instead of log2(N_v) dependent shuffle-adds
        // (the 32 magic offsets are left in: the sum is 0x68000000 + sum mod 2^32, and for
        // |sum| < 2^26 the sum is negative exactly when that is below 0x68000000, unsigned)
        const uint32_t tot = __reduce_add_sync(FULL, (uint32_t)__float_as_int(t0 + 12582912.0f));
        return tot < 0x68000000u;
    } else {
#pragma unroll
        for (int o = start; o >= 1; o /= 2) t0 = P::add(t0, __shfl_xor_sync(FULL, t0, o));
        return P::acc_neg(t0);
    }
}
template <class P, int n, int s0, class Src>
PD_INLINE void wRep(const Src& s, uint64_t& bw) {
    static_assert(n >= 64, "");
    constexpr uint64_t span = (n / 32 == 64) ? ~0ull : (((1ull << (n / 32)) - 1ull) << s0);
    if (wRepDecide<P, n>(s)) bw |= span;
}
template <class P, int n, class Src>
PD_INLINE uint32_t wRepm(const Src& s) {
    return wRepDecide<P, n>(s) ? low_mask(n) : 0u;
}

// SPC<n>: hard decisions; if their parity is odd flip the decision of the
// least reliable bit, the lowest index among equal magnitudes (reading C10).  int8 profile:
// the f32 bits of an integer magnitude <= 254 leave the low 16 mantissa bits zero, so
// (|alpha| bits | index) is one exact key and one redux.min finds both minimum and index.
// int8 SPC key (|x| f32 bits | element index < 2^16): the low 16 mantissa bits of an integer
// <= 254 are zero, so the key is one select-LOP3 of the value's bits 16-30 and the index
PD_INLINE uint32_t spc_key16(float x, uint32_t idx) {
    uint32_t key;
    asm("lop3.b32 %0, %1, %2, 0x7fff0000, 0xE4;" : "=r"(key) : "r"(__float_as_uint(x)), "r"(idx));
    return key;
}
template <class P, int n, class Src>
PD_INLINE uint32_t wSPCm(const Src& s) {
    static_assert(n <= 32, "");
    const auto x = s.one(n);
    const uint32_t hdm = __ballot_sync(FULL, P::hd(x)) & low_mask(n);
    const uint32_t parity = __popc(hdm) & 1u;
    uint32_t idx;
    if constexpr (P::kPackedKey) {
        // (|x| bits with the low log2(n) bits -- zero for an integer <= 254 -- replaced by the
        // lane's element index): one select-LOP3 instead of mask-then-or
        constexpr uint32_t KM = 0x7fffffffu & ~(uint32_t)(n - 1);
        uint32_t key;  // (x & KM) | (lane & ~KM): lane has no bit 31, KM none either
        asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(key) : "r"(__float_as_uint(x)), "r"(lane_id()), "n"(KM));
        idx = __reduce_min_sync(FULL, key) & 31u;
    } else {
        const uint32_t key = P::mag_key(x);
        const uint32_t mn = __reduce_min_sync(FULL, key);
        idx = __ffs(__ballot_sync(FULL, key == mn) & low_mask(n)) - 1;
    }
    return hdm ^ (parity << idx);
}
template <class P, int n, int s0, class Src>
PD_INLINE void wSPC(const Src& s, uint64_t& bw) {
    static_assert(n >= 64, "");
    constexpr int J = n / 32;
    // the lane's J decision bits: 32-bit arithmetic up to n = 1024 (64-bit shifts cost two
    // instructions each on the batch-1 critical path)
    using HB = typename cond_t<(J <= 32), uint32_t, uint64_t>::type;
    HB hb = 0;
    uint32_t idx;
    // balanced reductions (log2 J dependent steps instead of a J-long chain); the lowest index
    // among equal magnitudes still wins (C10): int8 packs the index into the key
    if constexpr (P::kPackedKey) {
        uint32_t kk[J];
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const auto x = s.v(j);
            hb |= (HB)P::hd(x) << j;
            kk[j] = spc_key16(x, (uint32_t)(j * 32) | lane_id());
        }
#pragma unroll
        for (int m = J; m > 1; m /= 2)
#pragma unroll
            for (int j = 0; j < m / 2; ++j) kk[j] = min(kk[j], kk[j + m / 2]);
        idx = __reduce_min_sync(FULL, kk[0]) & 0xffffu;
    } else {
        uint32_t kk[J], jj[J];
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const auto x = s.v(j);
            hb |= (HB)P::hd(x) << j;
            kk[j] = P::mag_key(x);
            jj[j] = j;
        }
        // adjacent pairs (j, j + s): every slot on the left holds lower indices than its
        // partner's, so keeping the left on equal keys keeps the lowest index
#pragma unroll
        for (int st = 1; st < J; st *= 2)
#pragma unroll
            for (int j = 0; j + st < J; j += 2 * st) {
                const bool r = kk[j + st] < kk[j];
                kk[j] = r ? kk[j + st] : kk[j];
                jj[j] = r ? jj[j + st] : jj[j];
            }
        const uint32_t mn = __reduce_min_sync(FULL, kk[0]);
        idx = __reduce_min_sync(FULL, kk[0] == mn ? jj[0] * 32u + lane_id() : 0xffffffffu);
    }
    const uint32_t parity = __popc(__ballot_sync(FULL, __popcll((uint64_t)hb) & 1)) & 1u;
    if (parity && lane_id() == (idx & 31u)) hb ^= (HB)1 << (idx >> 5);
    bw |= (uint64_t)hb << s0;
}

// ---------------------------------------------------- subtree decisions as warp-uniform words
// BW<NW>: the decision bits of a warp subtree of 32*NW values as NW words, w[s] bit l =
// beta[l + 32 s] -- the natural bit array itself, the same in every lane (ballots, XORs of
// ballots).  The alternative (one 64-bit word per lane, bit s = beta[lane + 32 s]) needs a
// transpose of ballots at the subtree's end and 64-bit shifts in every leaf and combine; here
// a Rate-1 slot is one ballot, a combine one XOR per word, a replicated node's mask is stored as
// is, and the store is lane 0 writing the words.  Used for subtrees up to 512 values (codegen).
template <int NW>
struct BW {
    uint32_t w[NW];
};
// sign-bit mask of this lane's bit of word x (beta[lane + 32 s] << 31)
PD_INLINE uint32_t lane_sgn(uint32_t x) { return (x << (31u - lane_id())) & 0x80000000u; }

template <class P, int n, int s0, class Src, int NW>
PD_INLINE void wG(const Src& s, typename P::v_t* c, const BW<NW>& bw, uint32_t ml) {
    if constexpr (n >= 64) {
#pragma unroll
        for (int j = 0; j < n / 64; ++j) c[j] = P::gs(s.v(j), s.v(j + n / 64), lane_sgn(bw.w[s0 + j]));
        PD_DUMPR(n, c);
    } else {
        wG<P, n, s0>(s, c, (uint64_t)0, ml);
    }
}
template <class P, int n, int s0, class Src, int NW>
PD_INLINE void wR1(const Src& s, BW<NW>& bw) {
    static_assert(n >= 64, "");
#pragma unroll
    for (int j = 0; j < n / 32; ++j) bw.w[s0 + j] = __ballot_sync(FULL, P::hd(s.v(j)));
}
template <class P, int n, int s0, class Src, int NW>
PD_INLINE void wRep(const Src& s, BW<NW>& bw) {
    static_assert(n >= 64, "");
    const uint32_t m = wRepDecide<P, n>(s) ? FULL : 0u;
#pragma unroll
    for (int j = 0; j < n / 32; ++j) bw.w[s0 + j] = m;
}
// SPC with the hard decisions as ballot words; the flip of the lowest-index least
// reliable bit (C10) lands in the word idx / 32 by an unrolled select.
template <class P, int n, int s0, class Src, int NW>
PD_INLINE void wSPC(const Src& s, BW<NW>& bw) {
    static_assert(n >= 64, "");
    constexpr int J = n / 32;
    uint32_t hw[J], par = 0, idx;
    if constexpr (P::kPackedKey) {
        uint32_t kk[J];
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const auto x = s.v(j);
            hw[j] = __ballot_sync(FULL, P::hd(x));
            par ^= hw[j];
            kk[j] = spc_key16(x, (uint32_t)(j * 32) | lane_id());
        }
#pragma unroll
        for (int m = J; m > 1; m /= 2)
#pragma unroll
            for (int j = 0; j < m / 2; ++j) kk[j] = min(kk[j], kk[j + m / 2]);
        idx = __reduce_min_sync(FULL, kk[0]) & 0xffffu;
    } else {
        uint32_t kk[J], jj[J];
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const auto x = s.v(j);
            hw[j] = __ballot_sync(FULL, P::hd(x));
            par ^= hw[j];
            kk[j] = P::mag_key(x);
            jj[j] = j;
        }
#pragma unroll
        for (int st = 1; st < J; st *= 2)
#pragma unroll
            for (int j = 0; j + st < J; j += 2 * st) {
                const bool r = kk[j + st] < kk[j];
                kk[j] = r ? kk[j + st] : kk[j];
                jj[j] = r ? jj[j + st] : jj[j];
            }
        const uint32_t mn = __reduce_min_sync(FULL, kk[0]);
        idx = __reduce_min_sync(FULL, kk[0] == mn ? jj[0] * 32u + lane_id() : 0xffffffffu);
    }
    const uint32_t flip = (__popc(par) & 1u) << (idx & 31u);
#pragma unroll
    for (int j = 0; j < J; ++j) bw.w[s0 + j] = hw[j] ^ ((idx >> 5) == (uint32_t)j ? flip : 0u);
}
template <int s, int NW>
PD_INLINE void wDeposit(BW<NW>& bw, uint32_t m) {
    bw.w[s] = m;
}
template <int n, int s0, int NW>
PD_INLINE void wComb(BW<NW>& bw) {
#pragma unroll
    for (int k = 0; k < n / 64; ++k) bw.w[s0 + k] ^= bw.w[s0 + n / 64 + k];
}
template <int n, int s0, int NW>
PD_INLINE void wComb0R(BW<NW>& bw) {
#pragma unroll
    for (int k = 0; k < n / 64; ++k) bw.w[s0 + k] |= bw.w[s0 + n / 64 + k];
}
template <int R, int NW>
PD_INLINE void wStoreBeta(const BW<NW>& bw, uint32_t* words) {
    static_assert(R / 32 == NW, "");
    if (lane_id() == 0) {
        if constexpr (NW >= 4) {
#pragma unroll
            for (int g = 0; g < NW / 4; ++g)
                *reinterpret_cast<uint4*>(words + 4 * g) = make_uint4(bw.w[4 * g], bw.w[4 * g + 1], bw.w[4 * g + 2], bw.w[4 * g + 3]);
        } else {
#pragma unroll
            for (int k = 0; k < NW; ++k) words[k] = bw.w[k];
        }
    }
}
// A subtree that is the right child of a CTA-level node also performs that node's Combine
// (eq:combine P:318-325) while its words are still in registers: left words ^= right words, or
// left = right for Combine_0R (ZL, the left child was Rate-0 and left its words zero).  Replaces
// the CTA-level combine op and its barrier.
template <int R, bool ZL, int NW>
PD_INLINE void wStoreBetaComb(const BW<NW>& bw, uint32_t* words, uint32_t* left) {
    static_assert(R / 32 == NW, "");
    if (lane_id() == 0) {
        if constexpr (NW >= 4) {
#pragma unroll
            for (int g = 0; g < NW / 4; ++g) {
                const uint4 r = make_uint4(bw.w[4 * g], bw.w[4 * g + 1], bw.w[4 * g + 2], bw.w[4 * g + 3]);
                *reinterpret_cast<uint4*>(words + 4 * g) = r;
                if constexpr (ZL) {
                    *reinterpret_cast<uint4*>(left + 4 * g) = r;
                } else {
                    const uint4 l = *reinterpret_cast<const uint4*>(left + 4 * g);
                    *reinterpret_cast<uint4*>(left + 4 * g) = make_uint4(l.x ^ r.x, l.y ^ r.y, l.z ^ r.z, l.w ^ r.w);
                }
            }
        } else {
#pragma unroll
            for (int k = 0; k < NW; ++k) {
                words[k] = bw.w[k];
                left[k] = ZL ? bw.w[k] : (left[k] ^ bw.w[k]);
            }
        }
    }
}
// shared subtree functions of 64 values return their two words packed in 64 bits
template <int s0, int NW>
PD_INLINE void wSetWords64(BW<NW>& bw, uint64_t m) {
    bw.w[s0] = (uint32_t)m;
    bw.w[s0 + 1] = (uint32_t)(m >> 32);
}

// RepSPC<n>: a node whose left child is a repetition code and right child an SPC
// code, decoded speculatively as the paper describes -- the repetition code and two instances
// of the SPC code, one assuming the repetition output is all 0's and the other all 1's, run
// side by side, and the repetition decision selects.  Bit-identical to the composition
// F<n>, Repetition<n/2>, G<n>, SPC<n/2>, Combine<n> (same f/g arithmetic, operands and sum
// order); the G with beta = 1 is b - a, with beta = 0 b + a.  Replicated nodes (n <= 32).
template <class P, int n, class Src>
PD_INLINE uint32_t wRepSPCm(const Src& s) {
    static_assert(n >= 4 && n <= 32, "");
    constexpr int h = n / 2;
    using V = typename P::v_t;
    V x, y;
    s.pair(h, x, y);  // own element (lane mod n) and the partner (xor h)
    V cf[1] = {P::f(x, y)};  // F: the left child, replicated (lane holds element lane mod h)
    PD_DUMPR(n, cf);
    const bool second = lane_id() & h;  // lanes holding alpha[i + h]
    const V a = second ? y : x, b = second ? x : y;
    V g0[1] = {P::g0(a, b)}, g1[1] = {P::g(a, b, 1u)};  // G for beta_l = 0 and 1
    const uint32_t m0 = wSPCm<P, h>(RegSrc<P>{g0});
    const uint32_t m1 = wSPCm<P, h>(RegSrc<P>{g1});
    const bool r = wRepDecide<P, h>(RegSrc<P>{cf});  // the repetition decision selects
#ifdef POLAR_DEBUG_DUMP
    V gs[1] = {r ? g1[0] : g0[0]};
    PD_DUMPR(n, gs);
#endif
    const uint32_t ml = r ? low_mask(h) : 0u, mr = r ? m1 : m0;
    return (ml ^ mr) | (mr << h);
}

// ------------------------------------------------------- lane-local tiny subtrees (n <= 16)
// A split node of a few elements is decoded inside every lane: its n values (replicated, lane
// k holds element k) are gathered once with n independent shuffles, then the whole subtree
// runs on compile-time-indexed registers with no further cross-lane latency; every lane
// computes the same beta mask (bit i = beta[i]).  Same op order as the warp versions.
template <class P, int n>
PD_INLINE void lGather(typename P::v_t x, typename P::v_t* q) {
#pragma unroll
    for (int k = 0; k < n; ++k) q[k] = __shfl_sync(FULL, x, k);
}
template <class P, int n>
PD_INLINE void lF(const typename P::v_t* a, typename P::v_t* c) {
#pragma unroll
    for (int i = 0; i < n / 2; ++i) c[i] = P::f(a[i], a[i + n / 2]);
}
template <class P, int n>
PD_INLINE void lG(const typename P::v_t* a, typename P::v_t* c, uint32_t ml) {
#pragma unroll
    for (int i = 0; i < n / 2; ++i) c[i] = P::g(a[i], a[i + n / 2], (ml >> i) & 1u);
}
template <class P, int n>
PD_INLINE void lG0R(const typename P::v_t* a, typename P::v_t* c) {
#pragma unroll
    for (int i = 0; i < n / 2; ++i) c[i] = P::g0(a[i], a[i + n / 2]);
}
template <class P, int n>
PD_INLINE uint32_t lR1(const typename P::v_t* a) {
    uint32_t m = 0;
#pragma unroll
    for (int i = 0; i < n; ++i) m |= (uint32_t)P::hd(a[i]) << i;
    return m;
}
template <class P, int n>
PD_INLINE uint32_t lRep(const typename P::v_t* a) {
    typename P::acc_t t[n];
#pragma unroll
    for (int i = 0; i < n; ++i) t[i] = P::acc(a[i]);
#pragma unroll
    for (int m = n; m > 1; m /= 2)
#pragma unroll
        for (int i = 0; i < m / 2; ++i) t[i] = P::add(t[i], t[i + m / 2]);
    return P::acc_neg(t[0]) ? low_mask(n) : 0u;
}
template <class P, int n>
PD_INLINE uint32_t lSPC(const typename P::v_t* a) {
    uint32_t h = 0, best = 0xffffffffu, idx = 0;
#pragma unroll
    for (int i = 0; i < n; ++i) {
        h |= (uint32_t)P::hd(a[i]) << i;
        const uint32_t k = P::mag_key(a[i]);
        if (k < best) { best = k; idx = i; }
    }
    return h ^ ((__popc(h) & 1u) << idx);
}

// Place the mask of a finished 32-bit node into bw slot s.
template <int s>
PD_INLINE void wDeposit(uint64_t& bw, uint32_t m) {
    bw |= (uint64_t)((m >> lane_id()) & 1u) << s;
}

// Combine<n> / Combine_0R<n> on bw (n >= 64), eq:combine P:318-325:
// left half of beta ^= right half; 0R: left half = right half (left was all zero).
template <int n, int s0>
PD_INLINE void wComb(uint64_t& bw) {
    constexpr int h = n / 64;
    constexpr uint64_t L = (((h == 64) ? ~0ull : ((1ull << h) - 1ull))) << s0;
    bw ^= (bw >> h) & L;
}
template <int n, int s0>
PD_INLINE void wComb0R(uint64_t& bw) {
    constexpr int h = n / 64;
    constexpr uint64_t L = (((h == 64) ? ~0ull : ((1ull << h) - 1ull))) << s0;
    bw |= (bw >> h) & L;
}

// Write the beta of a finished warp subtree of size R >= 32 into the natural bit array:
// word k (bits k*32 .. k*32+31 of the subtree) is the ballot of bw bit k.  The ballots are
// warp-uniform, so every lane holds all NW words and lanes 0.. store them as 16-byte groups: two
// instructions per word (predicate + vote) instead of seven (64-bit shift/compare, vote,
// per-lane select), measured 658 -> ~150 cycles per 512-subtree on the batch-1 path.
template <int R>
PD_INLINE void wStoreBeta(uint64_t bw, uint32_t* words) {
    static_assert(R >= 32 && R <= 2048, "");
    constexpr int NW = R / 32;
    const uint32_t lo = (uint32_t)bw, hi = (uint32_t)(bw >> 32);
    uint32_t wd[NW];
#pragma unroll
    for (int k = 0; k < NW; ++k) wd[k] = __ballot_sync(FULL, ((k < 32 ? lo : hi) >> (k & 31)) & 1u);
    // lane 0 stores them all (one predicate; a per-lane choice of group compiled to a jump table)
    if (lane_id() == 0) {
        if constexpr (NW >= 4) {
#pragma unroll
            for (int g = 0; g < NW / 4; ++g)
                *reinterpret_cast<uint4*>(words + 4 * g) = make_uint4(wd[4 * g], wd[4 * g + 1], wd[4 * g + 2], wd[4 * g + 3]);
        } else {
#pragma unroll
            for (int k = 0; k < NW; ++k) words[k] = wd[k];
        }
    }
}

// ------------------------------------------------------------------ CTA-scope operations
// T threads; n > W >= 64; src/dst are shared-memory (or, for the f32 channel, global)
// stages of the node; beta is the node's first word of the natural bit array.

// CLAMP: the source is the channel (int8 -128 -> -127, reading C8); stages never need it.
// SS / DS: state spaces of source and destination.  F32OUT: int8 profile writing the f32
// subtree-input stage.  Every distinct instance is one non-inlined function shared by all
// call sites of the unrolled decoder (the stage ops are loops; inlining ~100 of them made
// the N = 32768 kernels ~40% larger, profiles/r1_history.md).
// Software-pipelined: the loads of U iterations are issued before any of their stores, so a
// global (L2) stage keeps 2U 16-byte loads in flight per thread.
template <class P, int H, int T>
__host__ __device__ constexpr int stage_unroll() {
    constexpr int step = chunk_elems<P, H, T>() * T;
#ifndef POLAR_STAGE_U
#define POLAR_STAGE_U 4
#endif
    constexpr int umax = T == 32 ? POLAR_STAGE_U : 1;  // the latency CTA (shared-memory stages, 128-register cap) needs none
    return H / step >= umax ? umax : H / step >= 2 ? 2 : 1;
}
template <class P, int T, int n, bool CLAMP, int SS, int DS, class S, class D>
PD_INLINE void cF_body(const void* src, void* dst) {
    constexpr int H = n / 2, CE = chunk_elems<P, H, T>(), STEP = CE * T, U = stage_unroll<P, H, T>();
    constexpr int LH = CLAMP ? L2_FIRST : L2_LAST;
#pragma unroll 1
    for (int i0 = CE * gtid<T>(); i0 < H; i0 += STEP * U) {
        Chunk<P, CE> a[U], b[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i0 + u * STEP < H) {
                a[u].template load_raw<SS, LH>((const S*)src + i0 + u * STEP);
                b[u].template load_raw<SS, LH>((const S*)src + i0 + u * STEP + H);
            }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i0 + u * STEP < H) {
                a[u].template unpack_raw<S>(CLAMP);
                b[u].template unpack_raw<S>(CLAMP);
                chunk_f(a[u], b[u]);
                a[u].template store<DS, L2_LAST>((D*)dst + i0 + u * STEP);
            }
    }
}
template <class P, int T, int n, bool CLAMP, bool ZERO_LEFT, int SS, int DS, class S, class D>
PD_INLINE void cG_body(const void* src, void* dst, const uint32_t* beta) {
    constexpr int H = n / 2, CE = chunk_elems<P, H, T>(), STEP = CE * T, U = stage_unroll<P, H, T>();
    constexpr int LH = CLAMP ? L2_FIRST : L2_LAST;
#pragma unroll 1
    for (int i0 = CE * gtid<T>(); i0 < H; i0 += STEP * U) {
        Chunk<P, CE> a[U], b[U];
        uint32_t bits[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i0 + u * STEP < H) {
                const int i = i0 + u * STEP;
                a[u].template load_raw<SS, LH>((const S*)src + i);
                b[u].template load_raw<SS, LH>((const S*)src + i + H);
                bits[u] = ZERO_LEFT ? 0u : beta[i >> 5] >> (i & 31);
            }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i0 + u * STEP < H) {
                a[u].template unpack_raw<S>(CLAMP);
                b[u].template unpack_raw<S>(CLAMP);
                if constexpr (ZERO_LEFT) chunk_g0(a[u], b[u]);
                else chunk_g(a[u], b[u], bits[u]);
                a[u].template store<DS, L2_LAST>((D*)dst + i0 + u * STEP);
            }
    }
}
// Fused descent (XK then YK): X<n> of the node (F, G or G_0R) immediately followed by the first
// op of its CTA-level child, Y<n/2> (F, or G_0R when the child's left child is Rate-0), on the
// outputs X just produced.  Element i of Y's output needs X outputs i and i + n/4, i.e. the node
// values i, i + n/4, i + n/2, i + 3n/4: each thread loads those four chunks, computes both X
// chunks, stores them (the child's alpha, read again by its G later) and applies Y to them in
// registers -- the child stage is written but not re-read and re-unpacked, and one op boundary
// disappears.  Same f/g arithmetic and operands as the two ops it replaces.
enum : int { OP_F = 0, OP_G = 1, OP_G0R = 2 };
template <int K, class P, int CE>
PD_INLINE void chunk_op(Chunk<P, CE>& a, const Chunk<P, CE>& b, uint32_t bits) {
    if constexpr (K == OP_F) chunk_f(a, b);
    else if constexpr (K == OP_G) chunk_g(a, b, bits);
    else chunk_g0(a, b);
}
template <class P, int T, int n, bool CLAMP, int XK, int YK, int SS, int DS, int DS2, class S, class D, class D2>
PD_INLINE void cXY_body(const void* src, void* dst, void* dst2, const uint32_t* beta) {
    constexpr int Q = n / 4, CE = chunk_elems<P, Q, T>(), STEP = CE * T;
    constexpr int U = (T == 32 && Q / STEP >= 2) ? 2 : 1;
    constexpr int LH = CLAMP ? L2_FIRST : L2_LAST;
#pragma unroll 1
    for (int i0 = CE * gtid<T>(); i0 < Q; i0 += STEP * U) {
        Chunk<P, CE> a0[U], b0[U], a1[U], b1[U];
        uint32_t bits0[U], bits1[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i0 + u * STEP < Q) {
                const int i = i0 + u * STEP;
                a0[u].template load_raw<SS, LH>((const S*)src + i);
                b0[u].template load_raw<SS, LH>((const S*)src + i + 2 * Q);
                a1[u].template load_raw<SS, LH>((const S*)src + i + Q);
                b1[u].template load_raw<SS, LH>((const S*)src + i + 3 * Q);
                bits0[u] = XK == OP_G ? beta[i >> 5] >> (i & 31) : 0u;
                bits1[u] = XK == OP_G ? beta[(i + Q) >> 5] >> ((i + Q) & 31) : 0u;
            }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i0 + u * STEP < Q) {
                const int i = i0 + u * STEP;
                a0[u].template unpack_raw<S>(CLAMP);
                b0[u].template unpack_raw<S>(CLAMP);
                chunk_op<XK>(a0[u], b0[u], bits0[u]);
                a1[u].template unpack_raw<S>(CLAMP);
                b1[u].template unpack_raw<S>(CLAMP);
                chunk_op<XK>(a1[u], b1[u], bits1[u]);
                a0[u].template store<DS, L2_LAST>((D*)dst + i);
                a1[u].template store<DS, L2_LAST>((D*)dst + i + Q);
                chunk_op<YK>(a0[u], a1[u], 0u);
                a0[u].template store<DS2, L2_LAST>((D2*)dst2 + i);
            }
    }
}
template <class P, int T, int n, bool CLAMP, int XK, int YK, int SS, int DS, int DS2, class S, class D, class D2>
__device__ __noinline__ void cXY_impl(const void* src, void* dst, void* dst2, const uint32_t* beta) {
    cXY_body<P, T, n, CLAMP, XK, YK, SS, DS, DS2, S, D, D2>(src, dst, dst2, beta);
}
template <class P, int T, int n, bool CLAMP, int XK, int YK, int SS, int DS, int DS2, bool NI, class TS, class TD, class TD2>
PD_INLINE void cXY(const TS* src, TD* dst, TD2* dst2, const uint32_t* beta) {
    if constexpr (NI) cXY_impl<P, T, n, CLAMP, XK, YK, SS, DS, DS2, TS, TD, TD2>(src, dst, dst2, beta);
    else cXY_body<P, T, n, CLAMP, XK, YK, SS, DS, DS2, TS, TD, TD2>(src, dst, dst2, beta);
}

// Three-level fused descent: X<n>, then Y<n/2> on X's outputs, then Z<n/4> on Y's outputs (Y, Z:
// F, or G_0R when the node's left child is Rate-0), all CTA-level.  Element i of Z's output needs
// node values i + k n/8 (k = 0..7): eight chunk loads per thread, the X, Y and Z outputs stored
// (each is the alpha of a node whose G reads it later), none re-read.
// The int8 channel versions (the two root ops, streaming the frame from HBM) are software-
// pipelined: the eight 8-byte chunks of the next step are loaded before the current step is
// computed, so each HBM round trip overlaps the previous step's work.
// one step of cXYZ_pipe: compute the chunks in raw (step at i), after refilling raw with the
// step PD steps later (its loads stay in flight while this step computes)
template <class P, int n, bool CLAMP, int XK, int YK, int ZK, int DS, int DS2, int DS3, int PD, class S, class D, class D2,
          class D3>
PD_INLINE void cXYZ_pipe_step(int i, uint32_t (&raw)[8][2], const void* src, void* dst, void* dst2, void* dst3,
                              const uint32_t* beta) {
    constexpr int R = n / 8, CE = 8, STEP = CE * 32;
    constexpr int LH = CLAMP ? L2_FIRST : L2_LAST;
    Chunk<P, CE> a[4], b[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        a[k].w[0] = raw[k][0];
        a[k].w[1] = raw[k][1];
        b[k].w[0] = raw[k + 4][0];
        b[k].w[1] = raw[k + 4][1];
    }
    if (i + PD * STEP < R) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
            vld<SP_GLOBAL, 8, LH>((const S*)src + i + PD * STEP + (k & 3) * R + (k >> 2) * 4 * R, raw[k]);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t bits = XK == OP_G ? beta[(i + k * R) >> 5] >> ((i + k * R) & 31) : 0u;
        a[k].template unpack_raw<S>(CLAMP);
        b[k].template unpack_raw<S>(CLAMP);
        chunk_op<XK>(a[k], b[k], bits);
        a[k].template store<DS, L2_LAST>((D*)dst + i + k * R);
    }
    chunk_op<YK>(a[0], a[2], 0u);
    a[0].template store<DS2, L2_LAST>((D2*)dst2 + i);
    chunk_op<YK>(a[1], a[3], 0u);
    a[1].template store<DS2, L2_LAST>((D2*)dst2 + i + R);
    chunk_op<ZK>(a[0], a[1], 0u);
    a[0].template store<DS3, L2_LAST>((D3*)dst3 + i);
}
template <class P, int n, bool CLAMP, int XK, int YK, int ZK, int DS, int DS2, int DS3, class S, class D, class D2, class D3>
PD_INLINE void cXYZ_pipe(const void* src, void* dst, void* dst2, void* dst3, const uint32_t* beta) {
    constexpr int R = n / 8, CE = 8, STEP = CE * 32;
    constexpr int LH = CLAMP ? L2_FIRST : L2_LAST;
#ifndef POLAR_PIPE_DEPTH
#define POLAR_PIPE_DEPTH 1  // 2: two steps in flight (measured: 500 bytes of spills in the kernel)
#endif
    constexpr int PD = (POLAR_PIPE_DEPTH == 2 && R / STEP >= 2 && (R / STEP) % 2 == 0) ? 2 : 1;
    // the chunks of the next PD steps: k = 0..3 (node values i + kR), 4..7 (+ 4R)
    uint32_t raw0[8][2], raw1[8][2];
    int i = CE * (int)lane_id();
#pragma unroll
    for (int k = 0; k < 8; ++k) vld<SP_GLOBAL, 8, LH>((const S*)src + i + (k & 3) * R + (k >> 2) * 4 * R, raw0[k]);
    if constexpr (PD == 2) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
            vld<SP_GLOBAL, 8, LH>((const S*)src + i + STEP + (k & 3) * R + (k >> 2) * 4 * R, raw1[k]);
    }
#pragma unroll 1
    for (; i < R; i += PD * STEP) {
        cXYZ_pipe_step<P, n, CLAMP, XK, YK, ZK, DS, DS2, DS3, PD, S, D, D2, D3>(i, raw0, src, dst, dst2, dst3, beta);
        if constexpr (PD == 2)
            cXYZ_pipe_step<P, n, CLAMP, XK, YK, ZK, DS, DS2, DS3, PD, S, D, D2, D3>(i + STEP, raw1, src, dst, dst2, dst3, beta);
    }
}
template <class P, int T, int n, bool CLAMP, int XK, int YK, int ZK, int SS, int DS, int DS2, int DS3, class S, class D,
          class D2, class D3>
PD_INLINE void cXYZ_body(const void* src, void* dst, void* dst2, void* dst3, const uint32_t* beta) {
    constexpr int R = n / 8, CE = chunk_elems<P, R, T>(), STEP = CE * T;
    constexpr int LH = CLAMP ? L2_FIRST : L2_LAST;
    // the channel ops only: pipelining the L2-stage readers too (8-byte chunks) measured -1.2%
    constexpr bool kPipe = CLAMP && SS == SP_GLOBAL && T == 32 && sizeof(S) == 1 && R % 256 == 0;
    if constexpr (kPipe) {
        cXYZ_pipe<P, n, CLAMP, XK, YK, ZK, DS, DS2, DS3, S, D, D2, D3>(src, dst, dst2, dst3, beta);
        return;
    }
#pragma unroll 1
    for (int i = CE * gtid<T>(); i < R; i += STEP) {
        Chunk<P, CE> a[4], b[4];
        uint32_t bits[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            a[k].template load_raw<SS, LH>((const S*)src + i + k * R);
            b[k].template load_raw<SS, LH>((const S*)src + i + k * R + 4 * R);
            bits[k] = XK == OP_G ? beta[(i + k * R) >> 5] >> ((i + k * R) & 31) : 0u;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            a[k].template unpack_raw<S>(CLAMP);
            b[k].template unpack_raw<S>(CLAMP);
            chunk_op<XK>(a[k], b[k], bits[k]);
            a[k].template store<DS, L2_LAST>((D*)dst + i + k * R);
        }
        chunk_op<YK>(a[0], a[2], 0u);
        a[0].template store<DS2, L2_LAST>((D2*)dst2 + i);
        chunk_op<YK>(a[1], a[3], 0u);
        a[1].template store<DS2, L2_LAST>((D2*)dst2 + i + R);
        chunk_op<ZK>(a[0], a[1], 0u);
        a[0].template store<DS3, L2_LAST>((D3*)dst3 + i);
    }
}
template <class P, int T, int n, bool CLAMP, int XK, int YK, int ZK, int SS, int DS, int DS2, int DS3, class S, class D,
          class D2, class D3>
__device__ __noinline__ void cXYZ_impl(const void* src, void* dst, void* dst2, void* dst3, const uint32_t* beta) {
    cXYZ_body<P, T, n, CLAMP, XK, YK, ZK, SS, DS, DS2, DS3, S, D, D2, D3>(src, dst, dst2, dst3, beta);
}
template <class P, int T, int n, bool CLAMP, int XK, int YK, int ZK, int SS, int DS, int DS2, int DS3, bool NI, class TS,
          class TD, class TD2, class TD3>
PD_INLINE void cXYZ(const TS* src, TD* dst, TD2* dst2, TD3* dst3, const uint32_t* beta) {
    if constexpr (NI) cXYZ_impl<P, T, n, CLAMP, XK, YK, ZK, SS, DS, DS2, DS3, TS, TD, TD2, TD3>(src, dst, dst2, dst3, beta);
    else cXYZ_body<P, T, n, CLAMP, XK, YK, ZK, SS, DS, DS2, DS3, TS, TD, TD2, TD3>(src, dst, dst2, dst3, beta);
}

template <class P, int T, int n, bool CLAMP, int SS, int DS, class S, class D>
__device__ __noinline__ void cF_impl(const void* src, void* dst) {
    cF_body<P, T, n, CLAMP, SS, DS, S, D>(src, dst);
}
template <class P, int T, int n, bool CLAMP, bool ZERO_LEFT, int SS, int DS, class S, class D>
__device__ __noinline__ void cG_impl(const void* src, void* dst, const uint32_t* beta) {
    cG_body<P, T, n, CLAMP, ZERO_LEFT, SS, DS, S, D>(src, dst, beta);
}
// NI: call the shared non-inlined instance (throughput variant of large codes); otherwise
// inline (the call costs latency on the batch-1 critical path).
template <class P, int T, int n, bool CLAMP, int SS, int DS, bool NI, class TS, class TD>
PD_INLINE void cF(const TS* src, TD* dst) {
    if constexpr (NI) cF_impl<P, T, n, CLAMP, SS, DS, TS, TD>(src, dst);
    else cF_body<P, T, n, CLAMP, SS, DS, TS, TD>(src, dst);
}
template <class P, int T, int n, bool CLAMP, bool ZERO_LEFT, int SS, int DS, bool NI, class TS, class TD>
PD_INLINE void cG(const TS* src, TD* dst, const uint32_t* beta) {
    if constexpr (NI) cG_impl<P, T, n, CLAMP, ZERO_LEFT, SS, DS, TS, TD>(src, dst, beta);
    else cG_body<P, T, n, CLAMP, ZERO_LEFT, SS, DS, TS, TD>(src, dst, beta);
}
template <class P, int T, int n, bool CLAMP, int SS, int DS, bool NI, class TS, class TD>
PD_INLINE void cG0R(const TS* src, TD* dst) {
    cG<P, T, n, CLAMP, true, SS, DS, NI>(src, dst, nullptr);
}
// ---- packed-byte leaves on biased int8 stages (byte u = v + 128, never -128: stages only)
// 16 consecutive elements per thread and step (one 16-byte shared load).  v < 0 <=> bit 7 of u
// is clear; the four sign bits of a word gather into a nibble by one multiply (the partial
// products of 0x00204081 land on distinct bits, so there are no carries); 16 decision bits are
// stored as one 16-bit half of a beta word (little-endian: half 2k is bits 0-15 of word k).
PD_INLINE uint32_t hd16_biased(const uint32_t* w) {
    uint32_t h = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) h |= ((((~w[j]) & 0x80808080u) * 0x00204081u) >> 28) << (4 * j);
    return h;
}
template <int T, int n>
PD_INLINE void cR1_b(const uint8_t* __restrict__ src, uint32_t* beta) {
    static_assert(n % 16 == 0, "");
    for (int i = 16 * gtid<T>(); i < n; i += 16 * T) {
        const uint4 v4 = *reinterpret_cast<const uint4*>(src + i);  // generic: the stage may be in L2 scratch
        const uint32_t w[4] = {v4.x, v4.y, v4.z, v4.w};
        reinterpret_cast<uint16_t*>(beta)[i >> 4] = (uint16_t)hd16_biased(w);
    }
}
// SPC on a biased int8 stage: decisions as above; |v| = |u - 128| is one byte
// absolute difference per 4 values (vabsdiff4); the least reliable position is found on 16-bit
// keys (|v| << 8 | position in the thread's 16) by packed u16x2 minima, the lowest position winning
// ties (reading C10), then on 32-bit keys (|v| << 16 | element index) across the group.
template <int T, int n>
PD_INLINE void cSPC_b(const uint8_t* __restrict__ src, uint32_t* beta) {
    static_assert(n % 16 == 0 && n <= 65536, "");
    uint32_t best = 0xffffffffu, p = 0;
    for (int i = 16 * gtid<T>(); i < n; i += 16 * T) {
        const uint4 v4 = *reinterpret_cast<const uint4*>(src + i);  // generic: the stage may be in L2 scratch
        const uint32_t w[4] = {v4.x, v4.y, v4.z, v4.w};
        const uint32_t h = hd16_biased(w);
        reinterpret_cast<uint16_t*>(beta)[i >> 4] = (uint16_t)h;
        p ^= __popc(h);
        uint32_t k[8];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t m = __vabsdiffu4(w[j], 0x80808080u);  // |v| of the 4 bytes
            const uint32_t ix = 0x03020100u + 0x04040404u * j;    // their positions in the 16
            k[2 * j] = __byte_perm(m, ix, 0x1504);                // (|v0| << 8 | p0, |v1| << 8 | p1)
            k[2 * j + 1] = __byte_perm(m, ix, 0x3726);            // (|v2| << 8 | p2, |v3| << 8 | p3)
        }
#pragma unroll
        for (int m = 8; m > 1; m /= 2)
#pragma unroll
            for (int j = 0; j < m / 2; ++j) k[j] = __vminu2(k[j], k[j + m / 2]);
        const uint32_t k16 = min(k[0] & 0xffffu, k[0] >> 16);
        best = min(best, ((k16 >> 8) << 16) | (uint32_t)(i + (int)(k16 & 0xffu)));
    }
    best = __reduce_min_sync(FULL, best);
    p = __reduce_xor_sync(FULL, p) & 1u;
    if constexpr (T > 32) {
        __shared__ uint32_t redk[T / 32], par[T / 32];
        const int warp = gtid<T>() >> 5;
        if (lane_id() == 0) {
            redk[warp] = best;
            par[warp] = p;
        }
        group_sync<T>();
        best = __reduce_min_sync(FULL, lane_id() < T / 32 ? redk[lane_id()] : 0xffffffffu);
        p = __reduce_xor_sync(FULL, lane_id() < T / 32 ? par[lane_id()] : 0u) & 1u;
    }
    group_sync<T>();
    if (gtid<T>() == 0 && p) {
        const uint32_t idx = best & 0xffffu;
        beta[idx >> 5] ^= 1u << (idx & 31);
    }
    group_sync<T>();
}

template <class P, int T, int n, class TS>
PD_INLINE void cR1(const TS* __restrict__ src, uint32_t* beta) {
    if constexpr (same_t<TS, uint8_t>::value && n % 16 == 0) {
        cR1_b<T, n>(src, beta);
    } else {
        for (int k = (gtid<T>() >> 5); k < n / 32; k += T / 32) {
            const uint32_t w = __ballot_sync(FULL, P::hd(P::ld(src[32 * k + lane_id()])));
            if (lane_id() == 0) beta[k] = w;
        }
    }
}
// Repetition at CTA scope.  f32: pairwise-halving order (reading C13) run in
// place on `scratch` (the free child stage of size n/2); int8: exact integer sum.  A lone
// warp (T = 32, possibly one of several frame groups of a CTA) reduces with shuffles only.
template <class P, int T, int n, class TS, class TSc>
PD_INLINE void cRep(const TS* __restrict__ src, TSc* scratch, uint32_t* beta) {
    using A = typename P::acc_t;
    bool decision;
    if constexpr (P::kExactSum) {
        A s = 0;
        for (int i = gtid<T>(); i < n; i += T) s = P::add(s, P::acc(P::ld(src[i])));
#pragma unroll
        for (int o = 16; o; o >>= 1) s = P::add(s, __shfl_xor_sync(FULL, s, o));
        if constexpr (T == 32) {
            decision = P::acc_neg(s);
        } else {
            __shared__ A red[T / 32];
            if (lane_id() == 0) red[gtid<T>() >> 5] = s;
            group_sync<T>();
            A tot = lane_id() < T / 32 ? red[lane_id()] : A(0);  // exact: integer-valued, |sum| < 2^24
#pragma unroll
            for (int o = 16; o; o >>= 1) tot = P::add(tot, __shfl_xor_sync(FULL, tot, o));
            decision = P::acc_neg(tot);
        }
    } else {
        for (int i = gtid<T>(); i < n / 2; i += T) scratch[i] = P::st(P::add(P::ld(src[i]), P::ld(src[i + n / 2])));
        group_sync<T>();
        for (int m = n / 2; m > 32; m /= 2) {
            for (int i = gtid<T>(); i < m / 2; i += T) scratch[i] = P::add(scratch[i], scratch[i + m / 2]);
            group_sync<T>();
        }
        A t = scratch[lane_id()];  // every warp reduces the last 32 values the same way
#pragma unroll
        for (int o = 16; o; o >>= 1) t = P::add(t, __shfl_down_sync(FULL, t, o));
        decision = __shfl_sync(FULL, (int)P::acc_neg(t), 0) != 0;
    }
    const uint32_t w = decision ? FULL : 0u;
    for (int k = gtid<T>(); k < n / 32; k += T) beta[k] = w;
    group_sync<T>();
}

// SPC at CTA scope: ballot hard decisions per word, parity of all, flip the
// lowest-index least-magnitude bit when odd (reading C10); key = (|alpha| << 32) | index.
template <class P, int T, int n, class TS>
PD_INLINE void cSPC_w(const TS* __restrict__ src, uint32_t* beta);
template <class P, int T, int n, class TS>
PD_INLINE void cSPC(const TS* __restrict__ src, uint32_t* beta) {
    if constexpr (same_t<TS, uint8_t>::value && n % 16 == 0 && n <= 65536) cSPC_b<T, n>(src, beta);
    else cSPC_w<P, T, n>(src, beta);
}
// SPC with one element per lane and step (f32, f16 or channel sources)
template <class P, int T, int n, class TS>
PD_INLINE void cSPC_w(const TS* __restrict__ src, uint32_t* beta) {
    const int warp = (gtid<T>() >> 5);
    if constexpr (P::kPackedKey) {
        // int8: one 32-bit key (|alpha| f32 bits | index) per element, exact (see wSPCm);
        // redux.min per warp, then over the warps
        uint32_t best = 0xffffffffu, p = 0;
        for (int k = warp; k < n / 32; k += T / 32) {
            const auto x = P::ld(src[32 * k + lane_id()]);
            const uint32_t w = __ballot_sync(FULL, P::hd(x));
            if (lane_id() == 0) beta[k] = w;
            p ^= __popc(w) & 1u;
            best = min(best, P::mag_key(x) | (uint32_t)(32 * k + lane_id()));
        }
        best = __reduce_min_sync(FULL, best);
        if constexpr (T > 32) {
            __shared__ uint32_t redk[T / 32], par[T / 32];
            if (lane_id() == 0) {
                redk[warp] = best;
                par[warp] = p;
            }
            group_sync<T>();
            best = __reduce_min_sync(FULL, lane_id() < T / 32 ? redk[lane_id()] : 0xffffffffu);
            p = __popc(__ballot_sync(FULL, lane_id() < T / 32 ? (par[lane_id()] & 1u) : 0u)) & 1u;
        }
        group_sync<T>();
        if (gtid<T>() == 0 && p) {
            const uint32_t idx = best & 0xffffu;
            beta[idx >> 5] ^= 1u << (idx & 31);
        }
        group_sync<T>();
        return;
    }
    unsigned long long best = ~0ull;
    uint32_t p = 0;
    for (int k = warp; k < n / 32; k += T / 32) {
        const auto x = P::ld(src[32 * k + lane_id()]);
        const uint32_t w = __ballot_sync(FULL, P::hd(x));
        if (lane_id() == 0) beta[k] = w;
        p ^= __popc(w) & 1u;
        const unsigned long long key = ((unsigned long long)P::mag_key(x) << 32) | (uint32_t)(32 * k + lane_id());
        best = key < best ? key : best;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(FULL, best, o);
        best = other < best ? other : best;
    }
    if constexpr (T > 32) {
        __shared__ unsigned long long red[T / 32];
        __shared__ uint32_t par[T / 32];
        if (lane_id() == 0) {
            red[warp] = best;
            par[warp] = p;
        }
        group_sync<T>();
        best = lane_id() < T / 32 ? red[lane_id()] : ~0ull;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const unsigned long long other = __shfl_xor_sync(FULL, best, o);
            best = other < best ? other : best;
        }
        p = __popc(__ballot_sync(FULL, lane_id() < T / 32 ? (par[lane_id()] & 1u) : 0u)) & 1u;
    }
    group_sync<T>();
    if (gtid<T>() == 0 && p) {
        const uint32_t idx = (uint32_t)best;
        beta[idx >> 5] ^= 1u << (idx & 31);
    }
    group_sync<T>();
}

template <int T, int n>
PD_INLINE void cComb(uint32_t* beta) {
    for (int k = gtid<T>(); k < n / 64; k += T) beta[k] ^= beta[k + n / 64];
}
template <int T, int n>
PD_INLINE void cComb0R(uint32_t* beta) {
    for (int k = gtid<T>(); k < n / 64; k += T) beta[k] = beta[k + n / 64];
}

// ----------------------------------------------------------------------- frame output
// Systematic information bits x_hat[A] (reading C4/C5), packed LSB-first, A ascending.
// x_hat[A] is the codeword with the frozen positions squeezed out: for every codeword word k
// the information bits are pext(beta[k], imask[k]) and land at bit offset prefix[k] of the
// output (tab = {imask[0..NB), prefix[0..NB)}, NB = max(1, N/32), built at create time).
// The group's threads take codeword words k = tid, tid + T, ... and OR their runs into the
// shared staging words `stg` (ceil(K/32) words), which are then stored coalesced.
PD_INLINE uint32_t pext32(uint32_t x, uint32_t m) {
    if (m == 0xffffffffu) return x;
    uint32_t r = 0, at = 0;
    while (m) {
        const uint32_t s = __ffs(m) - 1;          // start of the lowest run of ones
        const uint32_t t = ~(m >> s);             // zeros where the run continues
        const uint32_t len = t ? __ffs(t) - 1 : 32 - s;
        const uint32_t lm = len >= 32 ? 0xffffffffu : ((1u << len) - 1u);
        r |= ((x >> s) & lm) << at;
        at += len;
        m &= ~(lm << s);
    }
    return r;
}

// Non-systematic output (reading C4): u_hat = x_hat G_N, computed in place on the N-bit array
// (x G_N: x[j] ^= x[j | d] for every bit d of the index, G_N[i][j] = [j subset of i])
// by the T threads of the frame group; the information bits are then u_hat[A].
template <int N, int T>
PD_INLINE void beta_transform(uint32_t* beta) {
    constexpr int NW = N >= 32 ? N / 32 : 1;
    constexpr uint32_t in_word[5] = {0x55555555u, 0x33333333u, 0x0F0F0F0Fu, 0x00FF00FFu, 0x0000FFFFu};
#pragma unroll
    for (int b = 0; b < 5; ++b) {
        if ((1 << b) >= N) break;
        for (int k = gtid<T>(); k < NW; k += T) {
            const uint32_t x = beta[k];
            beta[k] = x ^ ((x >> (1 << b)) & in_word[b]);
        }
        group_sync<T>();
    }
    for (int D = 1; D < NW; D <<= 1) {
        for (int k = gtid<T>(); k < NW; k += T)
            if (!(k & D)) beta[k] ^= beta[k | D];
        group_sync<T>();
    }
}

// Lane-interleaved piece-table gather (tab after the {imask, prefix} words, built at create
// time, polar_api.cu): output word q of x_hat[A] is the OR of its pieces -- maximal runs of
// consecutive information positions inside one output word ((32768,29492): 1,413 pieces for 922
// words) -- each a uint2 {lo << 16 | (hi - lo) << 5 | s, destination mask}: the run's bits are
// bits s.. of the 64-bit pair (beta[hi] : beta[lo]) (hi = lo + 1 when the run crosses a codeword
// word, else hi = lo and the funnel shift is a rotation).  Output words are taken 32 at a time
// (group g = words 32g .. 32g+31, one per lane); piece j of every word of a group is one
// coalesced 256-byte row, so a group's loads are independent of each other; a group holds as
// many rows as its longest word, rounded up to even (padding pieces have mask 0); hdr[g] = its
// first row, hdr[NG] = the total.  (r1/r2 form: per-word offsets, then uint4 pieces -- two
// dependent L2 loads per output word, 10% of the warp-stall samples of the (32768,29492)
// throughput kernel, profiles/r2n_tp32k.txt.)
__host__ __device__ constexpr int gather_hdr_words(int N, int K) {
    return (((K + 31) / 32 + 31) / 32 + 1 + 3) & ~3;
}
PD_INLINE uint32_t gather_piece(const uint32_t* beta, uint2 d) {
    const uint32_t lo = d.x >> 16, hi = lo + ((d.x >> 5) & 1u);
    return __funnelshift_r(beta[lo], beta[hi], d.x) & d.y;  // the shift is taken mod 32
}
template <int N, int K, int T>
PD_INLINE void gather_info(const uint32_t* beta, const uint32_t* __restrict__ tab, uint32_t* stg,
                           uint32_t* __restrict__ out) {
    (void)stg;
    constexpr int NB = N >= 32 ? N / 32 : 1;
    constexpr int NWK = (K + 31) / 32;
    constexpr int NG = (NWK + 31) / 32;
    constexpr int TB = (2 * NB + 3) & ~3;  // the {imask, prefix} words, padded
    const uint32_t* __restrict__ hdr = tab + TB;
    const uint2* __restrict__ pcs = reinterpret_cast<const uint2*>(tab + TB + gather_hdr_words(N, K)) + lane_id();
    // the first rows of groups 0..31 in one coalesced load, handed out by shuffles
    const uint32_t hv = lane_id() <= (unsigned)NG ? __ldg(hdr + lane_id()) : 0u;
    if constexpr (T == 32 && NG >= 4 && NG < 32) {  // (2048,1723), NG = 2: the per-group loop measured faster
        // one warp takes every group: the rows of all groups are consecutive, so they stream
        // through a register window PF rows ahead across group boundaries (a group's word is
        // complete when its last row pair has been consumed); no load waits on a computation
        constexpr int PF = 8;
        const int total = (int)__shfl_sync(FULL, hv, NG);
        uint2 d[PF];
#pragma unroll
        for (int u = 0; u < PF; ++u) d[u] = u < total ? __ldg(pcs + 32 * u) : make_uint2(0u, 0u);
        const uint2* p = pcs + 32 * PF;
        int gi = 0, gend = (int)__shfl_sync(FULL, hv, 1);
        uint32_t acc = 0;
        for (int r = 0; r < total; r += 2, p += 64) {
            acc |= gather_piece(beta, d[0]) | gather_piece(beta, d[1]);
#pragma unroll
            for (int u = 0; u < PF - 2; ++u) d[u] = d[u + 2];
            d[PF - 2] = r + PF < total ? __ldg(p) : make_uint2(0u, 0u);
            d[PF - 1] = r + PF + 1 < total ? __ldg(p + 32) : make_uint2(0u, 0u);
            if (r + 2 == gend) {
                const int q = 32 * gi + (int)lane_id();
                if (q < NWK) out[q] = acc;
                acc = 0;
                ++gi;
                gend = (int)__shfl_sync(FULL, hv, gi + 1);
            }
        }
        return;
    }
    for (int g = gtid<T>() >> 5; g < NG; g += T / 32) {
        const int r0 = (int)(g < 32 ? __shfl_sync(FULL, hv, g) : __ldg(hdr + g));
        const int r1 = (int)(g + 1 < 32 ? __shfl_sync(FULL, hv, g + 1) : __ldg(hdr + g + 1));
        const uint2* p = pcs + 32 * r0;
        uint32_t acc = 0;
        int r = r0;
        for (; r + 4 <= r1; r += 4, p += 128) {  // four rows in flight
            const uint2 d0 = __ldg(p), d1 = __ldg(p + 32), d2 = __ldg(p + 64), d3 = __ldg(p + 96);
            acc |= gather_piece(beta, d0) | gather_piece(beta, d1) | gather_piece(beta, d2) | gather_piece(beta, d3);
        }
        if (r < r1) {  // rows come in pairs
            const uint2 d0 = __ldg(p), d1 = __ldg(p + 32);
            acc |= gather_piece(beta, d0) | gather_piece(beta, d1);
        }
        const int q = 32 * g + (int)lane_id();
        if (q < NWK) out[q] = acc;
    }
}

// --------------------------------------------------------------- TMA bulk ingest helpers
PD_INLINE uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

PD_INLINE void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
PD_INLINE void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
PD_INLINE void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// One elected thread: expect `bytes` on bar and start a bulk global->shared copy
// (cp.async.bulk, completes on the mbarrier; bytes % 16 == 0, 16-B aligned addresses).
PD_INLINE void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

PD_INLINE void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    const uint32_t a = smem_u32(bar);
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    } while (!done);
}

}  // namespace pd
