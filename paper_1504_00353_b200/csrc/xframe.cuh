// xframe.cuh -- frame-interleaved (one lane = one frame) Fast-SSC building blocks, int8.
//
// Giard et al., arXiv:1504.00353 vectorise ONE frame across the SIMD lanes (P:580-582,
// P:790-795) and hence pay for the small nodes near the leaves, where a vector is mostly
// idle.  On a B200 the throughput variant can instead give every lane of a warp its own
// frame: the 32 frames of a warp run the same unrolled operation list (codegen.cpp, emitted
// per code exactly as the warp-cooperative decoders), so every lane does useful work at every
// node size, and there is no shuffle, ballot or barrier anywhere in the decode.
//
// Layout (per warp, lane-private data, so no synchronisation is ever needed):
//  * a stage of m int8 LLRs (the paper's alpha buffer of that level) is stored
//    as m/16 chunks of 16 bytes; chunk c of lane l is at byte c*512 + l*16, so a 16-byte
//    vector access of the 32 lanes is one contiguous 512-byte transaction (shared memory:
//    4 conflict-free wavefronts; global scratch: 4 full lines);
//  * the channel LLRs are read in place from the frame-major input ([n][N] int8);
//  * beta (the codeword estimate) is N/32 words per frame, word w of lane l at
//    w*32 + l;
//  * nodes of N_v <= 32 run on f32 registers holding the integers (lF/lG/lR1/lRep/lSPC of
//    decoder.cuh: exact, same op order as the oracle); stage ops on N_v >= 64 compute in
//    integer-valued f16x2 (XChunk: exact for |values| <= 254; the stages hold x + 128).
#pragma once

#include "decoder.cuh"

#ifndef XF_NI_SOP
#define XF_NI_SOP 128  // stage ops on nodes of at least this size are shared non-inlined loops
#endif
#ifndef XF_NI_LV
#define XF_NI_LV 64    // likewise for stage leaves
#endif

namespace pd {
namespace xf {

enum : int { CH = 0, SM = 1, GL = 2 };  // where an alpha stage lives: channel, shared, global

// Per-lane base pointers of the frame being decoded.
struct Ctx {
    const int8_t* chan;  // this lane's frame, natural order
    int8_t* sm;          // shared stage area + lane*16
    int8_t* gl;          // global stage slot + lane*16
    uint32_t* beta;      // beta words + lane
};

// The base pointers pass through an opaque move at every use: otherwise ptxas hoists the
// hundreds of loop-invariant stage and beta addresses of the unrolled decoder out of the
// frame loop and keeps them all live (255 registers and spills at N = 32768).
template <class T>
PD_INLINE T* launder(T* p) {
    asm volatile("" : "+l"(p));
    return p;
}
PD_INLINE uint32_t* bword(const Ctx& x, int w) { return launder(x.beta) + 32 * w; }

// Address of chunk c of a stage at byte offset OFF of its space.
template <int S, int OFF>
PD_INLINE const int8_t* cptr(const Ctx& x, int c) {
    if constexpr (S == CH) return launder(x.chan) + 16 * c;
    else if constexpr (S == SM) return launder(x.sm) + OFF + 512 * c;
    else return launder(x.gl) + OFF + 512 * c;
}
template <int S, int OFF>
PD_INLINE int8_t* wptr(const Ctx& x, int c) {
    static_assert(S != CH, "");
    if constexpr (S == SM) return launder(x.sm) + OFF + 512 * c;
    else return launder(x.gl) + OFF + 512 * c;
}
template <int S>
__host__ __device__ constexpr int space() { return S == SM ? SP_SHARED : SP_GLOBAL; }
// L2 hints: the channel is streamed once per root op (evict_first); stage scratch is re-read
template <int S>
__host__ __device__ constexpr int hint() { return S == CH ? L2_FIRST : S == GL ? L2_LAST : L2_NORMAL; }


// ------------------------------------------------------------- stage -> stage operations
// F<n> (eq:f), G<n> (eq:g with the left child's beta), G_0R<n>:
// the parent (n values, at S/SO) produces the child (n/2 values, at D/DO).  The channel
// parent (S == CH) reads -128 as -127 (reading C8).  U consecutive chunks of both halves are
// loaded before any is used (the accesses are volatile asm, so the compiler keeps their
// order): 2U loads in flight per lane, and each lane reads 16U contiguous bytes of the
// frame-major channel (whole 64-byte DRAM bursts at U = 4).
enum : int { OP_F = 0, OP_G = 1, OP_G0R = 2 };

// 16 int8 LLRs of one chunk, computed as integer-valued f16x2 (exact, |values| <= 254).
// XF_BIASED: the decoder's own stages hold x + 128 (bytes 1..255), so unpacking is one PRMT
// and one HADD2 per pair and packing drops the sign flip; the channel stays plain int8
// (-128 read as -127, reading C8).
#ifndef XF_BIASED
#define XF_BIASED 1
#endif
struct XChunk {
    uint32_t w[4];
    uint32_t h[8];
    template <int S>
    PD_INLINE void load(const int8_t* p) { vld<space<S>(), 16, hint<S>()>(p, w); }
    template <int S>
    PD_INLINE void unpack() {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t t = (S == CH || !XF_BIASED) ? w[q] ^ 0x80808080u : w[q];
            h[2 * q] = h2add(__byte_perm(t, 0x64646464u, 0x4140), 0xE480E480u);
            h[2 * q + 1] = h2add(__byte_perm(t, 0x64646464u, 0x4342), 0xE480E480u);
            if constexpr (S == CH) {
                h[2 * q] = h2max(h[2 * q], 0xD7F0D7F0u);
                h[2 * q + 1] = h2max(h[2 * q + 1], 0xD7F0D7F0u);
            }
        }
    }
    template <int D>
    PD_INLINE void store(int8_t* p) const {
        uint32_t o[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
            o[q] = __byte_perm(h2add(h[2 * q], 0x64806480u), h2add(h[2 * q + 1], 0x64806480u), 0x6420) ^
                   (XF_BIASED ? 0u : 0x80808080u);
        vst<space<D>(), 16, hint<D>()>(p, o);
    }
    PD_INLINE void f(const XChunk& b) {
#pragma unroll
        for (int q = 0; q < 8; ++q) h[q] = h2minxs(h[q], b.h[q]);
    }
    // h = sat(b + (beta ? -h : h)); bit k of bits = beta of element k (see Chunk<PI8>::g)
    PD_INLINE void g(const XChunk& b, uint32_t bits) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint32_t m = (((bits >> (2 * q)) & 3u) * 0x40008000u) & 0x80008000u;
            h[q] = h2minxs(h2add(b.h[q], h[q] ^ m), 0x57F057F0u);
        }
    }
    PD_INLINE void g0(const XChunk& b) {
#pragma unroll
        for (int q = 0; q < 8; ++q) h[q] = h2minxs(h2add(b.h[q], h[q]), 0x57F057F0u);
    }
};
// A stage word of 4 LLRs as signed bytes (for the leaves)
template <int S>
PD_INLINE uint32_t sbytes(uint32_t w) { return (S == CH || !XF_BIASED) ? w : w ^ 0x80808080u; }

// p: the parent's chunk 0 (channel: this lane's frame; stage: its interleaved base + lane*16)
template <int S>
PD_INLINE const int8_t* chunk_at(const int8_t* p, int c) { return p + (S == CH ? 16 : 512) * c; }
template <int S>
PD_INLINE int8_t* chunk_at(int8_t* p, int c) { return p + 512 * c; }

// p: parent chunk 0, d: child chunk 0, bw: the left child's first beta word (OP_G)
template <int OP, int n, int S, int D>
PD_INLINE void sOp_impl(const int8_t* p, int8_t* d, const uint32_t* bw) {
    constexpr int H = n / 32;  // chunks of the child
    constexpr int U = H < 4 ? H : 4;
#pragma unroll 1
    for (int c0 = 0; c0 < H; c0 += U) {
        XChunk a[U], b[U];
#pragma unroll
        for (int u = 0; u < U; ++u) a[u].template load<S>(chunk_at<S>(p, c0 + u));
#pragma unroll
        for (int u = 0; u < U; ++u) b[u].template load<S>(chunk_at<S>(p, c0 + u + H));
        uint32_t bits[(U + 1) / 2];
        if constexpr (OP == OP_G) {
#pragma unroll
            for (int k = 0; k < (U + 1) / 2; ++k) bits[k] = bw[32 * (c0 / 2 + k)];
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            a[u].template unpack<S>();
            b[u].template unpack<S>();
            if constexpr (OP == OP_F) a[u].f(b[u]);
            else if constexpr (OP == OP_G0R) a[u].g0(b[u]);
            else a[u].g(b[u], (bits[u / 2] >> (16 * (u & 1))) & 0xffffu);
            a[u].template store<D>(chunk_at<D>(d, c0 + u));
        }
    }
}
// Large nodes: one shared non-inlined loop per (op, size, spaces) keeps the unrolled decoder
// small (instruction fetch, compile time, registers); small ones stay inline.
template <int OP, int n, int S, int D>
__device__ __noinline__ void sOp_ni(const int8_t* p, int8_t* d, const uint32_t* bw) { sOp_impl<OP, n, S, D>(p, d, bw); }
template <int OP, int n, int S, int D>
PD_INLINE void sOp(const int8_t* p, int8_t* d, const uint32_t* bw) {
    if constexpr (n >= XF_NI_SOP) sOp_ni<OP, n, S, D>(p, d, bw);
    else sOp_impl<OP, n, S, D>(p, d, bw);
}
template <int n, int S, int SO, int D, int DO>
PD_INLINE void sF(const Ctx& x) { sOp<OP_F, n, S, D>(cptr<S, SO>(x, 0), wptr<D, DO>(x, 0), nullptr); }
template <int n, int S, int SO, int D, int DO>
PD_INLINE void sG(const Ctx& x, int bl) { sOp<OP_G, n, S, D>(cptr<S, SO>(x, 0), wptr<D, DO>(x, 0), bword(x, bl / 32)); }
template <int n, int S, int SO, int D, int DO>
PD_INLINE void sG0R(const Ctx& x) { sOp<OP_G0R, n, S, D>(cptr<S, SO>(x, 0), wptr<D, DO>(x, 0), nullptr); }

// --------------------------------------------------------- stage -> registers (n == 64)
// The 32 child values of a 64-node go straight into f32 registers.
PD_INLINE void h2_to_f32(const uint32_t* h, float* q) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const float2 v = __half22float2(*reinterpret_cast<const __half2*>(&h[k]));
        q[2 * k] = v.x;
        q[2 * k + 1] = v.y;
    }
}
template <int OP, int S>
PD_INLINE void rOp(const int8_t* p, float* q, uint32_t ml) {
    XChunk a[2], b[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) a[c].template load<S>(chunk_at<S>(p, c));
#pragma unroll
    for (int c = 0; c < 2; ++c) b[c].template load<S>(chunk_at<S>(p, c + 2));
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        a[c].template unpack<S>();
        b[c].template unpack<S>();
        if constexpr (OP == OP_F) a[c].f(b[c]);
        else if constexpr (OP == OP_G0R) a[c].g0(b[c]);
        else a[c].g(b[c], (ml >> (16 * c)) & 0xffffu);
        h2_to_f32(a[c].h, q + 16 * c);
    }
}
template <int S>
PD_INLINE void rF(const int8_t* p, float* q) { rOp<OP_F, S>(p, q, 0u); }
template <int S>
PD_INLINE void rG(const int8_t* p, float* q, uint32_t ml) { rOp<OP_G, S>(p, q, ml); }
template <int S>
PD_INLINE void rG0R(const int8_t* p, float* q) { rOp<OP_G0R, S>(p, q, 0u); }

// Whole frame in registers (N <= 32): the channel values, -128 read as -127.
template <int n>
PD_INLINE void rChan(const Ctx& x, float* q) {
#pragma unroll
    for (int i = 0; i < n; ++i) q[i] = PI8::ld(x.chan[i]);
}

// ------------------------------------------------------------------ beta words
PD_INLINE void stB(const Ctx& x, int w, uint32_t m) { *bword(x, w) = m; }
PD_INLINE uint32_t ldB(const Ctx& x, int w) { return x.beta[32 * w]; }

// Combine<n> (eq:combine) in place on the words of the node at bit offset b:
// left half ^= right half; Combine_0R: left half = right half; Zero: a Rate-0 right half
// (reading C16).  n >= 64, so both halves are whole words.
template <int n>
PD_INLINE void bComb(const Ctx& x, int b) {
    constexpr int HW = n / 64;
    uint32_t* bp = bword(x, b / 32);
#pragma unroll 8
    for (int k = 0; k < HW; ++k) bp[32 * k] ^= bp[32 * (HW + k)];
}
template <int n>
PD_INLINE void bComb0R(const Ctx& x, int b) {
    constexpr int HW = n / 64;
    uint32_t* bp = bword(x, b / 32);
#pragma unroll 8
    for (int k = 0; k < HW; ++k) bp[32 * k] = bp[32 * (HW + k)];
}
template <int nw>
PD_INLINE void bZero(const Ctx& x, int w0) {
    uint32_t* bp = bword(x, w0);
#pragma unroll 8
    for (int k = 0; k < nw; ++k) bp[32 * k] = 0u;
}

// ------------------------------------------------------------------ stage leaves (n >= 64)
// Hard decisions of 4 int8 values: bit j = sign bit of byte j (value < 0, eq:info P:444-449;
// integers, so no signed zero).
PD_INLINE uint32_t hd4(uint32_t w) { return (((w >> 7) & 0x01010101u) * 0x10204080u) >> 28; }

// Leaves on a stage (n >= 64): p = the node's chunk 0, bp = its first beta word.
// Rate-1: beta = HD(alpha).
template <int n, int S>
PD_INLINE void lvR1_impl(const int8_t* p, uint32_t* bp) {
#pragma unroll 4
    for (int c = 0; c < n / 16; c += 2) {
        uint32_t w[2][4];
#pragma unroll
        for (int h = 0; h < 2; ++h) vld<space<S>(), 16, hint<S>()>(chunk_at<S>(p, c + h), w[h]);
        uint32_t m = 0;
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int q = 0; q < 4; ++q) m |= hd4(sbytes<S>(w[h][q])) << (16 * h + 4 * q);
        bp[32 * (c / 2)] = m;
    }
}

// Repetition: all bits = (sum < 0), the exact integer sum (reading C12), the
// channel's -128 read as -127.
template <int n, int S>
PD_INLINE void lvRep_impl(const int8_t* p, uint32_t* bp) {
    int s = 0;
#pragma unroll 4
    for (int c = 0; c < n / 16; ++c) {
        uint32_t w[4];
        vld<space<S>(), 16, hint<S>()>(chunk_at<S>(p, c), w);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t v = S == CH ? (uint32_t)__vmaxs4(w[q], 0x81818181u) : sbytes<S>(w[q]);
            s = __dp4a((int)v, 0x01010101, s);
        }
    }
    const uint32_t m = s < 0 ? 0xffffffffu : 0u;
#pragma unroll 8
    for (int k = 0; k < n / 32; ++k) bp[32 * k] = m;
}

// SPC: beta = HD; if the parity is odd, flip the least reliable bit (lowest
// index on ties, reading C10).  key = |alpha| << 16 | index (|alpha| <= 127 after the clamp).
template <int n, int S>
PD_INLINE void lvSPC_impl(const int8_t* p, uint32_t* bp) {
    uint32_t par = 0, best = 0xffffffffu;
#pragma unroll 2
    for (int c = 0; c < n / 16; c += 2) {
        uint32_t w[2][4];
#pragma unroll
        for (int h = 0; h < 2; ++h) vld<space<S>(), 16, hint<S>()>(chunk_at<S>(p, c + h), w[h]);
        uint32_t m = 0;
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t sw = sbytes<S>(w[h][q]);
                m |= hd4(sw) << (16 * h + 4 * q);
                const uint32_t a = __vabsss4(sw);  // |v|, -128 -> 127 (the clamp's magnitude)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t key = (((a >> (8 * j)) & 0xffu) << 16) | (uint32_t)(16 * (c + h) + 4 * q + j);
                    best = min(best, key);
                }
            }
        par ^= m;
        bp[32 * (c / 2)] = m;
    }
    if (__popc(par) & 1u) {
        const int i = (int)(best & 0xffffu);
        bp[32 * (i >> 5)] ^= 1u << (i & 31);
    }
}

template <int K, int n, int S>
__device__ __noinline__ void lv_ni(const int8_t* p, uint32_t* bp) {
    if constexpr (K == 0) lvR1_impl<n, S>(p, bp);
    else if constexpr (K == 1) lvRep_impl<n, S>(p, bp);
    else lvSPC_impl<n, S>(p, bp);
}
template <int K, int n, int S, int SO>
PD_INLINE void lv(const Ctx& x, int b) {
    const int8_t* p = cptr<S, SO>(x, 0);
    uint32_t* bp = bword(x, b / 32);
    if constexpr (n >= XF_NI_LV) lv_ni<K, n, S>(p, bp);
    else if constexpr (K == 0) lvR1_impl<n, S>(p, bp);
    else if constexpr (K == 1) lvRep_impl<n, S>(p, bp);
    else lvSPC_impl<n, S>(p, bp);
}
template <int n, int S, int SO>
PD_INLINE void lvR1(const Ctx& x, int b) { lv<0, n, S, SO>(x, b); }
template <int n, int S, int SO>
PD_INLINE void lvRep(const Ctx& x, int b) { lv<1, n, S, SO>(x, b); }
template <int n, int S, int SO>
PD_INLINE void lvSPC(const Ctx& x, int b) { lv<2, n, S, SO>(x, b); }

// ------------------------------------------------------------------ frame output
// x_hat[A] packed LSB-first, A ascending (readings C4, C5): per codeword word k the
// information bits pext(beta[k], imask[k]) are appended; tab = {imask[NB], prefix[NB]}.
template <int N, int K>
PD_INLINE void gather_store(const Ctx& x, const uint32_t* __restrict__ tab, uint32_t* __restrict__ out) {
    constexpr int NB = N >= 32 ? N / 32 : 1;
    uint64_t acc = 0;
    int nacc = 0, q = 0;
    for (int k = 0; k < NB; ++k) {
        const uint32_t m = __ldg(tab + k);
        if (!m) continue;
        const uint32_t w = ldB(x, k);
        const uint32_t r = m == 0xffffffffu ? w : pext32(w, m);
        acc |= (uint64_t)r << nacc;
        nacc += __popc(m);
        if (nacc >= 32) {
            out[q++] = (uint32_t)acc;
            acc >>= 32;
            nacc -= 32;
        }
    }
    if (nacc > 0) out[q] = (uint32_t)acc;
}

}  // namespace xf

// k_xf<C, WPC>: WPC warps per CTA, each decoding 32 frames at a time (frame = 32 g + lane),
// persistent grid over frame groups g.  Lanes past the last frame decode a copy of it and
// store nothing.  gscratch: one slot of C::GSLOT bytes per warp of the grid.
template <class C, int WPC, int MINB>
__global__ void __launch_bounds__(32 * WPC, MINB)
    k_xf(const void* __restrict__ llr_, long long n_frames, uint32_t* __restrict__ out,
         const uint32_t* __restrict__ gtab, void* __restrict__ gscratch) {
    extern __shared__ __align__(128) unsigned char smem_all[];
    const int w = (int)(threadIdx.x >> 5);
    const int lane = (int)(threadIdx.x & 31u);
    const int8_t* llr = (const int8_t*)llr_;
    unsigned char* const sw = smem_all + w * C::SMEM_WARP;
    const long long slot = (long long)blockIdx.x * WPC + w;
    // gscratch: a 256-byte header holding the group counter (zeroed by the host before each
    // launch), then one slot of C::GSLOT bytes per warp of the grid
    unsigned long long* const gctr = (unsigned long long*)gscratch;
    unsigned char* const gw = (unsigned char*)gscratch + 256 + slot * C::GSLOT;
    xf::Ctx x;
    x.sm = (int8_t*)sw + 16 * lane;
    x.gl = (int8_t*)gw + 16 * lane;
    x.beta = (C::BETA_GL ? (uint32_t*)(gw + C::GSTAGE) : (uint32_t*)(sw + C::SSTAGE)) + lane;
    constexpr int NWK = (C::K + 31) / 32;
    const long long groups = (n_frames + 31) / 32;
    // after its first group each warp takes the next one from the counter (dynamic scheduling:
    // the groups in flight stay a compact window and the last wave balances)
    for (long long g = slot; g < groups;) {
        const long long f = 32 * g + lane;
        const long long fc = f < n_frames ? f : n_frames - 1;
        x.chan = llr + fc * C::N;
        C::decode(x);
        if (f < n_frames) xf::gather_store<C::N, C::K>(x, gtab, out + f * NWK);
        long long nxt = 0;
        if (lane == 0) nxt = (long long)gridDim.x * WPC + (long long)atomicAdd(gctr, 1ull);
        g = __shfl_sync(0xffffffffu, nxt, 0);
    }
}

}  // namespace pd
