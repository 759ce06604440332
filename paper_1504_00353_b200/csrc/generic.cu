// generic.cu -- the program-interpreted Fast-SSC decoder for any frozen set (N <= 32768).
//
// The paper has two decoder builders: the unrolled decoder generated per code (P:633-864,
// our build-time specialisation) and the instruction-based decoder that reads the list of
// operations at run time.  This is the latter: polar_code_create
// falls back to it for frozen sets no decoder was specialised for, so the ABI accepts every
// (N, K, mask).  One warp per frame, all stages in shared memory (stage(m) at N - 2m), beta
// as the natural bit array; the op list is tree.hpp::program().  Same f/g/leaf arithmetic
// and op order as the specialised kernels (decoder.cuh), so results are identical.
#include "decoder.cuh"
#include "tree.hpp"

namespace pd {
using namespace polar;  // OP_* opcodes of tree.hpp

__host__ __device__ inline int g_align16(int x) { return (x + 15) & ~15; }

template <class P>
__host__ __device__ inline int generic_smem(int N, int K) {
    const int stages = g_align16((N > 1 ? N - 1 : 1) * (int)sizeof(typename P::st_t));
    const int nb = N >= 32 ? N / 32 : 1;
    return stages + 4 * nb + 4 * ((K + 31) / 32) + 16;
}

// Write n < 32 bits (LSB-first) into the natural bit array at bit `off` (one word).
PD_INLINE void put_bits(uint32_t* beta, int off, int n, uint32_t bits) {
    const uint32_t m = low_mask(n) << (off & 31);
    uint32_t& w = beta[off >> 5];
    w = (w & ~m) | ((bits << (off & 31)) & m);
}

template <class P>
__global__ void __launch_bounds__(32) k_generic(const void* __restrict__ llr_, long long n_frames,
                                                uint32_t* __restrict__ out, const uint32_t* __restrict__ gtab,
                                                const uint32_t* __restrict__ prog, int n_ops, int N, int K,
                                                unsigned flags) {
    using S = typename P::st_t;
    using V = typename P::v_t;
    extern __shared__ __align__(16) unsigned char gsmem[];
    S* const st = (S*)gsmem;
    const int NB = N >= 32 ? N / 32 : 1;
    const int NWK = (K + 31) / 32;
    uint32_t* const beta = (uint32_t*)(gsmem + g_align16((N > 1 ? N - 1 : 1) * (int)sizeof(S)));
    uint32_t* const stg = beta + NB;
    using Ch = typename P::in_t;  // the channel (signed int8 or f32); stages are S (int8: biased bytes)
    const Ch* llr = (const Ch*)llr_;
    const int l = lane_id();
    for (long long f = blockIdx.x; f < n_frames; f += gridDim.x) {
        const Ch* chan = llr + f * N;
        for (int k = l; k < NB; k += 32) beta[k] = 0;
        __syncwarp();
        for (int pc = 0; pc < n_ops; ++pc) {
            const uint32_t w = __ldg(prog + pc);
            const int op = w & 15, n = 1 << ((w >> 4) & 31), off = (int)(w >> 9), h = n >> 1;
            const bool root = n == N;  // the root op reads the channel (uniform per op)
            const S* srcs = root ? st : st + (N - 2 * n);
            auto src_ld = [&](int i) -> V { return root ? P::ld(chan[i]) : P::ld(srcs[i]); };
            S* dst = st + (N - n);  // stage(n/2)
            switch (op) {
                case OP_F:
                    for (int i = l; i < h; i += 32) dst[i] = P::st(P::f(src_ld(i), src_ld(i + h)));
                    break;
                case OP_G:
                    for (int i = l; i < h; i += 32)
                        dst[i] = P::st(P::g(src_ld(i), src_ld(i + h), (beta[(off + i) >> 5] >> ((off + i) & 31)) & 1u));
                    break;
                case OP_G0R:
                    for (int i = l; i < h; i += 32) dst[i] = P::st(P::g0(src_ld(i), src_ld(i + h)));
                    break;
                case OP_R1:
                    for (int i0 = 0; i0 < n; i0 += 32) {
                        const uint32_t b = __ballot_sync(FULL, i0 + l < n && P::hd(src_ld(i0 + l)));
                        if (l == 0) {
                            if (n >= 32) beta[(off + i0) >> 5] = b;
                            else put_bits(beta, off, n, b);
                        }
                    }
                    break;
                case OP_REP: {
                    // repetition: the decision is [sum < 0]
                    bool neg;
                    if constexpr (P::kExactSum) {  // int8: exact, any order (reading C12)
                        typename P::acc_t t = 0;
                        for (int i = l; i < n; i += 32) t = P::add(t, P::acc(src_ld(i)));
#pragma unroll
                        for (int o = 16; o; o >>= 1) t = P::add(t, __shfl_xor_sync(FULL, t, o));
                        neg = P::acc_neg(t);
                    } else {  // f32: pairwise halving order (reading C13)
                        typename P::acc_t t;
                        int start;
                        if (n <= 32) {
                            t = P::acc(src_ld(l & (n - 1)));
                            start = h;
                        } else {
                            for (int i = l; i < h; i += 32) dst[i] = P::add(src_ld(i), src_ld(i + h));
                            __syncwarp();
                            for (int m = h; m > 32; m >>= 1) {
                                for (int i = l; i < m / 2; i += 32) dst[i] = P::add(dst[i], dst[i + m / 2]);
                                __syncwarp();
                            }
                            t = dst[l];
                            start = 16;
                        }
                        for (int o = start; o >= 1; o >>= 1) t = P::add(t, __shfl_xor_sync(FULL, t, o));
                        neg = P::acc_neg(t);
                    }
                    if (n >= 32) {
                        for (int k = l; k < n / 32; k += 32) beta[(off >> 5) + k] = neg ? FULL : 0u;
                    } else if (l == 0) {
                        put_bits(beta, off, n, neg ? FULL : 0u);
                    }
                    break;
                }
                case OP_SPC: {
                    // SPC: hard decisions, parity, flip the lowest-index least
                    // magnitude when the parity is odd (readings C10, C11)
                    uint32_t par = 0, best = 0xffffffffu, bi = 0xffffffffu;
                    for (int i0 = 0; i0 < n; i0 += 32) {
                        const int i = i0 + l;
                        const bool in = i < n;
                        const V x = in ? src_ld(i) : V(0);
                        const uint32_t b = __ballot_sync(FULL, in && P::hd(x));
                        par ^= __popc(b) & 1u;
                        if (l == 0) {
                            if (n >= 32) beta[(off + i0) >> 5] = b;
                            else put_bits(beta, off, n, b);
                        }
                        const uint32_t k = in ? P::mag_key(x) : 0xffffffffu;
                        if (k < best) { best = k; bi = i; }
                    }
                    uint32_t idx;
                    if constexpr (P::kPackedKey) {
                        idx = __reduce_min_sync(FULL, best == 0xffffffffu ? best : (best | bi)) & 0xffffu;
                    } else {
                        const uint32_t mn = __reduce_min_sync(FULL, best);
                        idx = __reduce_min_sync(FULL, best == mn ? bi : 0xffffffffu);
                    }
                    __syncwarp();
                    if (l == 0 && par) beta[(off + idx) >> 5] ^= 1u << ((off + idx) & 31);
                    break;
                }
                case OP_COMB:
                case OP_COMB0R:
                    if (n >= 64) {
                        for (int k = l; k < n / 64; k += 32) {
                            const uint32_t r = beta[(off >> 5) + n / 64 + k];
                            beta[(off >> 5) + k] = op == OP_COMB ? beta[(off >> 5) + k] ^ r : r;
                        }
                    } else if (l == 0) {
                        const uint32_t wv = beta[off >> 5];
                        const uint32_t r = (wv >> ((off & 31) + h)) & low_mask(h);
                        const uint32_t left = op == OP_COMB ? ((wv >> (off & 31)) & low_mask(h)) ^ r : r;
                        put_bits(beta, off, h, left);
                    }
                    break;
            }
            __syncwarp();
        }
        if (flags & 1u) {  // non-systematic: u_hat = x_hat G_N in place (as beta_transform)
            const uint32_t in_word[5] = {0x55555555u, 0x33333333u, 0x0F0F0F0Fu, 0x00FF00FFu, 0x0000FFFFu};
            for (int b = 0; b < 5 && (1 << b) < N; ++b) {
                for (int k = l; k < NB; k += 32) beta[k] ^= (beta[k] >> (1 << b)) & in_word[b];
                __syncwarp();
            }
            for (int D = 1; D < NB; D <<= 1) {
                for (int k = l; k < NB; k += 32)
                    if (!(k & D)) beta[k] ^= beta[k | D];
                __syncwarp();
            }
        }
        // information bits x_hat[A] (or u_hat[A]) (as gather_info, runtime sizes)
        for (int q = l; q < NWK; q += 32) stg[q] = 0;
        __syncwarp();
        for (int k = l; k < NB; k += 32) {
            const uint32_t m = __ldg(gtab + k);
            if (!m) continue;
            const uint32_t p = __ldg(gtab + NB + k);
            const uint32_t r = pext32(beta[k], m);
            const uint32_t sh = p & 31;
            atomicOr(stg + (p >> 5), r << sh);
            if (sh && sh + __popc(m) > 32) atomicOr(stg + (p >> 5) + 1, r >> (32 - sh));
        }
        __syncwarp();
        for (int q = l; q < NWK; q += 32) out[f * NWK + q] = stg[q];
        __syncwarp();
    }
}

// ------------------------------------------------------------------ long codes (N > 32768)
// The paper's answer for codes too long to unroll (N up to 2^24, "the instruction-based decoders
// are very suitable"): the same program interpreter with one CTA of T threads per frame
// (every op a CTA-wide loop ended by a barrier), stages of size <= GB_SMEM_MAX in shared
// memory, larger ones in a per-CTA global slot (L2-resident at the top of the tree), the
// decision bits in shared memory (N/8 bytes), the output by the piece table (gather_info).
// Same f/g/leaf arithmetic and op order as every other decoder.
constexpr int GB_SMEM_MAX = 8192;  // largest stage (elements) kept in shared memory
constexpr int GB_T = 512;

template <class P>
__host__ __device__ inline int generic_big_smem(int N) {
    const int small = 2 * (N < 2 * GB_SMEM_MAX ? N / 2 : GB_SMEM_MAX);  // stages of size <= GB_SMEM_MAX
    return g_align16(small * (int)sizeof(typename P::st_t)) + 4 * (N / 32) + 64 * 8 + 64;
}
template <class P>
__host__ __device__ inline long long generic_big_gslot(int N) {  // global stage elements per CTA
    return N > 2 * GB_SMEM_MAX ? (long long)N - 2 * GB_SMEM_MAX : 0;
}

template <class P>
__global__ void __launch_bounds__(GB_T) k_generic_big(const void* __restrict__ llr_, long long n_frames,
                                                      uint32_t* __restrict__ out, const uint32_t* __restrict__ gtab,
                                                      const uint32_t* __restrict__ prog, int n_ops, int N, int K,
                                                      unsigned flags, void* __restrict__ gslot_all) {
    using S = typename P::st_t;
    using V = typename P::v_t;
    extern __shared__ __align__(16) unsigned char gsmem[];
    const int small = 2 * (N < 2 * GB_SMEM_MAX ? N / 2 : GB_SMEM_MAX);
    S* const sst = (S*)gsmem;
    uint32_t* const beta = (uint32_t*)(gsmem + g_align16(small * (int)sizeof(S)));
    const int NB = N / 32;
    const int NWK = (K + 31) / 32;
    unsigned long long* const red = (unsigned long long*)(beta + NB);  // per-warp reduction slots
    uint32_t* const redp = (uint32_t*)(red + 32);
    S* const gst = (S*)gslot_all + (long long)blockIdx.x * generic_big_gslot<P>(N);
    using Ch = typename P::in_t;  // the channel (signed int8 or f32); stages are S (int8: biased bytes)
    const Ch* llr = (const Ch*)llr_;
    const int tid = threadIdx.x, l = lane_id(), wid = tid >> 5;
    // alpha of a node of size m (m < N): stage(m) at 2*GB - 2m in shared memory, else N - 2m globally
    auto stage = [&](int m) -> S* { return m <= GB_SMEM_MAX ? sst + (small - 2 * m) : gst + ((long long)N - 2LL * m); };
    for (long long f = blockIdx.x; f < n_frames; f += gridDim.x) {
        const Ch* chan = llr + f * (long long)N;
        for (int k = tid; k < NB; k += GB_T) beta[k] = 0;
        __syncthreads();
        for (int pc = 0; pc < n_ops; ++pc) {
            const uint32_t w = __ldg(prog + pc);
            const int op = w & 15, n = 1 << ((w >> 4) & 31), off = (int)(w >> 9), h = n >> 1;
            const bool root = n == N;  // the root op reads the channel (uniform per op)
            const S* srcs = root ? gst : stage(n);
            auto src_ld = [&](int i) -> V { return root ? P::ld(chan[i]) : P::ld(srcs[i]); };
            S* dst = stage(h);
            switch (op) {
                case OP_F:
                    for (int i = tid; i < h; i += GB_T) dst[i] = P::st(P::f(src_ld(i), src_ld(i + h)));
                    break;
                case OP_G:
                    for (int i = tid; i < h; i += GB_T)
                        dst[i] = P::st(P::g(src_ld(i), src_ld(i + h), (beta[(off + i) >> 5] >> ((off + i) & 31)) & 1u));
                    break;
                case OP_G0R:
                    for (int i = tid; i < h; i += GB_T) dst[i] = P::st(P::g0(src_ld(i), src_ld(i + h)));
                    break;
                case OP_R1:
                    for (int i0 = 32 * wid; i0 < n; i0 += GB_T) {
                        const uint32_t b = __ballot_sync(FULL, i0 + l < n && P::hd(src_ld(i0 + l)));
                        if (l == 0) {
                            if (n >= 32) beta[(off + i0) >> 5] = b;
                            else put_bits(beta, off, n, b);
                        }
                    }
                    break;
                case OP_REP: {  // P:431-440; int8 exact sum (C12), f32 pairwise halving (C13)
                    bool neg;
                    if constexpr (P::kExactSum) {
                        typename P::acc_t t = 0;
                        for (int i = tid; i < n; i += GB_T) t = P::add(t, P::acc(src_ld(i)));
#pragma unroll
                        for (int o = 16; o; o >>= 1) t = P::add(t, __shfl_xor_sync(FULL, t, o));
                        if (l == 0) red[wid] = __float_as_uint(t);
                        __syncthreads();
                        typename P::acc_t u = l < GB_T / 32 ? __uint_as_float((uint32_t)red[l]) : 0.0f;
#pragma unroll
                        for (int o = 16; o; o >>= 1) u = P::add(u, __shfl_xor_sync(FULL, u, o));
                        neg = P::acc_neg(u);
                    } else {
                        V t;
                        if (n <= 32) {
                            t = src_ld(l & (n - 1));
                            for (int o = h; o >= 1; o >>= 1) t = P::add(t, __shfl_xor_sync(FULL, t, o));
                        } else {
                            for (int i = tid; i < h; i += GB_T) dst[i] = P::add(src_ld(i), src_ld(i + h));
                            __syncthreads();
                            for (int m = h; m > 32; m >>= 1) {
                                for (int i = tid; i < m / 2; i += GB_T) dst[i] = P::add(dst[i], dst[i + m / 2]);
                                __syncthreads();
                            }
                            t = dst[l];
                            for (int o = 16; o >= 1; o >>= 1) t = P::add(t, __shfl_xor_sync(FULL, t, o));
                        }
                        neg = P::acc_neg(t);
                    }
                    if (n >= 32) {
                        for (int k = tid; k < n / 32; k += GB_T) beta[(off >> 5) + k] = neg ? FULL : 0u;
                    } else if (tid == 0) {
                        put_bits(beta, off, n, neg ? FULL : 0u);
                    }
                    break;
                }
                case OP_SPC: {  // P:442-459, readings C10/C11; 64-bit keys (index up to 2^20)
                    uint32_t par = 0;
                    unsigned long long best = ~0ull;
                    for (int i0 = 32 * wid; i0 < n; i0 += GB_T) {
                        const int i = i0 + l;
                        const bool in = i < n;
                        const V x = in ? src_ld(i) : V(0);
                        const uint32_t b = __ballot_sync(FULL, in && P::hd(x));
                        par ^= __popc(b) & 1u;
                        if (l == 0) {
                            if (n >= 32) beta[(off + i0) >> 5] = b;
                            else put_bits(beta, off, n, b);
                        }
                        const unsigned long long k = in ? ((unsigned long long)P::mag_key(x) << 32) | (uint32_t)i : ~0ull;
                        best = k < best ? k : best;
                    }
#pragma unroll
                    for (int o = 16; o; o >>= 1) {
                        const unsigned long long other = __shfl_xor_sync(FULL, best, o);
                        best = other < best ? other : best;
                    }
                    if (l == 0) {
                        red[wid] = best;
                        redp[wid] = par;
                    }
                    __syncthreads();
                    if (wid == 0) {
                        unsigned long long b2 = l < GB_T / 32 ? red[l] : ~0ull;
#pragma unroll
                        for (int o = 16; o; o >>= 1) {
                            const unsigned long long other = __shfl_xor_sync(FULL, b2, o);
                            b2 = other < b2 ? other : b2;
                        }
                        const uint32_t p2 = __popc(__ballot_sync(FULL, l < GB_T / 32 && (redp[l] & 1u))) & 1u;
                        if (l == 0 && p2) {
                            const uint32_t idx = (uint32_t)b2;
                            beta[(off + idx) >> 5] ^= 1u << ((off + idx) & 31);
                        }
                    }
                    break;
                }
                case OP_COMB:
                case OP_COMB0R:
                    if (n >= 64) {
                        for (int k = tid; k < n / 64; k += GB_T) {
                            const uint32_t r = beta[(off >> 5) + n / 64 + k];
                            beta[(off >> 5) + k] = op == OP_COMB ? beta[(off >> 5) + k] ^ r : r;
                        }
                    } else if (tid == 0) {
                        const uint32_t wv = beta[off >> 5];
                        const uint32_t r = (wv >> ((off & 31) + h)) & low_mask(h);
                        const uint32_t left = op == OP_COMB ? ((wv >> (off & 31)) & low_mask(h)) ^ r : r;
                        put_bits(beta, off, h, left);
                    }
                    break;
            }
            __syncthreads();
        }
        if (flags & 1u) {  // non-systematic output: u_hat = x_hat G_N (beta_transform, runtime N)
            const uint32_t in_word[5] = {0x55555555u, 0x33333333u, 0x0F0F0F0Fu, 0x00FF00FFu, 0x0000FFFFu};
            for (int b = 0; b < 5; ++b) {
                for (int k = tid; k < NB; k += GB_T) beta[k] ^= (beta[k] >> (1 << b)) & in_word[b];
                __syncthreads();
            }
            for (int D = 1; D < NB; D <<= 1) {
                for (int k = tid; k < NB; k += GB_T)
                    if (!(k & D)) beta[k] ^= beta[k | D];
                __syncthreads();
            }
        }
        // information bits by the piece table (as gather_info, runtime sizes)
        const int TB = (2 * NB + 3) & ~3;
        const int NG = (NWK + 31) / 32;
        const uint32_t* hdr = gtab + TB;
        const uint2* pcs = reinterpret_cast<const uint2*>(gtab + TB + ((NG + 1 + 3) & ~3));
        for (int q = tid; q < NWK; q += GB_T) {
            uint32_t acc = 0;
            const int g = q >> 5, r1 = (int)__ldg(hdr + g + 1);
            for (int r = (int)__ldg(hdr + g); r < r1; ++r) acc |= gather_piece(beta, __ldg(pcs + r * 32 + (q & 31)));
            out[f * NWK + q] = acc;
        }
        __syncthreads();
    }
}

}  // namespace pd

// Entry points for polar_api.cu (kernel addresses and shared-memory sizes).
const void* polar_generic_big_kernel(bool i8) {
    return i8 ? (const void*)&pd::k_generic_big<pd::PI8> : (const void*)&pd::k_generic_big<pd::PF32>;
}
int polar_generic_big_smem(bool i8, int N) {
    return i8 ? pd::generic_big_smem<pd::PI8>(N) : pd::generic_big_smem<pd::PF32>(N);
}
long long polar_generic_big_gslot_bytes(bool i8, int N) {
    return i8 ? pd::generic_big_gslot<pd::PI8>(N) : 4 * pd::generic_big_gslot<pd::PF32>(N);
}
int polar_generic_big_threads() { return pd::GB_T; }
const void* polar_generic_kernel(bool i8) {
    return i8 ? (const void*)&pd::k_generic<pd::PI8> : (const void*)&pd::k_generic<pd::PF32>;
}
int polar_generic_smem(bool i8, int N, int K) {
    return i8 ? pd::generic_smem<pd::PI8>(N, K) : pd::generic_smem<pd::PF32>(N, K);
}
