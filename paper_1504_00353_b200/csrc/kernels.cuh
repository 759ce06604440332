// kernels.cuh -- the two decode kernel shapes every specialised code is instantiated into.
//
//  k_warp (N <= 2048, the throughput codes): one warp decodes one frame at a time; a CTA
//    holds WARPS independent warps; the grid is persistent (frames are strided over all
//    warps of the grid).  Each warp double-buffers its frames' channel LLRs in shared
//    memory with TMA bulk copies (cp.async.bulk + mbarrier), so the ingest of frame i+1
//    overlaps the decode of frame i (the paper counts the copy in the latency).
//  * k_cta (N > 2048): one CTA decodes one frame: nodes larger than the warp subtree size
//    W run CTA-wide on shared-memory stages, subtrees of size W run on warp 0 in
//    registers.  int8 channel LLRs are brought in by one TMA bulk copy; the f32 channel
//    (128 KB at N = 32768) stays in global memory and is read by the two root ops only.
//
// Both kernels end with the systematic information-bit gather (gather_info).
#pragma once

#include "decoder.cuh"

namespace pd {

__host__ __device__ constexpr int align16(int x) { return (x + 15) & ~15; }

template <class P, class C>
struct WarpLayout {
    using in_t = typename P::in_t;
    static constexpr int FRAME_BYTES = C::N * (int)sizeof(in_t);
    static constexpr bool kTma = FRAME_BYTES % 16 == 0;
    static constexpr int BUF = align16(FRAME_BYTES);
    static constexpr int BETA = align16((C::N >= 32 ? C::N / 32 : 1) * 4);
    static constexpr int PER_WARP = 2 * BUF + BETA + 16;
    static constexpr int SMEM = C::WARPS * PER_WARP;
};

template <class P, class C>
__global__ void __launch_bounds__(C::WARPS * 32, C::MIN_BLOCKS)
    k_warp(const void* __restrict__ llr_, long long n_frames, uint32_t* __restrict__ out,
           const uint16_t* __restrict__ pos) {
    using L = WarpLayout<P, C>;
    using in_t = typename P::in_t;
    constexpr int N = C::N;
    constexpr int NWK = (C::K + 31) / 32;
    extern __shared__ __align__(128) unsigned char smem[];
    const int warp = threadIdx.x >> 5;
    const unsigned lane = lane_id();
    unsigned char* base = smem + warp * L::PER_WARP;
    in_t* const buf0 = (in_t*)base;
    in_t* const buf1 = (in_t*)(base + L::BUF);
    uint32_t* beta = (uint32_t*)(base + 2 * L::BUF);
    uint64_t* bar = (uint64_t*)(base + 2 * L::BUF + L::BETA);
    const in_t* llr = (const in_t*)llr_;

    long long f = (long long)blockIdx.x * C::WARPS + warp;
    const long long stride = (long long)gridDim.x * C::WARPS;
    if constexpr (L::kTma) {
        if (lane == 0) {
            mbar_init(bar, 1);
            mbar_init(bar + 1, 1);
            fence_barrier_init();
            if (f < n_frames) tma_load_1d(buf0, llr + f * N, L::FRAME_BYTES, bar);
        }
        __syncwarp();
    }
    for (int it = 0; f < n_frames; f += stride, ++it) {
        in_t* cur = (it & 1) ? buf1 : buf0;
        if constexpr (L::kTma) {
            const long long nf = f + stride;
            if (lane == 0 && nf < n_frames) {
                fence_proxy_async();
                tma_load_1d((it & 1) ? buf0 : buf1, llr + nf * N, L::FRAME_BYTES, bar + ((it + 1) & 1));
            }
            mbar_wait(bar + (it & 1), (it >> 1) & 1);
        } else {
            for (int i = lane; i < N; i += 32) cur[i] = llr[f * N + i];
            __syncwarp();
        }
        C::template decode_warp<P>(cur, beta);
        __syncwarp();
        gather_info<C::K>(beta, pos, out + f * NWK, 0, 1);
        __syncwarp();
    }
}

template <class P, class C>
struct CtaLayout {
    using in_t = typename P::in_t;
    using st_t = typename P::st_t;
    static constexpr int FRAME_BYTES = C::N * (int)sizeof(in_t);
    static constexpr int CHAN = P::kChanInSmem ? align16(FRAME_BYTES) : 0;
    static constexpr int STAGES = align16(C::STAGE_ELEMS * (int)sizeof(st_t));
    static constexpr int BETA = align16(C::N / 32 * 4);
    static constexpr int SMEM = CHAN + STAGES + BETA + 16;
};

template <class P, class C>
__global__ void __launch_bounds__(C::T, 1)
    k_cta(const void* __restrict__ llr_, long long n_frames, uint32_t* __restrict__ out,
          const uint16_t* __restrict__ pos) {
    using L = CtaLayout<P, C>;
    using in_t = typename P::in_t;
    using st_t = typename P::st_t;
    constexpr int N = C::N;
    constexpr int NWK = (C::K + 31) / 32;
    extern __shared__ __align__(128) unsigned char smem[];
    in_t* chanbuf = (in_t*)smem;
    st_t* stages = (st_t*)(smem + L::CHAN);
    uint32_t* beta = (uint32_t*)(smem + L::CHAN + L::STAGES);
    uint64_t* bar = (uint64_t*)(smem + L::CHAN + L::STAGES + L::BETA);
    const in_t* llr = (const in_t*)llr_;
    if constexpr (P::kChanInSmem) {
        if (threadIdx.x == 0) {
            mbar_init(bar, 1);
            fence_barrier_init();
        }
        __syncthreads();
    }
    int it = 0;
    for (long long f = blockIdx.x; f < n_frames; f += gridDim.x, ++it) {
        if constexpr (P::kChanInSmem) {
            if (threadIdx.x == 0) {
                fence_proxy_async();
                tma_load_1d(chanbuf, llr + f * N, L::FRAME_BYTES, bar);
            }
        }
        for (int k = threadIdx.x; k < N / 32; k += C::T) beta[k] = 0;
        __syncthreads();
        if constexpr (P::kChanInSmem) {
            mbar_wait(bar, it & 1);
            C::template decode_cta<P>((const in_t*)chanbuf, stages, beta);
        } else {
            C::template decode_cta<P>(llr + f * N, stages, beta);
        }
        __syncthreads();
        gather_info<C::K>(beta, pos, out + f * NWK, threadIdx.x >> 5, C::T / 32);
        __syncthreads();
    }
}

}  // namespace pd
