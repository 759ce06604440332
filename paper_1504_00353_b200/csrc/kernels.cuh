// kernels.cuh -- the decode kernel every specialised code is instantiated into.
//
// k_frame<P, C, T, CHAN_SMEM>: a group of T threads (one CTA) decodes one frame at a time;
// the grid is persistent (frames strided over CTAs).  Two instantiations per code:
//
//  * throughput (T = 32): one warp per frame, many frames resident per SM.  Nodes larger
//    than the warp-subtree size W run warp-wide on shared-memory stages, subtrees of size W
//    in registers.  Channel LLRs: double-buffered TMA bulk copies into shared memory when
//    two frames fit in 16 KB (N <= 2048), else read from global memory by the root ops,
//    with the next frame prefetched into L2 (cp.async.bulk.prefetch.L2).
//  * latency (T = C::T_LAT, e.g. 512 for N = 32768): one CTA per frame; CTA-wide ops on
//    shared-memory stages, warp 0 runs the register subtrees; int8 channel by one TMA bulk
//    copy (the f32 channel, 128 KB at N = 32768, stays in global memory).
//
// The paper counts the frame copy into decoder memory in its latency.  Every frame
// ends with the systematic information-bit gather (gather_info).
#pragma once

#include "decoder.cuh"

namespace pd {

__host__ __device__ constexpr int align16(int x) { return (x + 15) & ~15; }

#ifndef POLAR_DYN
#define POLAR_DYN 1  // dynamic frame-group scheduling of the throughput variant with global stages
#endif
// bytes at the start of a throughput variant's global scratch (frame-group counter)
constexpr int SCRATCH_HDR = 256;

PD_INLINE void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Op-boundary barrier of a frame group.  Latency variant: the whole CTA.  Throughput variant:
// all active warps of the CTA (named barrier 1), so that the FPC warps, each decoding its
// own frame through the same unrolled code, stay in lockstep and share instruction fetch.
// It also carries the L2 prefetch of the group's next frame, issued right after the root G
// (the last read of the current frame's channel LLRs), so that each frame slot holds one
// channel in L2 at a time.
template <int T>
struct OpSync {
    uint32_t threads;
    const void* next;     // next frame's channel LLRs (nullptr: none / not prefetched)
    uint32_t next_bytes;
    PD_INLINE void operator()() const {
        if constexpr (T > 32) asm volatile("bar.sync 1, %0;" ::"n"(T) : "memory");
        else asm volatile("bar.sync 1, %0;" ::"r"(threads) : "memory");
    }
    // the frame group's barrier regardless of lockstep (the shared frame hand-out)
    PD_INLINE void group() const {
        if constexpr (T > 32) asm volatile("bar.sync 1, %0;" ::"n"(T) : "memory");
        else asm volatile("bar.sync 1, %0;" ::"r"(threads) : "memory");
    }
    // after a warp subtree call: the full op barrier -- without it the throughput warps drift
    // apart and stop sharing instruction fetch (measured: no lockstep at all 433 -> 320 Gbps,
    // lockstep everywhere but here 433 -> 435, profiles/r1_history.md)
    PD_INLINE void sub() const { (*this)(); }
    // after a Combine (a few word XORs on the group's own decision bits): in the throughput
    // variant only the warp's own lanes need to see them, so the frame group is not held in
    // lockstep there (+0.3%, same-box A/B)
    PD_INLINE void comb() const {
        if constexpr (T == 32) __syncwarp();
        else (*this)();
    }
    PD_INLINE void root_g_done() const {
        if (next && (threadIdx.x & (T - 1)) == 0) prefetch_l2(next, next_bytes);
    }
    // Instruction run-ahead (latency variant, Code::HELPER): warp 0 signals (barrier 2, 64
    // threads) just before the stage op that feeds its next register subtree; the helper warp
    // waits on it and then runs that subtree's (shared, non-inlined) code on dummy data about
    // one stage op ahead of warp 0, so warp 0 finds the instructions in the SM's caches.
    PD_INLINE void helper_arrive() const {
        if constexpr (T > 32) asm volatile("bar.arrive 2, 64;" ::: "memory");
    }
    PD_INLINE void helper_wait() const {
        if constexpr (T > 32) asm volatile("bar.sync 2, 64;" ::: "memory");
    }
};

template <class P, class C, int T, int FPC, bool CHAN_SMEM, bool GTOP, bool H16>
struct FrameLayout {
    using in_t = typename P::in_t;
    using st_t = typename P::st_t;
    static constexpr int FRAME_BYTES = C::N * (int)sizeof(in_t);
    static constexpr bool kBulk = FRAME_BYTES % 16 == 0;  // cp.async.bulk size rule
    // throughput warps double-buffer (prefetch the next frame), the latency CTA single-buffers
    static constexpr int NBUF = CHAN_SMEM ? (T == 32 ? 2 : 1) : 0;
    static constexpr int BUF = align16(FRAME_BYTES);
    // WF32 (latency variant): the stage of size W, read element by element by the register
    // subtrees, is kept as f32 in its own array
    static constexpr bool WF32 = T > 32;
    // H16: the int8 throughput variant's stages of size <= the code's H16 option are f16
    static constexpr int WST_OFF =
        align16(H16 ? C::STAGE_BYTES_SMEM_H : (GTOP ? C::STAGE_ELEMS_SMEM : C::STAGE_ELEMS) * (int)sizeof(st_t));
    static constexpr int STAGES = WST_OFF + (WF32 ? align16(C::WST * (int)sizeof(typename P::v_t)) : 0);
    // helper warp (latency variant, Code::HELPER): dummy subtree input and decision bits
    static constexpr bool HELP = WF32 && C::HELPER > 0;
    static constexpr int HSRC = HELP ? align16(C::WST * 4) : 0;
    static constexpr int HBETA = HELP ? align16((C::N >= 32 ? C::N / 32 : 1) * 4) : 0;
    // GTOP && C::GBETA: the decision bits also live in the frame slot's global scratch
    static constexpr bool GB = GTOP && C::GBETA;
    static constexpr int BETA_BYTES = align16((C::N >= 32 ? C::N / 32 : 1) * 4);
    static constexpr int BETA = GB ? 0 : BETA_BYTES;
    static constexpr int GSTAGE_BYTES = align16(H16 ? C::GSTAGE_BYTES_H : C::GSTAGE_ELEMS * (int)sizeof(st_t));
    static constexpr int GSLOT = GSTAGE_BYTES + (GB ? BETA_BYTES : 0);  // global bytes per slot
    // output staging words: the stage area is free after the decode when it is large enough
    static constexpr int OUTW = align16((C::K + 31) / 32 * 4);
    static constexpr int STG = STAGES >= OUTW ? 0 : OUTW;
    static constexpr int PER_FRAME = NBUF * BUF + STAGES + BETA + STG + 16 + HSRC + HBETA;
    static constexpr int SMEM = FPC * PER_FRAME;
};

// FPC frame groups of T threads per CTA (FPC > 1 only with T = 32).
// GTOP: the largest stages (N/2 and N/4 by default) live in global scratch (L2-resident), one slot per frame
// group of the persistent grid, so that more frames fit in shared memory per SM.
template <class P, class C, int T, int FPC, bool CHAN_SMEM, bool GTOP, bool H16, int MINB = 1>
__global__ void __launch_bounds__(T * FPC + (T > 32 ? 32 * C::HELPER : 0), MINB)
    k_frame(const void* __restrict__ llr_, long long n_frames, uint32_t* __restrict__ out,
            const uint32_t* __restrict__ gtab, void* __restrict__ gscratch,
            unsigned flags  // bit 0: non-systematic output u_hat[A] (polar_code_set_output)
#ifdef POLAR_DEBUG_DUMP
            , float* __restrict__ dump  // [n_frames][dump_stride(N)] alpha stages (decoder.cuh)
#endif
    ) {
    static_assert(FPC == 1 || T == 32, "");
    using L = FrameLayout<P, C, T, FPC, CHAN_SMEM, GTOP, H16>;
    using in_t = typename P::in_t;
    using st_t = typename P::st_t;
    constexpr int N = C::N;
    constexpr int NWK = (C::K + 31) / 32;
    constexpr bool TMA = CHAN_SMEM && L::kBulk;
    constexpr bool DBL = L::NBUF > 1;
    extern __shared__ __align__(128) unsigned char smem_all[];
    const int grp = FPC > 1 ? (int)(threadIdx.x >> 5) : 0;
    unsigned char* const smem = smem_all + grp * L::PER_FRAME;
    in_t* const buf0 = (in_t*)smem;
    in_t* const buf1 = (in_t*)(smem + (DBL ? L::BUF : 0));
    st_t* const stages = (st_t*)(smem + L::NBUF * L::BUF);
    typename P::v_t* const wst = (typename P::v_t*)(smem + L::NBUF * L::BUF + L::WST_OFF);
    // DYN: frame groups after the first round are handed out by an atomic counter (the first
    // SCRATCH_HDR bytes of gscratch, zeroed by the host before each launch), so the frames in
    // flight stay a compact window of the input; with static striding the slots drift apart
    // over hundreds of rounds (1M frames at N = 32768: 261 vs 281 Gbps for 64 launches of 16K).
    constexpr bool DYN = POLAR_DYN && T == 32 && GTOP && !CHAN_SMEM;
    constexpr int HDR = (T == 32 && GTOP) ? SCRATCH_HDR : 0;
    unsigned long long* const gctr = (unsigned long long*)gscratch;
    __shared__ long long s_next;
    unsigned char* const gslot =
        GTOP ? (unsigned char*)gscratch + HDR + ((long long)blockIdx.x * FPC + grp) * L::GSLOT : nullptr;
    uint32_t* const beta = L::GB ? (uint32_t*)(gslot + L::GSTAGE_BYTES) : (uint32_t*)(smem + L::NBUF * L::BUF + L::STAGES);
    uint32_t* const stg = (uint32_t*)(L::STG ? smem + L::NBUF * L::BUF + L::STAGES + L::BETA : (unsigned char*)stages);
    uint64_t* const bar = (uint64_t*)(smem + L::NBUF * L::BUF + L::STAGES + L::BETA + L::STG);
    float* const hsrc = (float*)(smem + L::NBUF * L::BUF + L::STAGES + L::BETA + L::STG + 16);
    uint32_t* const hbeta = (uint32_t*)((unsigned char*)hsrc + L::HSRC);
    const in_t* llr = (const in_t*)llr_;
    st_t* const gst = (st_t*)gslot;
    const unsigned tid = FPC > 1 ? (threadIdx.x & 31u) : threadIdx.x;  // thread index in its group
    const bool leader = tid == 0;

#ifdef POLAR_TRACE
    if (threadIdx.x == 0 && blockIdx.x == 0) g_ptrace = T > 32 ? (unsigned long long*)gscratch : nullptr;
    __syncthreads();
#endif
    if constexpr (L::HELP) {
        for (int i = threadIdx.x; i < C::WST; i += blockDim.x) hsrc[i] = 0.0f;
        __syncthreads();
        if (threadIdx.x >= T) {  // the helper warp: run-ahead only, never touches real data
            if (threadIdx.x < T + 32 * (C::HELPER - 1)) return;  // spacer warps put it on scheduler HELPER-1
            for (long long g = blockIdx.x; g < n_frames; g += gridDim.x) {
                const OpSync<T> hs{0, nullptr, 0};
                C::template helper<P>(hsrc, hbeta, hs);
            }
            return;
        }
    }
    // frames of round r: (r * gridDim.x + blockIdx.x) * FPC + grp
    const long long stride = (long long)gridDim.x * FPC;
    long long f = (long long)blockIdx.x * FPC + grp;
    if constexpr (TMA) {
        if (leader) {
            mbar_init(bar, 1);
            mbar_init(bar + 1, 1);
            fence_barrier_init();
            if (f < n_frames) tma_load_1d(buf0, llr + f * N, L::FRAME_BYTES, bar);
        }
        __syncwarp();
        if constexpr (T > 32) group_sync<T>();
    }
    for (int it = 0; f < n_frames; ++it) {
        // warps of this round that have a frame: they alone take part in the op barriers
        const long long base = f - grp;
        const long long nf = f + stride;
        // without shared-memory ingest the next frame is prefetched into L2 after the root G
        // Off by default: measured slower at N = 32768 (each frame slot would then hold a second
        // channel in L2 besides its live stage scratch; profiles/r1_sweep.md).
#ifdef POLAR_PREFETCH_NEXT
        const bool pf = !CHAN_SMEM && L::kBulk && C::STAGE_ELEMS > 0 && nf < n_frames;
#else
        const bool pf = false;
#endif
        const OpSync<T> sync{(uint32_t)(32 * (FPC > 1 ? (int)min((long long)FPC, n_frames - base) : 1)),
                             pf ? (const void*)(llr + nf * N) : nullptr, (uint32_t)L::FRAME_BYTES};
        const in_t* chan;
        if constexpr (TMA) {
            in_t* cur = (DBL && (it & 1)) ? buf1 : buf0;
            if (DBL && leader && nf < n_frames) {
                // buffer (it+1)&1 was last read in round it-1, which ended with a barrier
                fence_proxy_async();
                tma_load_1d((it & 1) ? buf0 : buf1, llr + nf * N, L::FRAME_BYTES, bar + ((it + 1) & 1));
            }
            mbar_wait(bar + (DBL ? (it & 1) : 0), DBL ? ((it >> 1) & 1) : (it & 1));
            chan = cur;
        } else if constexpr (CHAN_SMEM) {
            for (int i = tid; i < N; i += T) buf0[i] = llr[f * N + i];
            sync();
            chan = buf0;
        } else {
            if (C::STAGE_ELEMS == 0 && L::kBulk && leader && nf < n_frames) prefetch_l2(llr + nf * N, L::FRAME_BYTES);
            chan = llr + f * N;
        }
        if constexpr (C::STAGE_ELEMS > 0) {
            for (int k = tid; k < N / 32; k += T) beta[k] = 0;
            sync();
        }
#ifdef POLAR_DEBUG_DUMP
        if (leader) {
            const unsigned w = T == 32 ? (threadIdx.x >> 5) : 0u;
            s_dbase[w] = dump + f * (long long)dump_stride(N);
            s_dpos[w] = 0;
        }
        if constexpr (T == 32) __syncwarp(); else group_sync<T>();
#endif
        C::template decode<P, T, GTOP, L::WF32, CHAN_SMEM ? SP_SHARED : SP_GLOBAL, H16>(chan, stages, gst, wst, beta, sync);
        sync();
        if (flags & 1u) {  // uniform per launch
            if constexpr (T == 32) beta_transform<N, 32>(beta);
            else beta_transform<N, T>(beta);
        }
        gather_info<N, C::K, T>(beta, gtab, stg, out + f * NWK);
        sync();
        if constexpr (TMA && !DBL) {
            // single buffer: the next frame's copy starts once every thread is done with this one
            if (leader && nf < n_frames) {
                fence_proxy_async();
                tma_load_1d(buf0, llr + nf * N, L::FRAME_BYTES, bar);
            }
        }
        if constexpr (DYN) {
            if (threadIdx.x == 0) s_next = ((long long)gridDim.x + (long long)atomicAdd(gctr, 1ull)) * FPC;
            sync.group();
            f = s_next + grp;
            sync.group();  // every warp has read s_next before warp 0 may overwrite it
        } else {
            f += stride;
        }
    }
}

}  // namespace pd

namespace pd {

// ------------------------------------------------------------- batch-1 mailbox (NEXT N3)
// The paper's latency includes copying the frame to decoder memory and the estimate back
// (GPU: P:1005).  k_mailbox is a persistent one-CTA instance of the latency variant
// that waits for frames in host-mapped pinned memory: the host writes the N channel LLRs,
// then bumps ctl->req; thread 0 sees it (acquire load over PCIe), the CTA copies the frame
// into a device buffer, decodes it with the same unrolled code as k_frame, writes x_hat[A]
// straight into host-mapped memory and releases ctl->done = req.  No launch, no memcpy call
// and no stream synchronisation per frame.  req = ~0 stops it; so does `idle_ns` without a
// request (the kernel can never outlive a crashed host process by more than that).
struct MailboxCtl {
    unsigned int req;
    unsigned int pad0[31];
    unsigned int done;
    unsigned int pad1[31];
};

PD_INLINE unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <class P, class C, int T>
__global__ void __launch_bounds__(T, 1)
    k_mailbox(const int8_t* __restrict__ hframe, uint32_t* __restrict__ hout, MailboxCtl* ctl, int8_t* __restrict__ dbuf,
              const uint32_t* __restrict__ gtab, unsigned long long idle_ns, unsigned flags) {
    static_assert(T > 32 && C::N % 16 == 0 && C::N >= 64, "");
    // the frame goes straight from host-mapped memory into the shared-memory channel buffer
    // (as the TMA copy of k_frame's latency variant would put it); dbuf is unused
    using L = FrameLayout<P, C, T, 1, true, false, false>;
    constexpr int N = C::N;
    extern __shared__ __align__(128) unsigned char smem_all[];
    __shared__ unsigned int s_req;
    using st_t = typename P::st_t;
    int8_t* const chan = (int8_t*)smem_all;
    st_t* const stages = (st_t*)(smem_all + L::NBUF * L::BUF);
    typename P::v_t* const wst = (typename P::v_t*)(smem_all + L::NBUF * L::BUF + L::WST_OFF);
    uint32_t* const beta = (uint32_t*)(smem_all + L::NBUF * L::BUF + L::STAGES);
    uint32_t* const stg = (uint32_t*)(L::STG ? smem_all + L::NBUF * L::BUF + L::STAGES + L::BETA : (unsigned char*)stages);
    const OpSync<T> sync{(uint32_t)T, nullptr, 0};
    unsigned int seq = 0;
    (void)dbuf;
    for (;;) {
        if (threadIdx.x == 0) {
            const unsigned long long t0 = globaltimer_ns();
            unsigned int r;
            for (;;) {
                asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(r) : "l"(&ctl->req) : "memory");
                if (r != seq) break;
                if (globaltimer_ns() - t0 > idle_ns) {
                    r = 0xffffffffu;
                    break;
                }
            }
            s_req = r;
        }
        __syncthreads();
        const unsigned int r = s_req;
        if (r == 0xffffffffu) break;
        seq = r;
        constexpr int V = N / 16;  // 16-byte vectors of the frame; all loads of a thread first
        constexpr int PER = (V + T - 1) / T;
        int4 v[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k)
            if (threadIdx.x + k * T < V) v[k] = __ldcv((const int4*)hframe + threadIdx.x + k * T);
#pragma unroll
        for (int k = 0; k < PER; ++k)
            if (threadIdx.x + k * T < V) ((int4*)chan)[threadIdx.x + k * T] = v[k];
        if constexpr (C::STAGE_ELEMS > 0)
            for (int k = threadIdx.x; k < N / 32; k += T) beta[k] = 0;
        __syncthreads();
        C::template decode<P, T, false, L::WF32, SP_SHARED, false>((const int8_t*)chan, stages, (st_t*)nullptr, wst, beta, sync);
        sync();
        if (flags & 1u) beta_transform<N, T>(beta);
        gather_info<N, C::K, T>(beta, gtab, stg, hout);
        __threadfence_system();
        __syncthreads();
        if (threadIdx.x == 0) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(&ctl->done), "r"(seq) : "memory");
    }
}

}  // namespace pd
