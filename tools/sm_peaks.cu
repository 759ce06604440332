// sm_peaks.cu -- microbenchmark of the sm_100a pipes the Fast-SSC kernels issue on (the ALU and
// shared-memory ceilings of the roofline; VERDICT r1 "make the roofline real").
//
// For each instruction: a full-occupancy grid (8 x #SMs CTAs of 256 threads) runs a loop of 8
// independent dependency chains per thread (enough ILP to saturate the pipe, not its
// latency); inline PTX pins the instruction; the chains feed one store guarded by a runtime
// value so nothing is dead.  Result: warp instructions per clock per SM, at the SM clock
// measured by clock64() against %globaltimer inside the same kernel (no clock assumption).
// Shared memory: ld.shared.v4 bandwidth in bytes per clock per SM.
//
// Build/run (on the GPU box): nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sm_peaks
//   tools/sm_peaks.cu && ./sm_peaks > profiles/peaks_sm.json
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x)                                                                           \
    do {                                                                                \
        cudaError_t e = (x);                                                            \
        if (e != cudaSuccess) {                                                         \
            fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e));                     \
            return 1;                                                                   \
        }                                                                               \
    } while (0)

constexpr int ITERS = 4096;
constexpr int CH = 8;  // independent chains per thread

__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// one op of each kind: x = op(x, y) with y loop-invariant
template <int K>
__device__ __forceinline__ uint32_t op(uint32_t x, uint32_t y) {
    uint32_t d;
    if constexpr (K == 0) asm volatile("lop3.b32 %0, %1, %2, %1, 0x96;" : "=r"(d) : "r"(x), "r"(y));
    else if constexpr (K == 1) asm volatile("prmt.b32 %0, %1, %2, 0x5140;" : "=r"(d) : "r"(x), "r"(y));
    else if constexpr (K == 2) asm volatile("add.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(y));
    else if constexpr (K == 3) asm volatile("min.xorsign.abs.f16x2 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(y));
    else if constexpr (K == 4) asm volatile("min.xorsign.abs.f32 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(y));
    else if constexpr (K == 5) asm volatile("add.rn.f32 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(y));
    else if constexpr (K == 6) asm volatile("mad.lo.u32 %0, %1, %2, %1;" : "=r"(d) : "r"(x), "r"(y));
    else if constexpr (K == 7) asm volatile("shfl.sync.bfly.b32 %0, %1, 1, 0x1f, -1;" : "=r"(d) : "r"(x));
    else if constexpr (K == 8) asm volatile("{.reg .pred p; setp.ne.u32 p, %1, %2; vote.sync.ballot.b32 %0, p, -1;}" : "=r"(d) : "r"(x), "r"(y));
    else if constexpr (K == 9) asm volatile("redux.sync.min.u32 %0, %1, -1;" : "=r"(d) : "r"(x));
    else if constexpr (K == 10) asm volatile("add.u32 %0, %1, %2;" : "=r"(d) : "r"(x), "r"(y));
    else if constexpr (K == 11) asm volatile("shf.l.wrap.b32 %0, %1, %2, 7;" : "=r"(d) : "r"(x), "r"(y));
    else asm volatile("fma.rn.f16x2 %0, %1, %2, %1;" : "=r"(d) : "r"(x), "r"(y));
    return d ^ (K == 7 || K == 8 || K == 9 ? y : 0u);  // keep the cross-lane ops dependent on y too
}

template <int K>
__global__ void k_pipe(uint32_t seed, uint32_t* out, unsigned long long* clk) {
    uint32_t x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = seed * (threadIdx.x + 3 * c + 1);
    const uint32_t y = seed ^ 0x3c003c00u;
    __syncthreads();
    const uint64_t c0 = clock64(), t0 = gtimer();
#pragma unroll 1
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = op<K>(x[c], y);
    const uint64_t c1 = clock64(), t1 = gtimer();
    uint32_t r = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) r ^= x[c];
    if (r == seed) out[blockIdx.x * blockDim.x + threadIdx.x] = r;  // never true in practice
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        clk[0] = c1 - c0;
        clk[1] = t1 - t0;
    }
}

// shared-memory load bandwidth: 16-byte loads, conflict-free (consecutive lanes, consecutive 16 B)
__global__ void k_lds(uint32_t seed, uint32_t* out, unsigned long long* clk) {
    __shared__ __align__(16) uint32_t buf[9 * 1024];
    for (int i = threadIdx.x; i < 9 * 1024; i += blockDim.x) buf[i] = seed + i;
    __syncthreads();
    uint32_t acc = 0;
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(buf) + 16 * (threadIdx.x % 256);
    const uint64_t c0 = clock64(), t0 = gtimer();
#pragma unroll 1
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            uint32_t a, b, d, e;
            // the address moves with i (one 512-byte row per step), so the loads stay in the loop
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(d), "=r"(e)
                         : "r"(base + 4096 * c + 512 * (i & 3)) : "memory");
            acc += a ^ b ^ d ^ e;
        }
    }
    const uint64_t c1 = clock64(), t1 = gtimer();
    if (acc == seed) out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        clk[0] = c1 - c0;
        clk[1] = t1 - t0;
    }
}

// dependent-chain latency: one warp, one chain, ITERS ops; cycles per op by clock64
template <int K>
__global__ void k_lat(uint32_t seed, uint32_t* out, unsigned long long* clk) {
    uint32_t x = seed * (threadIdx.x + 1);
    const uint32_t y = seed ^ 0x3c003c00u;
    __shared__ uint32_t sm[64];
    sm[threadIdx.x] = threadIdx.x;
    __syncwarp();
    const uint64_t c0 = clock64();
#pragma unroll 1
    for (int i = 0; i < ITERS / 16; ++i)
#pragma unroll
    for (int u = 0; u < 16; ++u) {  // 16 dependent ops per trip: the loop overhead is amortised
        if constexpr (K == 100) x = (uint32_t)__shfl_xor_sync(0xffffffffu, (int)x, 1) + 1u;  // SHFL + IADD
        else if constexpr (K == 101) x = __ballot_sync(0xffffffffu, (x & (1u << (threadIdx.x & 31))) != 0) + 1u;
        else if constexpr (K == 102) x = __reduce_min_sync(0xffffffffu, x) + threadIdx.x;
        else if constexpr (K == 103) x = __float_as_uint(__fadd_rn(__uint_as_float(x), 1.0f));
        else if constexpr (K == 104) x = sm[x & 31] + 1u;  // LDS (dependent address)
        else if constexpr (K == 105) { asm volatile("bar.sync 1, 512;" ::: "memory"); x += 1u; }
        else x = op<K>(x, y);
    }
    const uint64_t c1 = clock64();
    if (x == seed) out[threadIdx.x] = x;
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        clk[0] = c1 - c0;
        clk[1] = 0;
    }
}

template <int K>
static int lat(const char* name, uint32_t* out, unsigned long long* dclk, int threads, bool last) {
    k_lat<K><<<1, threads>>>(12345u, out, dclk);
    CK(cudaDeviceSynchronize());
    unsigned long long clk[2];
    CK(cudaMemcpy(clk, dclk, sizeof clk, cudaMemcpyDeviceToHost));
    printf("    \"%s\": %.1f%s\n", name, (double)clk[0] / ITERS, last ? "" : ",");
    return 0;
}

template <class Kern>
static int run(const char* name, Kern kern, int nsm, uint32_t* out, unsigned long long* dclk, double per_thread_ops,
               const char* unit, bool last) {
    const int blocks = nsm * 8, threads = 256;
    kern<<<blocks, threads>>>(12345u, out, dclk);  // warm-up
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<<<blocks, threads>>>(12345u, out, dclk);
    cudaEventRecord(b);
    CK(cudaDeviceSynchronize());
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    unsigned long long clk[2];
    CK(cudaMemcpy(clk, dclk, sizeof clk, cudaMemcpyDeviceToHost));
    const double mhz = clk[1] ? 1e3 * (double)clk[0] / (double)clk[1] : 0.0;  // cycles per us
    const double total = per_thread_ops * blocks * threads;                   // lane ops (or bytes)
    const double per_clk_sm = total / (ms * 1e-3) / (mhz * 1e6) / nsm;
    const bool bytes = unit[0] == 'B';
    printf("    \"%s\": {\"per_clk_per_sm\": %.3f, \"unit\": \"%s\", \"warp_inst_per_clk_per_sm\": %.3f, \"sm_mhz\": %.0f, "
           "\"ms\": %.4f}%s\n",
           name, per_clk_sm, unit, bytes ? per_clk_sm / 512.0 : per_clk_sm / 32.0, mhz, ms, last ? "" : ",");
    return 0;
}

int main() {
    int dev = 0, nsm = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, dev));
    uint32_t* out;
    unsigned long long* clk;
    CK(cudaMalloc(&out, (size_t)nsm * 8 * 256 * 4));
    CK(cudaMalloc(&clk, 16));
    const double ops = (double)ITERS * CH;
    printf("{\n  \"device\": \"%s\", \"sms\": %d,\n  \"method\": \"tools/sm_peaks.cu: 8 x SMs CTAs x 256 threads, 8 independent "
           "chains per thread, %d iterations; rate = lane ops / (CUDA-event time x clock64/globaltimer SM clock x SMs)\",\n"
           "  \"pipes\": {\n", p.name, nsm, ITERS);
    run("LOP3", k_pipe<0>, nsm, out, clk, ops, "lane-ops", false);
    run("PRMT", k_pipe<1>, nsm, out, clk, ops, "lane-ops", false);
    run("HADD2", k_pipe<2>, nsm, out, clk, ops, "lane-ops", false);
    run("HMNMX2", k_pipe<3>, nsm, out, clk, ops, "lane-ops", false);
    run("FMNMX", k_pipe<4>, nsm, out, clk, ops, "lane-ops", false);
    run("FADD", k_pipe<5>, nsm, out, clk, ops, "lane-ops", false);
    run("IMAD", k_pipe<6>, nsm, out, clk, ops, "lane-ops", false);
    run("SHFL", k_pipe<7>, nsm, out, clk, ops, "lane-ops", false);
    run("VOTE", k_pipe<8>, nsm, out, clk, ops, "lane-ops", false);
    run("REDUX", k_pipe<9>, nsm, out, clk, ops, "lane-ops", false);
    run("IADD", k_pipe<10>, nsm, out, clk, ops, "lane-ops", false);
    run("SHF", k_pipe<11>, nsm, out, clk, ops, "lane-ops", false);
    run("HFMA2", k_pipe<12>, nsm, out, clk, ops, "lane-ops", false);
    run("LDS128", k_lds, nsm, out, clk, ops * 16.0, "B", true);
    printf("  },\n  \"latency_cycles_per_dependent_op\": {\n");
    lat<100>("SHFL+IADD", out, clk, 32, false);
    lat<101>("VOTE.ballot+IADD", out, clk, 32, false);
    lat<102>("REDUX.min+IADD", out, clk, 32, false);
    lat<103>("FADD", out, clk, 32, false);
    lat<4>("FMNMX", out, clk, 32, false);
    lat<0>("LOP3", out, clk, 32, false);
    lat<104>("LDS+IADD", out, clk, 32, false);
    lat<105>("bar.sync 512 threads+IADD", out, clk, 512, true);
    printf("  }\n}\n");
    return 0;
}
