/*
 * polar.h -- C ABI of the B200 Fast-SSC polar decoder (libpolar.so).
 *
 * The hot path is the Fast-SSC decoding of batches of systematic polar frames of
 * Giard, Sarkis, Leroux, Thibeault and Gross, "Low-Latency Software Polar Decoders"
 * (arXiv:1504.00353).  Citations "P:n" are line numbers of the paper's source text
 * (PAPER.md); "reading Cn" refers to the readings listed in DESIGN.md section 3.
 *
 * Conventions (all calls):
 *   - plain C types only; no exception crosses the ABI; every call returns a polar_status;
 *   - "device" pointers are CUDA device pointers (e.g. torch CUDA tensors), "host" pointers
 *     are ordinary host memory; the library never frees memory it did not allocate;
 *   - information bits are packed LSB-first into uint32 words, in ascending order of the
 *     information set A (reading C5); per-frame stride W = ceil(K/32) words;
 *   - channel LLRs are frame-major [n_frames][N], natural index order,
 *     positive LLR = bit 0 more likely (BPSK 0 -> +1, eq:info P:444-449);
 *   - decode calls are stream-ordered and asynchronous; they never allocate device
 *     memory and never synchronise the stream;
 *   - there is no CPU fallback: without a usable sm_100 device the decode calls return
 *     POLAR_ERR_CUDA.
 */
#ifndef POLAR_H
#define POLAR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum polar_status {
    POLAR_OK = 0,
    POLAR_ERR_INVALID_ARGUMENT = 1, /* bad size, null or misaligned pointer, bad mask   */
    POLAR_ERR_UNSUPPORTED_CODE = 2, /* operation not available for this code or build   */
    POLAR_ERR_CUDA = 3,             /* a CUDA runtime call or kernel launch failed      */
    POLAR_ERR_OUT_OF_MEMORY = 4
} polar_status;

/* Opaque, immutable code handle: (N, K, frozen set), its Fast-SSC tree and the
 * kernels specialised for it.  Thread-safe to share once created: decode calls on one handle
 * from several threads and streams are correct (kernel variants that use the handle's global
 * stage scratch are ordered by an event when consecutive launches come from different
 * streams; inside a CUDA graph capture that ordering is left to the caller).  The
 * exceptions are polar_code_set_variant and the mailbox calls, as documented there. */
typedef struct polar_code polar_code;

/* Opaque CUDA stream (cudaStream_t); NULL = the legacy default stream. */
typedef void* polar_stream;

/* Human-readable text for a status code (static storage). */
const char* polar_status_string(polar_status s);

/* Message of the last failing call on this thread ("" if none). */
const char* polar_last_error(void);

/* Create a code handle.
 *   N            code length, a power of two, 2 <= N <= 32768;
 *   K            number of information bits, 1 <= K <= N;
 *   frozen_mask  host, N bytes, 1 = frozen, natural indexing; exactly N-K
 *                entries must be 1.  The library copies it.
 *   out          receives the handle.
 * Frozen sets the library was specialised for at build time get the unrolled decoders
 * (P:637-656); any other frozen set gets the generic, program-interpreted decoder
 * (the paper's instruction-based decoder: same results, lower throughput; see
 * polar_code_is_specialised).  Host-side only, except one-time uploads of small tables;
 * without a CUDA device the handle is still created (query and schedule work) and the
 * device calls return POLAR_ERR_CUDA. */
polar_status polar_code_create(uint32_t N, uint32_t K, const uint8_t* frozen_mask,
                               polar_code** out);

/* Free a handle (NULL is a no-op). */
void polar_code_destroy(polar_code* h);

/* Query a handle.  Any output pointer may be NULL.
 *   n_ops       number of Fast-SSC operations of the unrolled schedule (Listing-1 count,
 *               P:644-656; SURVEY Appendix A definition);
 *   smem_bytes  dynamic shared memory per CTA of the throughput kernel;
 *   warp_root   size W of the subtrees decoded by one warp in registers. */
polar_status polar_code_query(const polar_code* h, uint32_t* N, uint32_t* K, uint32_t* n_ops,
                              uint32_t* smem_bytes, uint32_t* warp_root);

/* The unrolled op list of the handle's decoder in Listing 1's vocabulary,
 * ';'-separated ("F<8>;G_0R<4>;Info<2>;...").  Writes at most cap bytes including the
 * terminating NUL into buf (may be NULL); *needed (may be NULL) receives the full size. */
polar_status polar_code_schedule(const polar_code* h, char* buf, uint32_t cap, uint32_t* needed);

/* *specialised = 1 if the handle uses a decoder unrolled for its code at build time, 2 if
 * polar_code_create specialised one at run time (below), 0 if it uses the generic
 * program-interpreted decoder (then polar_last_error() says why the run-time specialisation
 * did not happen). */
polar_status polar_code_is_specialised(const polar_code* h, int* specialised);

/* Run-time specialisation (the paper generates an unrolled decoder per code):
 * polar_code_create gives a frozen set without a build-time decoder its own, generated by the
 * library's code generator and compiled with NVRTC for sm_100a (the four throughput/latency x
 * float/int8 kernels; no frame-interleaved or mailbox kernel).  Compiled cubins are cached on
 * disk under a hash of the generated source ($POLAR_JIT_CACHE, default ~/.cache/polar_jit) and
 * shared by handles of the same code in a process.  POLAR_JIT=0 disables it (generic decoder);
 * so does an unrolled length above POLAR_JIT_MAX_OPS Fast-SSC ops (default 4096: the GA codes
 * of this repo have 300-3,600; a random frozen set of N = 32768 has ~60,000, where -- as the
 * paper says of long codes, P:1277 -- the instruction-based decoder is the practical one).
 * POLAR_JIT_FORCE=1 specialises at run time even codes that have a build-time decoder.
 * polar_jit_compile runs the generation and compilation only (no device needed), for checks:
 * POLAR_OK and the cache tag in log, or POLAR_ERR_UNSUPPORTED_CODE and NVRTC's log. */
polar_status polar_jit_compile(uint32_t N, uint32_t K, const uint8_t* frozen_mask, char* log, uint32_t cap);

/* Kernel variant used by the decode calls: 0 = automatic (default: the latency variant,
 * one CTA per frame, when n_frames <= number of SMs (x4 for N >= 16384); for int8 codes with
 * N <= 1024 and n_frames >= 128 x number of SMs the frame-interleaved variant; else the
 * throughput variant, one warp per frame), 1 = always throughput, 2 = always latency,
 * 3 = the generic program-interpreted decoder, 4 = frame-interleaved (one lane per frame,
 * int8 only; f32 calls use the throughput variant).  All decode identically (bit for bit).
 * Returns POLAR_ERR_INVALID_ARGUMENT for any other value.  Not thread-safe with concurrent
 * decode calls on the same handle. */
polar_status polar_code_set_variant(polar_code* h, int variant);

/* Information bits the decode calls return (default POLAR_OUTPUT_SYSTEMATIC):
 *   POLAR_OUTPUT_SYSTEMATIC     x_hat[A], the systematic code's information bits (reading C4);
 *   POLAR_OUTPUT_NONSYSTEMATIC  u_hat[A] with u_hat = x_hat G_N (G_N its own inverse):
 *                               the information bits of the non-systematic code x = u G_N.
 * Same decoder either way; the kernels apply the polar transform to the decoded codeword
 * before the gather.  The frame-interleaved variant (4) is systematic only (its decode calls
 * then return POLAR_ERR_UNSUPPORTED_CODE); a mailbox opened afterwards uses the mode.  Not
 * thread-safe with concurrent decode calls on the same handle. */
enum { POLAR_OUTPUT_SYSTEMATIC = 0, POLAR_OUTPUT_NONSYSTEMATIC = 1 };
polar_status polar_code_set_output(polar_code* h, int mode);

/* Copy the handle's frozen mask (N bytes, 1 = frozen) into host buffer mask_out. */
polar_status polar_code_mask(const polar_code* h, uint8_t* mask_out);

/* Fast-SSC decoding, float profile (min-sum f eq:f P:295-302, g eq:g
 * P:304-315, combine eq:combine P:318-325, Rate-0/Rate-1 P:327-328, repetition
 * P:431-440, SPC P:442-459).
 *   llr        device, float32 [n_frames][N], 16-byte aligned;
 *   n_frames   >= 0 (0 is a no-op);
 *   info_bits  device, uint32 [n_frames][ceil(K/32)]: the systematic information bits
 *              x_hat[A] of each decoded codeword (reading C4/C5); padding bits are 0;
 *   stream     CUDA stream.
 * Every f/g is one IEEE binary32 operation (no FMA contraction); repetition sums use the
 * pairwise-halving order (reading C13); ties follow readings C9-C11. */
polar_status polar_decode_f32(const polar_code* h, const float* llr, int64_t n_frames,
                              uint32_t* info_bits, polar_stream stream);

/* Fast-SSC decoding, 8-bit fixed-point profile: int8 LLRs in [-127,127]
 * (an input of -128 is clamped to -127 on ingest, reading C8); only g can grow a
 * magnitude and it saturates to [-127,127]; repetition sums are exact (reading C12).
 * Arguments as polar_decode_f32 with llr = device int8 [n_frames][N], 16-byte aligned. */
polar_status polar_decode_i8(const polar_code* h, const int8_t* llr, int64_t n_frames,
                             uint32_t* info_bits, polar_stream stream);

/* End-to-end variants over HOST buffers (the paper's latency includes copying the frame
 * to decoder memory and the codeword back): host llr -> device (chunked,
 * overlapped over the handle's internal streams) -> decode -> host info bits.  Blocking:
 * returns when host_info is written.  host buffers may be pageable or pinned (pinned is
 * faster).  Uses device staging buffers owned by the handle, allocated on first use. */
polar_status polar_decode_f32_host(polar_code* h, const float* host_llr, int64_t n_frames,
                                   uint32_t* host_info);
polar_status polar_decode_i8_host(polar_code* h, const int8_t* host_llr, int64_t n_frames,
                                  uint32_t* host_info);

/* Batch-1 mailbox (the paper's latency includes the frame copy in and the
 * estimate out).  polar_mailbox_open launches ONE persistent CTA running the
 * handle's unrolled int8 latency decoder, which polls a control word in host-mapped pinned
 * memory; it occupies one SM until polar_mailbox_close (or until idle_seconds, in (0, 3600],
 * pass without a request, after which it exits on its own).  polar_mailbox_decode_i8 copies
 * one frame of N int8 LLRs from host_llr (any host memory) into the mapped frame buffer,
 * posts it, spins until the kernel has written x_hat[A] (ceil(K/32) words, same packing as
 * polar_decode_i8) and copies it to host_info: no kernel launch, memcpy call or stream
 * synchronisation per frame.  Blocking; not thread-safe on one handle; while the mailbox is
 * open, a device-wide synchronisation (cudaDeviceSynchronize) would wait for the kernel to
 * exit, so use stream synchronisation for other work on the device.
 * Errors: POLAR_ERR_UNSUPPORTED_CODE if no mailbox kernel was built for the code (codes.txt
 * MAILBOX=1); POLAR_ERR_INVALID_ARGUMENT for null pointers, bad idle_seconds, a second open or
 * a decode without open; POLAR_ERR_CUDA if the kernel does not answer within timeout_seconds
 * (it timed out idle or faulted: close and reopen); POLAR_ERR_OUT_OF_MEMORY. */
polar_status polar_mailbox_open(polar_code* h, double idle_seconds);
polar_status polar_mailbox_decode_i8(polar_code* h, const int8_t* host_llr, uint32_t* host_info,
                                     double timeout_seconds);
polar_status polar_mailbox_close(polar_code* h);

/* ---------------------------------------------------------------- non-hot helpers ---- */

/* Gaussian-approximation construction (reading C1; the paper constructs with Tal-Vardy
 * at an unstated design SNR): freezes the N-K bit channels with the smallest GA
 * mean LLR for BPSK-AWGN at design_ebn0_db and rate K/N; ties freeze the lower index.
 * mask_out: host, N bytes. Deterministic; host only. */
polar_status polar_construct_ga(uint32_t N, uint32_t K, double design_ebn0_db,
                                uint8_t* mask_out);

/* Systematic encoding (reading C4): codeword x with x[A] = d and x = u G_N, u[frozen] = 0
 * (G_N = F^{(x) log2 N}, natural indexing), computed as x = mask_A(v G) G with
 * v[A] = d, v[F] = 0.  Needs an information set closed under bit-superset (true of every
 * reliability construction); otherwise POLAR_ERR_UNSUPPORTED_CODE (also for the generator).
 *   info      device uint32 [n_frames][ceil(K/32)] packed information bits;
 *   codeword  device uint32 [n_frames][ceil(N/32)] packed codeword bits. */
polar_status polar_encode_systematic(const polar_code* h, const uint32_t* info, int64_t n_frames,
                                     uint32_t* codeword, polar_stream stream);

/* BPSK-AWGN frame generator (the paper's random codewords; readings C6/C7):
 * for global frames first_frame .. first_frame+n_frames-1, draws K random information
 * bits, encodes them systematically, maps 0 -> +1, 1 -> -1, adds N(0, sigma^2) noise with
 * sigma^2 = 1/(2 (K/N) 10^(ebn0_db/10)), and writes LLR = 2y/sigma^2.  Random numbers come
 * from Philox4x32-10 keyed by seed with counter (frame, word), so a frame does not depend
 * on batching.  Outputs (device; any may be NULL):
 *   llr_f32  float  [n_frames][N];
 *   llr_i8   int8   [n_frames][N], q = clamp(rint(q_scale * LLR), -127, 127);
 *   info     uint32 [n_frames][ceil(K/32)], the transmitted information bits. */
polar_status polar_gen_bpsk_awgn(const polar_code* h, uint64_t seed, uint64_t first_frame,
                                 int64_t n_frames, double ebn0_db, float q_scale,
                                 float* llr_f32, int8_t* llr_i8, uint32_t* info,
                                 polar_stream stream);

/* Error counting (bench / FER mode): compares decoded and transmitted information bits
 * of n_frames frames and ADDS into counters (device int64[3]):
 *   counters[0] += n_frames, counters[1] += bit errors, counters[2] += frame errors. */
polar_status polar_count_errors(const polar_code* h, const uint32_t* decoded,
                                const uint32_t* truth, int64_t n_frames, int64_t* counters,
                                polar_stream stream);

/* Diagnostics of POLAR_TRACE builds only (otherwise POLAR_ERR_UNSUPPORTED_CODE): copy the
 * clock64() stamps the latency variant recorded after each operation of its last decoded
 * frame 0 (host buffer, n entries; labels in build/gen/trace_<code>.txt). */
polar_status polar_trace_fetch(const polar_code* h, uint64_t* host, uint32_t n);

/* Diagnostics of POLAR_DEBUG_DUMP builds only (libpolar_dump.so; otherwise
 * POLAR_ERR_UNSUPPORTED_CODE).  Each decode of at most 8 frames by the throughput or latency
 * variant of a specialised code appends, per frame and in the decoder's op order (Listing 1,
 * P:644-656), every F / G / G_0R output vector (eq:f P:295-302, eq:g P:304-315) as floats
 * (int8 profile: the integer values).  *stride = floats reserved per frame (N log2 N; unused
 * entries are NaN); fetch copies n floats of frames 0.. of the last decode into host. */
polar_status polar_debug_dump_stride(const polar_code* h, uint64_t* stride);
polar_status polar_debug_dump_fetch(const polar_code* h, float* host, uint64_t n);

/* Number of specialised codes compiled into this library, and the i-th one's (N, K) and
 * frozen mask (host buffer of at least N bytes; may be NULL to query N and K only). */
uint32_t polar_registry_size(void);
polar_status polar_registry_entry(uint32_t i, uint32_t* N, uint32_t* K, uint8_t* mask_out);

#ifdef __cplusplus
}
#endif

#endif /* POLAR_H */
