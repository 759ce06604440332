/*
 * polar_oracle.c -- TEST INFRASTRUCTURE ONLY (never linked by the product).
 *
 * A plain, slow, obviously-correct CPU reference for what the hot path computes:
 * Fast-SSC decoding of polar codes as stated in Giard et al., "Low-Latency Software
 * Polar Decoders" (arXiv:1504.00353).  Citations "P:n" are line numbers of
 * /root/reference/PAPER.md (the LaTeX source) at the time this file was written.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference leg may
 * load this library.  It shares no code, header, table or constant with the product
 * (paper_1504_00353_b200/, include/): the two are written independently from the paper.
 *
 * Built with `gcc -O2 -std=c11 -fno-fast-math -ffp-contract=off` so that every float
 * operation is one IEEE binary32 operation in source order (reading C17 in DESIGN.md).
 *
 * Contents (each cites the passage it follows):
 *   or_f_f32 / or_g_f32 / or_f_i8 / or_g_i8     eq:f P:295-302, eq:g P:304-315, int8 P:485-486
 *   or_encode, or_encode_matrix                 G_N = F_2^{(x)log2 N}, natural indexing P:139-155
 *   or_encode_systematic                        systematic encoding by definition (reading C4)
 *   or_sc_decode_{f32,i8}        (O1)           plain SC
 *   or_fastssc_decode_{f32,i8}   (O2)           Fast-SSC node rules P:327-328
 *   or_ml_decode_f32             (O3)           brute-force ML over all codewords (N <= 16)
 *   or_rep_*, or_spc_*                          the node decoders on their own
 *   or_construct_ga                             construction (reading C1: Gaussian approximation)
 *   or_bhattacharyya_bec                        textbook BEC recursion used only as a cross-pin
 *
 * Parity pins live in tests/test_oracle_*.py.  Functions without an independent pin say
 * so in their header comment ("parity unpinned") and in DESIGN.md.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------ */
/* Node primitives.                                                                     */
/* ------------------------------------------------------------------------------------ */

/* eq:f: f(a,b) = sgn(a) sgn(b) min(|a|,|b|) (min-sum).  A zero operand gives a
 * zero result whatever sign bit it carries; decisions never read the sign of a zero
 * (reading C9), so the sign chosen for a zero result is irrelevant. */
float or_f_f32(float a, float b) {
    float ma = fabsf(a), mb = fabsf(b);
    float m = (mb < ma) ? mb : ma;
    int negative = (a < 0.0f) != (b < 0.0f);
    return negative ? -m : m;
}

/* eq:g: g(a,b,beta) = b + a when beta = 0, b - a otherwise, where
 * a = alpha_v[i], b = alpha_v[i + N_v/2].  One IEEE operation (reading C17). */
float or_g_f32(float a, float b, int beta) {
    return beta ? (b - a) : (b + a);
}

/* int8 profile: 8-bit LLRs, "only the G function adds to the amplitude of
 * LLRs and it is carried out with saturating adders".  Range [-127, 127] (reading C8:
 * Listing 4 P:842-864 clamps with max(-127, .)).  f needs no saturation: min(|a|,|b|) <= 127. */
int or_f_i8(int a, int b) {
    int ma = a < 0 ? -a : a, mb = b < 0 ? -b : b;
    int m = mb < ma ? mb : ma;
    int negative = (a < 0) != (b < 0);
    return negative ? -m : m;
}

int or_g_i8(int a, int b, int beta) {
    int s = beta ? (b - a) : (b + a);
    if (s > 127) s = 127;
    if (s < -127) s = -127;
    return s;
}

/* Ingest of an int8 channel LLR: -128 is outside the symmetric range and is clamped to
 * -127 (reading C8; the ABI documents the same). */
static int ingest_i8(int8_t v) { return v < -127 ? -127 : (int)v; }

/* Hard decision, eq:info: 0 when alpha >= 0, 1 otherwise.  By comparison, so
 * -0.0 decides 0 (reading C9). */
static uint8_t hd_f32(float a) { return a < 0.0f ? 1 : 0; }
static uint8_t hd_i8(int a) { return a < 0 ? 1 : 0; }

/* ------------------------------------------------------------------------------------ */
/* Encoding: x = u G_N with G_N = F_2^{(x) log2 N}, F_2 = [1 0; 1 1], natural indexing     */
/* (P:139-155).                                                                          */
/* ------------------------------------------------------------------------------------ */

/* By the matrix definition: G_N[i][j] = 1 iff the bits of j are a subset of the bits of i
 * (the Kronecker power of the lower-triangular F_2).  O(N^2); used for small N and as a
 * pin of or_encode.  Pinned against G_4 as printed at P:142-151. */
void or_encode_matrix(int N, const uint8_t* u, uint8_t* x) {
    for (int j = 0; j < N; ++j) {
        uint8_t acc = 0;
        for (int i = 0; i < N; ++i)
            if ((i & j) == j) acc ^= (uint8_t)(u[i] & 1);
        x[j] = acc;
    }
}

/* By the block form G_N = [G_{N/2} 0; G_{N/2} G_{N/2}]:
 * x = (u_L G ^ u_R G, u_R G), recursively. */
static void encode_rec(int n, const uint8_t* u, uint8_t* x) {
    if (n == 1) { x[0] = u[0] & 1; return; }
    int h = n / 2;
    encode_rec(h, u, x);
    encode_rec(h, u + h, x + h);
    for (int i = 0; i < h; ++i) x[i] ^= x[i + h];
}

void or_encode(int N, const uint8_t* u, uint8_t* x) { encode_rec(N, u, x); }

/* Systematic encoding (reading C4; the paper's decoders return the codeword estimate,
 * P:477, and the north star asks for systematic frames).  By definition: find the
 * codeword x = u G with u[F] = 0 and x[A] = d (A = information set in ascending order).
 * x[j] = XOR_{i superset of j} u[i] (G_N[i][j] = [j subset i]), so for j in A, from the
 * highest index down, u[j] = d_j XOR (XOR_{i strict superset of j} u[i]).  This works for
 * any frozen set; it does not use the two-pass shortcut the product uses. */
void or_encode_systematic(int N, const uint8_t* frozen, const uint8_t* d, uint8_t* x) {
    uint8_t* u = (uint8_t*)calloc((size_t)N, 1);
    int K = 0;
    for (int j = 0; j < N; ++j) K += frozen[j] ? 0 : 1;
    int t = K;
    for (int j = N - 1; j >= 0; --j) {
        if (frozen[j]) continue;
        --t;
        uint8_t acc = d[t] & 1;
        /* enumerate strict supersets i of j within [0, N) */
        int comp = (N - 1) & ~j;
        for (int s = comp; s != 0; s = (s - 1) & comp) acc ^= u[j | s];
        u[j] = acc;
    }
    or_encode(N, u, x);
    free(u);
}

/* ------------------------------------------------------------------------------------ */
/* O1: plain successive-cancellation decoding, no node specialisation.       */
/* The tree is traversed depth first, left before right, down to size-1 leaves; frozen   */
/* leaves decide 0, information leaves threshold-detect.                         */
/* ------------------------------------------------------------------------------------ */

typedef struct {
    int zero_decisions; /* information leaves decided on an exactly-zero LLR */
} sc_stats;

static void sc_f32(int n, const uint8_t* frozen, const float* alpha, uint8_t* beta,
                   uint8_t* uhat, float* scratch, sc_stats* st) {
    if (n == 1) {
        if (frozen[0]) beta[0] = 0;
        else {
            beta[0] = hd_f32(alpha[0]);
            if (alpha[0] == 0.0f) st->zero_decisions++;
        }
        uhat[0] = beta[0];
        return;
    }
    int h = n / 2;
    float* child = scratch; /* h values; the rest of scratch belongs to deeper levels */
    for (int i = 0; i < h; ++i) child[i] = or_f_f32(alpha[i], alpha[i + h]);
    sc_f32(h, frozen, child, beta, uhat, scratch + h, st);
    for (int i = 0; i < h; ++i) child[i] = or_g_f32(alpha[i], alpha[i + h], beta[i]);
    sc_f32(h, frozen + h, child, beta + h, uhat + h, scratch + h, st);
    for (int i = 0; i < h; ++i) beta[i] ^= beta[i + h]; /* eq:combine P:318-325 */
}

static void sc_i8(int n, const uint8_t* frozen, const int* alpha, uint8_t* beta,
                  uint8_t* uhat, int* scratch, sc_stats* st) {
    if (n == 1) {
        if (frozen[0]) beta[0] = 0;
        else {
            beta[0] = hd_i8(alpha[0]);
            if (alpha[0] == 0) st->zero_decisions++;
        }
        uhat[0] = beta[0];
        return;
    }
    int h = n / 2;
    int* child = scratch;
    for (int i = 0; i < h; ++i) child[i] = or_f_i8(alpha[i], alpha[i + h]);
    sc_i8(h, frozen, child, beta, uhat, scratch + h, st);
    for (int i = 0; i < h; ++i) child[i] = or_g_i8(alpha[i], alpha[i + h], beta[i]);
    sc_i8(h, frozen + h, child, beta + h, uhat + h, scratch + h, st);
    for (int i = 0; i < h; ++i) beta[i] ^= beta[i + h];
}

/* Decode n_frames frames of N LLRs each (frame-major).  xhat, uhat: n_frames*N bytes
 * (uhat may be NULL).  zero_dec (may be NULL): per-frame count of information-leaf
 * decisions taken on an exactly-zero LLR ("tie frames", SURVEY 8(c) pin 5/6). */
void or_sc_decode_f32(int N, const uint8_t* frozen, const float* llr, long n_frames,
                      uint8_t* xhat, uint8_t* uhat, int* zero_dec) {
    float* scratch = (float*)malloc(sizeof(float) * (size_t)N);
    uint8_t* ub = (uint8_t*)malloc((size_t)N);
    for (long fr = 0; fr < n_frames; ++fr) {
        sc_stats st = {0};
        sc_f32(N, frozen, llr + fr * N, xhat + fr * N, ub, scratch, &st);
        if (uhat) memcpy(uhat + fr * N, ub, (size_t)N);
        if (zero_dec) zero_dec[fr] = st.zero_decisions;
    }
    free(ub);
    free(scratch);
}

void or_sc_decode_i8(int N, const uint8_t* frozen, const int8_t* llr, long n_frames,
                     uint8_t* xhat, uint8_t* uhat, int* zero_dec) {
    int* in = (int*)malloc(sizeof(int) * (size_t)N);
    int* scratch = (int*)malloc(sizeof(int) * (size_t)N);
    uint8_t* ub = (uint8_t*)malloc((size_t)N);
    for (long fr = 0; fr < n_frames; ++fr) {
        sc_stats st = {0};
        for (int i = 0; i < N; ++i) in[i] = ingest_i8(llr[fr * N + i]);
        sc_i8(N, frozen, in, xhat + fr * N, ub, scratch, &st);
        if (uhat) memcpy(uhat + fr * N, ub, (size_t)N);
        if (zero_dec) zero_dec[fr] = st.zero_decisions;
    }
    free(ub);
    free(scratch);
    free(in);
}

/* ------------------------------------------------------------------------------------ */
/* Fast-SSC node decoders.                                        */
/* ------------------------------------------------------------------------------------ */

enum { OR_RATE0 = 0, OR_RATE1 = 1, OR_REP = 2, OR_SPC = 3, OR_SPLIT = 4 };

/* Node classification in priority order (reading C14): Rate-0 (all frozen),
 * Rate-1 (none frozen), Repetition (only the last bit is information),
 * SPC (only the first bit is frozen), otherwise split into two halves. */
int or_classify(int n, const uint8_t* frozen) {
    int nf = 0;
    for (int i = 0; i < n; ++i) nf += frozen[i] ? 1 : 0;
    if (nf == n) return OR_RATE0;
    if (nf == 0) return OR_RATE1;
    if (nf == n - 1 && !frozen[n - 1]) return OR_REP;
    if (nf == 1 && frozen[0]) return OR_SPC;
    return OR_SPLIT;
}

/* Repetition: beta = 0 everywhere when sum(alpha) >= 0, else 1 everywhere.
 * f32: the sum is taken in pairwise-halving order, x[i] <- x[i] + x[i + m/2] for
 * m = n, n/2, ..., 2 (reading C13; the paper does not fix an order). */
void or_rep_f32(int n, const float* alpha, uint8_t* beta) {
    float* t = (float*)malloc(sizeof(float) * (size_t)n);
    memcpy(t, alpha, sizeof(float) * (size_t)n);
    for (int m = n; m > 1; m /= 2)
        for (int i = 0; i < m / 2; ++i) t[i] = t[i] + t[i + m / 2];
    uint8_t b = t[0] < 0.0f ? 1 : 0;
    for (int i = 0; i < n; ++i) beta[i] = b;
    free(t);
}

/* int8: the sum is exact in int (reading C12). */
void or_rep_i8(int n, const int* alpha, uint8_t* beta) {
    long s = 0;
    for (int i = 0; i < n; ++i) s += alpha[i];
    uint8_t b = s < 0 ? 1 : 0;
    for (int i = 0; i < n; ++i) beta[i] = b;
}

/* SPC: hard decisions (eq:info), parity of the decisions, and when the parity
 * is 1 flip the decision at argmin |alpha|.  Ties in argmin take the lowest index
 * (reading C10; Listing 2's tzcnt, returns the lowest lane). */
void or_spc_f32(int n, const float* alpha, uint8_t* beta) {
    uint8_t parity = 0;
    int idx = 0;
    float best = fabsf(alpha[0]);
    for (int i = 0; i < n; ++i) {
        beta[i] = hd_f32(alpha[i]);
        parity ^= beta[i];
        float m = fabsf(alpha[i]);
        if (m < best) { best = m; idx = i; }
    }
    if (parity) beta[idx] ^= 1;
}

void or_spc_i8(int n, const int* alpha, uint8_t* beta) {
    uint8_t parity = 0;
    int idx = 0;
    int best = alpha[0] < 0 ? -alpha[0] : alpha[0];
    for (int i = 0; i < n; ++i) {
        beta[i] = hd_i8(alpha[i]);
        parity ^= beta[i];
        int m = alpha[i] < 0 ? -alpha[i] : alpha[i];
        if (m < best) { best = m; idx = i; }
    }
    if (parity) beta[idx] ^= 1;
}

/* ------------------------------------------------------------------------------------ */
/* O2: straightforward Fast-SSC (function vocabulary P:472).                   */
/* Written separately from O1: the same recursion, but every node is first classified    */
/* and Rate-0 / Rate-1 / Repetition / SPC nodes are decoded by their rules.  A split node */
/* whose left child is Rate-0 runs G_0R (beta_l = 0) and Combine_0R; one whose right     */
/* child is Rate-0 leaves beta = (beta_l, 0) (reading C16).                              */
/* An optional trace records the op sequence in Listing 1's vocabulary.      */
/* ------------------------------------------------------------------------------------ */

typedef struct {
    char* buf;
    int cap;
    int len;
    /* node set (0 Fast-SSC, 1 no SPC, 2 SSC, 3 plain SC): the paper's algorithm ablation
     * (tab:impl:tp:algo-unroll; the GPU decoder without SPC nodes P:1134-1136) */
    int set;
    /* optional alpha dump: every F / G / G_0R output vector appended in op order (the
     * intermediate LLRs the north star's float bar compares, 1e-5 relative); records only */
    float* af;
    int* ai;
    long apos, acap;
} or_trace;

/* or_classify restricted to the trace's node set: SC splits every node of size > 1, SSC
 * keeps only Rate-0 / Rate-1, "no SPC" keeps Rate-0 / Rate-1 / repetition. */
static int classify_set(int n, const uint8_t* frozen, const or_trace* tr) {
    const int set = tr ? tr->set : 0;
    if (set == 3 && n > 1) return OR_SPLIT;
    const int k = or_classify(n, frozen);
    if (set == 2 && (k == OR_REP || k == OR_SPC)) return OR_SPLIT;
    if (set == 1 && k == OR_SPC) return OR_SPLIT;
    return k;
}

static void dump_f32(or_trace* tr, const float* v, int h) {
    if (!tr || !tr->af) return;
    for (int i = 0; i < h && tr->apos < tr->acap; ++i) tr->af[tr->apos++] = v[i];
}
static void dump_i8(or_trace* tr, const int* v, int h) {
    if (!tr || !tr->ai) return;
    for (int i = 0; i < h && tr->apos < tr->acap; ++i) tr->ai[tr->apos++] = v[i];
}

static void trace_op(or_trace* tr, const char* name, int n) {
    if (!tr || !tr->buf) return;
    char tmp[64];
    int k = 0;
    const char* p = name;
    while (*p && k < 40) tmp[k++] = *p++;
    tmp[k++] = '<';
    /* decimal n */
    char digits[16];
    int nd = 0;
    int v = n;
    do { digits[nd++] = (char)('0' + v % 10); v /= 10; } while (v);
    while (nd) tmp[k++] = digits[--nd];
    tmp[k++] = '>';
    tmp[k++] = ';';
    if (tr->len + k + 1 >= tr->cap) return;
    memcpy(tr->buf + tr->len, tmp, (size_t)k);
    tr->len += k;
    tr->buf[tr->len] = 0;
}

static void fssc_f32(int n, const uint8_t* frozen, const float* alpha, uint8_t* beta,
                     float* scratch, or_trace* tr) {
    int kind = classify_set(n, frozen, tr);
    if (kind == OR_RATE0) { for (int i = 0; i < n; ++i) beta[i] = 0; return; }
    if (kind == OR_RATE1) {
        trace_op(tr, "Info", n);
        for (int i = 0; i < n; ++i) beta[i] = hd_f32(alpha[i]);
        return;
    }
    if (kind == OR_REP) { trace_op(tr, "Repetition", n); or_rep_f32(n, alpha, beta); return; }
    if (kind == OR_SPC) { trace_op(tr, "SPC", n); or_spc_f32(n, alpha, beta); return; }
    int h = n / 2;
    float* child = scratch;
    int left = classify_set(h, frozen, tr), right = classify_set(h, frozen + h, tr);
    if (left == OR_RATE0) {
        trace_op(tr, "G_0R", n);
        for (int i = 0; i < h; ++i) { beta[i] = 0; child[i] = or_g_f32(alpha[i], alpha[i + h], 0); }
        dump_f32(tr, child, h);
        fssc_f32(h, frozen + h, child, beta + h, scratch + h, tr);
        trace_op(tr, "Combine_0R", n);
        for (int i = 0; i < h; ++i) beta[i] = beta[i + h];
        return;
    }
    trace_op(tr, "F", n);
    for (int i = 0; i < h; ++i) child[i] = or_f_f32(alpha[i], alpha[i + h]);
    dump_f32(tr, child, h);
    fssc_f32(h, frozen, child, beta, scratch + h, tr);
    if (right == OR_RATE0) {
        trace_op(tr, "Combine_R0", n);
        for (int i = 0; i < h; ++i) beta[i + h] = 0;
        return;
    }
    trace_op(tr, "G", n);
    for (int i = 0; i < h; ++i) child[i] = or_g_f32(alpha[i], alpha[i + h], beta[i]);
    dump_f32(tr, child, h);
    fssc_f32(h, frozen + h, child, beta + h, scratch + h, tr);
    trace_op(tr, "Combine", n);
    for (int i = 0; i < h; ++i) beta[i] ^= beta[i + h];
}

static void fssc_i8(int n, const uint8_t* frozen, const int* alpha, uint8_t* beta,
                    int* scratch, or_trace* tr) {
    int kind = classify_set(n, frozen, tr);
    if (kind == OR_RATE0) { for (int i = 0; i < n; ++i) beta[i] = 0; return; }
    if (kind == OR_RATE1) {
        trace_op(tr, "Info", n);
        for (int i = 0; i < n; ++i) beta[i] = hd_i8(alpha[i]);
        return;
    }
    if (kind == OR_REP) { trace_op(tr, "Repetition", n); or_rep_i8(n, alpha, beta); return; }
    if (kind == OR_SPC) { trace_op(tr, "SPC", n); or_spc_i8(n, alpha, beta); return; }
    int h = n / 2;
    int* child = scratch;
    int left = classify_set(h, frozen, tr), right = classify_set(h, frozen + h, tr);
    if (left == OR_RATE0) {
        trace_op(tr, "G_0R", n);
        for (int i = 0; i < h; ++i) { beta[i] = 0; child[i] = or_g_i8(alpha[i], alpha[i + h], 0); }
        dump_i8(tr, child, h);
        fssc_i8(h, frozen + h, child, beta + h, scratch + h, tr);
        trace_op(tr, "Combine_0R", n);
        for (int i = 0; i < h; ++i) beta[i] = beta[i + h];
        return;
    }
    trace_op(tr, "F", n);
    for (int i = 0; i < h; ++i) child[i] = or_f_i8(alpha[i], alpha[i + h]);
    dump_i8(tr, child, h);
    fssc_i8(h, frozen, child, beta, scratch + h, tr);
    if (right == OR_RATE0) {
        trace_op(tr, "Combine_R0", n);
        for (int i = 0; i < h; ++i) beta[i + h] = 0;
        return;
    }
    trace_op(tr, "G", n);
    for (int i = 0; i < h; ++i) child[i] = or_g_i8(alpha[i], alpha[i + h], beta[i]);
    dump_i8(tr, child, h);
    fssc_i8(h, frozen + h, child, beta + h, scratch + h, tr);
    trace_op(tr, "Combine", n);
    for (int i = 0; i < h; ++i) beta[i] ^= beta[i + h];
}

void or_fastssc_decode_f32(int N, const uint8_t* frozen, const float* llr, long n_frames,
                           uint8_t* xhat) {
    float* scratch = (float*)malloc(sizeof(float) * (size_t)N);
    for (long fr = 0; fr < n_frames; ++fr)
        fssc_f32(N, frozen, llr + fr * N, xhat + fr * N, scratch, NULL);
    free(scratch);
}

void or_fastssc_decode_i8(int N, const uint8_t* frozen, const int8_t* llr, long n_frames,
                          uint8_t* xhat) {
    int* in = (int*)malloc(sizeof(int) * (size_t)N);
    int* scratch = (int*)malloc(sizeof(int) * (size_t)N);
    for (long fr = 0; fr < n_frames; ++fr) {
        for (int i = 0; i < N; ++i) in[i] = ingest_i8(llr[fr * N + i]);
        fssc_i8(N, frozen, in, xhat + fr * N, scratch, NULL);
    }
    free(scratch);
    free(in);
}

/* O2 restricted to a node set (set: 0 Fast-SSC = or_fastssc_decode_*, 1 no SPC, 2 SSC,
 * 3 plain SC through the same traversal): the references of the GPU ablation builds. */
void or_nodeset_decode_f32(int N, const uint8_t* frozen, const float* llr, long n_frames, uint8_t* xhat, int set) {
    float* scratch = (float*)malloc(sizeof(float) * (size_t)N);
    or_trace tr = {NULL, 0, 0, set, NULL, NULL, 0, 0};
    for (long fr = 0; fr < n_frames; ++fr) fssc_f32(N, frozen, llr + fr * N, xhat + fr * N, scratch, &tr);
    free(scratch);
}

void or_nodeset_decode_i8(int N, const uint8_t* frozen, const int8_t* llr, long n_frames, uint8_t* xhat, int set) {
    int* in = (int*)malloc(sizeof(int) * (size_t)N);
    int* scratch = (int*)malloc(sizeof(int) * (size_t)N);
    or_trace tr = {NULL, 0, 0, set, NULL, NULL, 0, 0};
    for (long fr = 0; fr < n_frames; ++fr) {
        for (int i = 0; i < N; ++i) in[i] = ingest_i8(llr[fr * N + i]);
        fssc_i8(N, frozen, in, xhat + fr * N, scratch, &tr);
    }
    free(scratch);
    free(in);
}

int or_nodeset_trace(int N, const uint8_t* frozen, int set, char* buf, int cap) {
    float* llr = (float*)calloc((size_t)N, sizeof(float));
    float* scratch = (float*)malloc(sizeof(float) * (size_t)N);
    uint8_t* xhat = (uint8_t*)malloc((size_t)N);
    or_trace tr = {buf, cap, 0, set, NULL, NULL, 0, 0};
    if (cap > 0) buf[0] = 0;
    fssc_f32(N, frozen, llr, xhat, scratch, &tr);
    free(xhat);
    free(scratch);
    free(llr);
    return tr.len;
}

/* Listing-1-style trace of the op sequence O2 executes on one f32 frame ("F<8>;G_0R<4>;..."). */
int or_fastssc_trace(int N, const uint8_t* frozen, char* buf, int cap) {
    float* llr = (float*)calloc((size_t)N, sizeof(float));
    float* scratch = (float*)malloc(sizeof(float) * (size_t)N);
    uint8_t* xhat = (uint8_t*)malloc((size_t)N);
    or_trace tr = {buf, cap, 0, 0, NULL, NULL, 0, 0};
    if (cap > 0) buf[0] = 0;
    fssc_f32(N, frozen, llr, xhat, scratch, &tr);
    free(xhat);
    free(scratch);
    free(llr);
    return tr.len;
}

/* O2 on one frame, recording every F / G / G_0R output vector in op order (or_trace.af/ai):
 * returns the number of values written (at most cap).  The decode itself is unchanged. */
long or_fastssc_dump_f32(int N, const uint8_t* frozen, const float* llr, uint8_t* xhat, float* out, long cap) {
    float* scratch = (float*)malloc(sizeof(float) * (size_t)N);
    or_trace tr = {NULL, 0, 0, 0, out, NULL, 0, cap};
    fssc_f32(N, frozen, llr, xhat, scratch, &tr);
    free(scratch);
    return tr.apos;
}

long or_fastssc_dump_i8(int N, const uint8_t* frozen, const int8_t* llr, uint8_t* xhat, int* out, long cap) {
    int* in = (int*)malloc(sizeof(int) * (size_t)N);
    int* scratch = (int*)malloc(sizeof(int) * (size_t)N);
    for (int i = 0; i < N; ++i) in[i] = ingest_i8(llr[i]);
    or_trace tr = {NULL, 0, 0, 0, NULL, out, 0, cap};
    fssc_i8(N, frozen, in, xhat, scratch, &tr);
    free(scratch);
    free(in);
    return tr.apos;
}

/* Standalone node decoders for unit pins (int8 versions take int8 inputs). */
void or_rep_i8_bytes(int n, const int8_t* alpha, uint8_t* beta) {
    int* t = (int*)malloc(sizeof(int) * (size_t)n);
    for (int i = 0; i < n; ++i) t[i] = ingest_i8(alpha[i]);
    or_rep_i8(n, t, beta);
    free(t);
}
void or_spc_i8_bytes(int n, const int8_t* alpha, uint8_t* beta) {
    int* t = (int*)malloc(sizeof(int) * (size_t)n);
    for (int i = 0; i < n; ++i) t[i] = ingest_i8(alpha[i]);
    or_spc_i8(n, t, beta);
    free(t);
}

/* ------------------------------------------------------------------------------------ */
/* O3: brute-force maximum-likelihood decoding, N <= 16.  Enumerates every  */
/* u with u[F] = 0 in increasing order, x = u G, and keeps the first x maximising          */
/* sum_i (1 - 2 x_i) alpha_i (in double).                                                 */
/* ------------------------------------------------------------------------------------ */
void or_ml_decode_f32(int N, const uint8_t* frozen, const float* llr, long n_frames,
                      uint8_t* xhat) {
    int info[16];
    int K = 0;
    for (int i = 0; i < N; ++i) if (!frozen[i]) info[K++] = i;
    uint8_t u[16], x[16];
    for (long fr = 0; fr < n_frames; ++fr) {
        const float* a = llr + fr * N;
        double best = -INFINITY;
        for (long m = 0; m < (1L << K); ++m) {
            memset(u, 0, sizeof u);
            for (int t = 0; t < K; ++t) u[info[t]] = (uint8_t)((m >> t) & 1);
            or_encode_matrix(N, u, x);
            double metric = 0.0;
            for (int i = 0; i < N; ++i) metric += (x[i] ? -1.0 : 1.0) * (double)a[i];
            if (metric > best) {
                best = metric;
                memcpy(xhat + fr * N, x, (size_t)N);
            }
        }
    }
}

/* ------------------------------------------------------------------------------------ */
/* Construction (reading C1).  The paper constructs its codes "according to [Tal2011a]"   */
/* at an unstated design SNR; we use the Gaussian approximation (GA) with Chung's  */
/* two-piece phi, evaluated in the log domain, designed at the configuration's Eb/N0.     */
/* Natural indexing: index bit (n-1) is the transform closest to the channel, so  */
/* one recursion step maps entry j to 2j (check-node / "minus") and 2j+1 (variable-node /  */
/* "plus").  The N-K smallest means are frozen; ties freeze the lower index.             */
/* parity unpinned (the paper's exact frozen sets are not printed): pinned only by        */
/* invariants (bit-dominance monotonicity, agreement with the textbook BEC ordering at    */
/* N = 8, FER close to the GA prediction) -- see DESIGN.md.                               */
/* ------------------------------------------------------------------------------------ */

/* log phi(x), phi(x) = exp(-0.4527 x^0.86 + 0.0218) for x < 10,
 *                      sqrt(pi/x) exp(-x/4) (1 - 10/(7x)) otherwise. */
double or_log_phi(double x) {
    if (x < 10.0) return -0.4527 * pow(x, 0.86) + 0.0218;
    return 0.5 * log(M_PI / x) - x / 4.0 + log(1.0 - 10.0 / (7.0 * x));
}

/* phi^{-1} in the log domain by bisection: the x with log phi(x) = y. */
double or_inv_log_phi(double y) {
    double lo = 0.0, hi = 1.0;
    while (or_log_phi(hi) > y) hi *= 2.0;
    for (int it = 0; it < 200; ++it) {
        double mid = 0.5 * (lo + hi);
        if (or_log_phi(mid) > y) lo = mid; else hi = mid;
    }
    return 0.5 * (lo + hi);
}

/* GA means of the N bit channels for BPSK-AWGN at design Eb/N0 (dB) and rate K/N:
 * sigma^2 = 1 / (2 R 10^(EbN0/10)) (reading C6), channel LLR mean m0 = 2/sigma^2.
 * minus: m- = phi^{-1}(1 - (1 - phi(m))^2); plus: m+ = 2 m. */
void or_ga_means(int N, int K, double design_ebn0_db, double* m_out) {
    double R = (double)K / (double)N;
    double sigma2 = 1.0 / (2.0 * R * pow(10.0, design_ebn0_db / 10.0));
    double* cur = (double*)malloc(sizeof(double) * (size_t)N);
    double* nxt = (double*)malloc(sizeof(double) * (size_t)N);
    cur[0] = 2.0 / sigma2;
    for (int len = 1; len < N; len *= 2) {
        for (int j = 0; j < len; ++j) {
            double m = cur[j];
            double lp = or_log_phi(m);
            double p = exp(lp);
            /* log(1 - (1 - p)^2) = log(p (2 - p)) = lp + log(2 - p) */
            double lminus = lp + log(2.0 - p);
            nxt[2 * j] = or_inv_log_phi(lminus);
            nxt[2 * j + 1] = 2.0 * m;
        }
        double* t = cur; cur = nxt; nxt = t;
    }
    memcpy(m_out, cur, sizeof(double) * (size_t)N);
    free(cur);
    free(nxt);
}

void or_construct_ga(int N, int K, double design_ebn0_db, uint8_t* frozen_out) {
    double* m = (double*)malloc(sizeof(double) * (size_t)N);
    int* order = (int*)malloc(sizeof(int) * (size_t)N);
    or_ga_means(N, K, design_ebn0_db, m);
    for (int i = 0; i < N; ++i) order[i] = i;
    /* insertion sort by (m, index): plain and stable; O(N^2) worst case is fine here */
    for (int i = 1; i < N; ++i) {
        int v = order[i];
        int j = i - 1;
        while (j >= 0 && m[order[j]] > m[v]) { order[j + 1] = order[j]; --j; }
        order[j + 1] = v;
    }
    for (int i = 0; i < N; ++i) frozen_out[i] = 0;
    for (int t = 0; t < N - K; ++t) frozen_out[order[t]] = 1;
    free(order);
    free(m);
}

/* Textbook Bhattacharyya recursion on the BEC(z0) (Arikan 2009): z- = 2z - z^2, z+ = z^2,
 * same natural-index recursion as or_ga_means.  Used only to cross-pin the GA ordering. */
void or_bhattacharyya_bec(int N, double z0, double* z_out) {
    double* cur = (double*)malloc(sizeof(double) * (size_t)N);
    double* nxt = (double*)malloc(sizeof(double) * (size_t)N);
    cur[0] = z0;
    for (int len = 1; len < N; len *= 2) {
        for (int j = 0; j < len; ++j) {
            double z = cur[j];
            nxt[2 * j] = 2.0 * z - z * z;
            nxt[2 * j + 1] = z * z;
        }
        double* t = cur; cur = nxt; nxt = t;
    }
    memcpy(z_out, cur, sizeof(double) * (size_t)N);
    free(cur);
    free(nxt);
}
