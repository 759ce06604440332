// codegen.cpp -- build-time emitter of the unrolled Fast-SSC decoders (product code).
//
// The paper's unrolled decoders are generated per code as a straight list of function calls
// with compile-time sizes (Listing 1; "the decoder ... is generated", P:641;
// template sizes and unrolled loops).  This program does the same for SIMT:
// for every code listed in the spec file it walks the Fast-SSC tree (tree.hpp) depth first
// and writes build/gen/code_<name>.cu, a sequence of calls to the device templates of
// decoder.cuh with every size, register stage and bit offset a compile-time constant, and
// the registry (build/gen/registry.cpp) that polar_code_create searches.
//
// Spec file lines:  <name> <N> <K> ga <design Eb/N0 dB> [W=<warp root>] [T=<threads>]
//                   <name> <N> <K> mask <N characters 0/1, 1 = frozen>   [...]
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <algorithm>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "jit.hpp"
#include "tree.hpp"

namespace polar {
void construct_ga(int N, int K, double design_ebn0_db, uint8_t* frozen);
}

using namespace polar;

namespace {

int ilog2(int n) {
    int k = 0;
    while ((1 << k) < n) ++k;
    return k;
}

struct Spec {
    std::string name;
    int N = 0, K = 0;
    std::vector<uint8_t> mask;
    int W = 1024;   // warp subtree size for CTA mode
    int T = 512;    // threads per CTA in CTA mode
    int fpc_max = 16;  // most lockstep frames (warps) per CTA in the throughput variant
    std::set<int> dedup;  // sizes of subtrees shared as noinline functions (DEDUP=16,32,..)
    int ll = 0;           // lane-local tiny subtrees up to this size (LL=8 enables; measured slower, profiles/r1_history.md)
    int cps = 1;          // throughput variant: CTAs per SM requested from ptxas (__launch_bounds__ min blocks)
    int wlat = 0;         // latency variant's warp-subtree size (WLAT=; default W)
    int wf = 0;           // f32 throughput variant's warp-subtree size (WF=; default W)
    int xw = 0;           // latency variant: CTA-level nodes up to XW run on warp 0 alone (XW=)
    int helper = 0;       // latency variant: run-ahead helper warp on scheduler HELPER-1 (HELPER=1|2)
    bool latni = false;   // latency variant: non-inlined subtree copies (LATNI=1)
    bool gbeta = false;   // throughput variant: decision bits in the global slot scratch too (GBETA=1)
    int gs = -1;          // stages of size >= gs live in global scratch in the throughput variant
    int h16 = 0;          // int8 throughput variant: stages of size <= h16 stored as f16 (H16=; 0: none)
    NodeSet nodes = NodeSet::FastSSC;  // NODES=fastssc|nospc|ssc|sc: the algorithm ablation (tree.hpp)
    bool repspc = false;  // speculative RepSPC nodes in the warp subtrees (REPSPC=1; measured
                          // neutral for batch-1 latency and -2% throughput at N = 32768: opt-in)
    int xsm = 48 * 1024;  // frame-interleaved variant: shared-memory budget per warp (XSM=; 24K/48K/72K
                          // measured 162/262/207 Gbps at (2048,1723), profiles/r1_history.md)
    int xwpc = 1;         // frame-interleaved variant: warps per CTA (XWPC=)
    bool mailbox = false; // batch-1 persistent mailbox kernel of the int8 latency variant (MAILBOX=1)
    bool fcomb = false;   // FCOMB=1: a warp-subtree right child performs its CTA-level parent's Combine
                          // (measured: (32768,29492) +0.6%, (2048,1723) -1.4%, batch-1 -0.2%: opt-in)
    int fuse = 3;         // CTA-level fused descents: X<n> and the first ops of up to FUSE-1 split
                          // descendants as one op (FUSE=2: pairs, FUSE=0/1: none)
};

// Distinct small-subtree patterns emitted once as __noinline__ device functions, so that the
// unrolled code of a large code stays small enough for the instruction caches: at (32768,29492)
// the 120 size-32 split subtrees have 28 distinct frozen patterns.
// Trace marks (POLAR_TRACE builds): PTRACE(k) records clock64() after op k of the latency
// variant's critical path; labels[k] names it (written to gen/trace_<code>.txt).
struct TraceMarks {
    std::vector<std::string> labels;
    std::string mark(const std::string& label) {
        labels.push_back(label);
        return "PTRACE(" + std::to_string(labels.size() - 1) + ");";
    }
};
TraceMarks* g_marks = nullptr;
int g_ll = 0;  // lane-local threshold of the code being emitted
bool g_repspc = true;  // speculative RepSPC for the code being emitted

struct SharedFns {
    const std::vector<uint8_t>& mask;
    std::set<int> sizes;                 // node sizes that are deduplicated
    std::map<std::string, std::string> by_key;
    std::ostringstream defs;
};

struct Emitter {
    const Tree& t;
    std::ostringstream& o;
    SharedFns* sh = nullptr;
    bool marks = true;  // emit PTRACE marks (not inside shared noinline functions)
    int next_mask = 0;
    std::string ind = "        ";
    int body_root = -1;  // the node whose shared function body is being emitted
    bool words = true;   // decisions as warp-uniform words (decoder.cuh BW<>), else one 64-bit word per lane

    std::string mask_name() { return "m" + std::to_string(next_mask++); }
    void mk(const std::string& label) {
        if (marks && g_marks) o << ind << g_marks->mark(label) << "\n";
    }

    // Emit the warp-scope decode of node id (size n) at bit offset off relative to the
    // subtree root.  src: the C++ expression of its LLR source.  Returns the name of the
    // uniform mask holding its beta when n <= 32, "" when beta was written into bw.
    std::string shared_fn(int id);
    int ll = g_ll;  // split nodes (and repetition leaves) of size <= ll are decoded lane-locally

    // Lane-local decode of node id whose n values are in register array `arr` (every lane
    // holds all of them); returns the name of its beta mask.
    int lane_blocks = 0;
    std::string lane_pfx;
    std::string lane(int id, const std::string& arr, int depth) {
        const Node& v = t.nodes[id];
        const int n = v.n;
        const std::string N_ = std::to_string(n);
        std::string m;
        switch (v.kind) {
            case Kind::Rate0: return "0u";
            case Kind::Rate1: m = mask_name(); o << ind << "const uint32_t " << m << " = lR1<P, " << N_ << ">(" << arr << ");\n"; return m;
            case Kind::Rep: m = mask_name(); o << ind << "const uint32_t " << m << " = lRep<P, " << N_ << ">(" << arr << ");\n"; return m;
            case Kind::Spc: m = mask_name(); o << ind << "const uint32_t " << m << " = lSPC<P, " << N_ << ">(" << arr << ");\n"; return m;
            case Kind::Split: break;
        }
        const int h = n / 2;
        const std::string H = std::to_string(h);
        const std::string c = lane_pfx + "q" + std::to_string(depth + 1) + "_" + std::to_string(next_mask);
        o << ind << "V " << c << "[" << h << "];\n";
        const Node& l = t.nodes[v.left];
        const Node& r = t.nodes[v.right];
        if (l.kind == Kind::Rate0) {
            o << ind << "lG0R<P, " << N_ << ">(" << arr << ", " << c << ");\n";
            std::string mr = lane(v.right, c, depth + 1);
            m = mask_name();
            o << ind << "const uint32_t " << m << " = " << mr << " | (" << mr << " << " << H << ");\n";
            return m;
        }
        o << ind << "lF<P, " << N_ << ">(" << arr << ", " << c << ");\n";
        std::string ml = lane(v.left, c, depth + 1);
        if (r.kind == Kind::Rate0) return ml;
        o << ind << "lG<P, " << N_ << ">(" << arr << ", " << c << ", " << ml << ");\n";
        std::string mr = lane(v.right, c, depth + 1);
        m = mask_name();
        o << ind << "const uint32_t " << m << " = (" << ml << " ^ " << mr << ") | (" << mr << " << " << H << ");\n";
        return m;
    }

    std::string warp(int id, int off, const std::string& src, const std::string& src_arr = "") {
        const Node& v = t.nodes[id];
        const int n = v.n;
        const int s0 = off / 32;
        const std::string N_ = std::to_string(n), S0 = std::to_string(s0);
        if (!src_arr.empty() && n <= ll && n >= 4 && (v.kind == Kind::Split || v.kind == Kind::Rep)) {
            lane_pfx = "L" + std::to_string(lane_blocks++) + "_";
            const std::string arr = lane_pfx + "q0";
            o << ind << "V " << arr << "[" << n << "];\n";
            o << ind << "lGather<P, " << N_ << ">(" << src_arr << "[0], " << arr << ");\n";
            std::string m = lane(id, arr, 0);
            mk("lane<" + N_ + ">");
            return m;
        }
        if (sh && v.kind == Kind::Split && !src_arr.empty() && sh->sizes.count(n) && id != body_root) {
            const std::string fn = shared_fn(id);
            std::string args;
            for (int j = 0; j < (n >= 32 ? n / 32 : 1); ++j) args += (j ? ", " : "") + src_arr + "[" + std::to_string(j) + "]";
            const std::string m = mask_name();
            o << ind << "const " << (n == 64 ? "uint64_t " : "uint32_t ") << m << " = " << fn << "<P>(" << args << ");\n";
            mk("shared<" + N_ + ">");
            if (n <= 32) return m;
            if (n != 64 || !words) {
                std::cerr << "codegen: shared subtree functions above 32 values need decision words and size 64\n";
                std::exit(3);
            }
            o << ind << "wSetWords64<" << s0 << ">(bw, " << m << ");\n";
            return "";
        }
        switch (v.kind) {
            case Kind::Rate0:
                return n <= 32 ? "0u" : "";
            case Kind::Rate1:
                if (n <= 32) {
                    std::string m = mask_name();
                    o << ind << "const uint32_t " << m << " = wR1m<P, " << N_ << ">(" << src << ");\n";
                    mk("Info<" + N_ + ">");
                    return m;
                }
                o << ind << "wR1<P, " << N_ << ", " << S0 << ">(" << src << ", bw);\n";
                mk("Info<" + N_ + ">");
                return "";
            case Kind::Rep:
                if (n <= 32) {
                    std::string m = mask_name();
                    o << ind << "const uint32_t " << m << " = wRepm<P, " << N_ << ">(" << src << ");\n";
                    mk("Repetition<" + N_ + ">");
                    return m;
                }
                o << ind << "wRep<P, " << N_ << ", " << S0 << ">(" << src << ", bw);\n";
                mk("Repetition<" + N_ + ">");
                return "";
            case Kind::Spc:
                if (n <= 32) {
                    std::string m = mask_name();
                    o << ind << "const uint32_t " << m << " = wSPCm<P, " << N_ << ">(" << src << ");\n";
                    mk("SPC<" + N_ + ">");
                    return m;
                }
                o << ind << "wSPC<P, " << N_ << ", " << S0 << ">(" << src << ", bw);\n";
                mk("SPC<" + N_ + ">");
                return "";
            case Kind::Split:
                break;
        }
        const int h = n / 2;
        const std::string H = std::to_string(h);
        const std::string child = "r" + std::to_string(ilog2(h));
        const std::string csrc = "RegSrc<P>{" + child + "}";
        // children read the register stage `child`
        const Node& l = t.nodes[v.left];
        const Node& r = t.nodes[v.right];
        if (g_repspc && n >= 4 && n <= 32 && l.kind == Kind::Rep && r.kind == Kind::Spc) {
            std::string m = mask_name();  // speculative RepSPC, one fused op
            o << ind << "const uint32_t " << m << " = wRepSPCm<P, " << N_ << ">(" << src << ");\n";
            mk("RepSPC<" + N_ + ">");
            return m;
        }
        if (l.kind == Kind::Rate0) {
            o << ind << "wG0R<P, " << N_ << ">(" << src << ", " << child << ");\n";
            mk("G_0R<" + N_ + ">");
            std::string mr = warp(v.right, off + h, csrc, child);
            if (n <= 32) {
                std::string m = mask_name();
                o << ind << "const uint32_t " << m << " = " << mr << " | (" << mr << " << " << H << ");\n";
                return m;
            }
            if (h == 32 && mr != "0u") o << ind << "wDeposit<" << (off + h) / 32 << ">(bw, " << mr << ");\n";
            o << ind << "wComb0R<" << N_ << ", " << S0 << ">(bw);\n";
            return "";
        }
        o << ind << "wF<P, " << N_ << ">(" << src << ", " << child << ");\n";
        mk("F<" + N_ + ">");
        std::string ml = warp(v.left, off, csrc, child);
        if (h == 32 && ml != "0u") o << ind << "wDeposit<" << s0 << ">(bw, " << ml << ");\n";
        if (r.kind == Kind::Rate0) return n <= 32 ? ml : "";
        if (n <= 32 && l.kind == Kind::Rep)  // the left mask is all ones or zero: uniform sign
            o << ind << "wGu<P, " << N_ << ">(" << src << ", " << child << ", " << ml << ");\n";
        else
            o << ind << "wG<P, " << N_ << ", " << S0 << ">(" << src << ", " << child << ", bw, "
              << (n <= 32 ? ml : std::string("0u")) << ");\n";
        mk("G<" + N_ + ">");
        std::string mr = warp(v.right, off + h, csrc, child);
        if (n <= 32) {
            std::string m = mask_name();
            o << ind << "const uint32_t " << m << " = (" << ml << " ^ " << mr << ") | (" << mr << " << " << H
              << ");\n";
            return m;
        }
        if (h == 32 && mr != "0u") o << ind << "wDeposit<" << (off + h) / 32 << ">(bw, " << mr << ");\n";
        o << ind << "wComb<" << N_ << ", " << S0 << ">(bw);\n";
        return "";
    }
};

// Emit (once per distinct frozen pattern) a __noinline__ function decoding the split node id
// from its stage values passed in registers; it returns the node's beta: the warp-uniform
// mask for n <= 32, else the lane's n/32 slot bits.
std::string Emitter::shared_fn(int id) {
    const Node& v = t.nodes[id];
    const int n = v.n;
    std::string key = std::to_string(n) + ":";
    for (int i = v.off; i < v.off + n; ++i) key += sh->mask[i] ? '1' : '0';
    auto it = sh->by_key.find(key);
    if (it != sh->by_key.end()) return it->second;
    const std::string fn = "sf" + std::to_string(n) + "_" + std::to_string(sh->by_key.size());
    std::ostringstream body;
    Emitter e{t, body, sh};
    e.body_root = id;
    e.marks = false;
    const int S = n >= 32 ? n / 32 : 1;
    for (int k = ilog2(n) - 1; k >= 0; --k)
        body << "    V r" << k << "[" << ((1 << k) >= 32 ? (1 << k) / 32 : 1) << "];\n";
    body << "    BW<" << std::max(1, n / 32) << "> bw{};\n    (void)bw;\n";
    e.ind = "    ";
    std::string m = e.warp(id, 0, "RegSrc<P>{in}", "in");
    // the name is reserved only after the body: nested patterns get their definitions first
    sh->by_key[key] = fn;
    sh->defs << "template <class P>\n__device__ __noinline__ " << (n == 64 ? "uint64_t " : "uint32_t ") << fn << "(";
    for (int j = 0; j < S; ++j) sh->defs << (j ? ", " : "") << "typename P::v_t a" << j;
    sh->defs << ") {\n    using V = typename P::v_t;\n    V in[" << S << "] = {";
    for (int j = 0; j < S; ++j) sh->defs << (j ? ", " : "") << "a" << j;
    sh->defs << "};\n" << body.str() << "    return "
             << (n <= 32 ? m : std::string("(uint64_t)bw.w[0] | ((uint64_t)bw.w[1] << 32)")) << ";\n}\n\n";
    return fn;
}

// A warp subtree function: root node id, whose input LLRs are at `src` (shared memory).
// comb: the subtree is the right child of a CTA-level node whose Combine it performs at its end
// (1: Combine, left words ^= right words; 2: Combine_0R, left words = right words) -- the CTA op
// and its barrier disappear (decoder.cuh wStoreBetaComb)
void emit_warp_sub(std::ostringstream& o, const Tree& t, int id, const std::string& fname, SharedFns* sh,
                   bool chan = false, bool noinline = false, int comb = 0) {
    const Node& v = t.nodes[id];
    const int R = v.n;
    o << "    template <class P, class SrcT>\n"
      << "    static " << (noinline ? "__device__ __noinline__" : "PD_INLINE") << " void " << fname
      << "(const SrcT* src_ptr, uint32_t* beta) {\n"
      << "        using V = typename P::v_t;\n"
      << "        const MemSrc<P, SrcT, " << (chan ? "true" : "false") << "> src{src_ptr};\n";
    for (int k = ilog2(R) - 1; k >= 0; --k) {
        const int size = 1 << k;
        o << "        V r" << k << "[" << (size >= 32 ? size / 32 : 1) << "];\n";
    }
    // decisions as warp-uniform words up to 512 values (16 registers), else one 64-bit word per lane
    const bool words = R <= 512;
    if (words) o << "        BW<" << std::max(1, R / 32) << "> bw{};\n        (void)bw;\n";
    else o << "        uint64_t bw = 0;\n        (void)bw;\n";
    Emitter e{t, o, sh};
    e.words = words;
    std::string m = e.warp(id, 0, "src");
    if (R >= 64 && comb && words) {
        o << "        wStoreBetaComb<" << R << ", " << (comb == 2 ? "true" : "false") << ">(bw, beta + " << v.off / 32
          << ", beta + " << (v.off - R) / 32 << ");\n";
        if (g_marks) o << "        " << g_marks->mark("StoreBetaComb<" + std::to_string(R) + ">") << "\n";
    } else if (R >= 64) {
        o << "        wStoreBeta<" << R << ">(bw, beta + " << v.off / 32 << ");\n";
        if (g_marks) o << "        " << g_marks->mark("StoreBeta<" + std::to_string(R) + ">") << "\n";
    } else {
        // R <= 32 only when the whole frame is this subtree (N <= 32): word 0.
        o << "        if (lane_id() == 0) beta[" << v.off / 32 << "] = " << m << ";\n";
    }
    o << "    }\n";
}

struct CtaEmitter {
    const Tree& t;
    std::ostringstream& body;   // decode_cta body
    std::ostringstream& subs;   // warp subtree functions
    int W, T, N;
    std::map<int, int> stage_off;  // stage size -> element offset, all stages in shared memory
    std::map<int, int> soff, goff;  // split layout (GTOP): shared-memory part, global part
    int n_subs = 0;
    SharedFns* sh = nullptr;

    // GTOP (template flag of decode): the largest stages live in per-frame global scratch.
    // The stage of size W (the register subtrees' input) is kept as f32 in `wst` (WF32).
    // H16 (template flag; int8 throughput variant, spec option H16=): stages of size <= h16
    // are f16 values (the f16x2 stage ops then load and store them without conversion), laid
    // out by byte offsets hoff (global or shared).  Statements name a stage by the placeholder
    // @S<m>@ and its state space by @P<m>@; emit_raw writes one copy per layout.
    int h16 = 0;
    std::map<int, int> hoff;  // H16 layout: stage size -> byte offset (in gst or stages)
    std::string stage(int m) { return "@S" + std::to_string(m) + "@"; }
    std::string stage_s(int m) {  // default layout (element offsets of P::st_t)
        if (goff.count(m)) return "(GTOP ? gst + " + std::to_string(goff.at(m)) + " : stages + " + std::to_string(stage_off.at(m)) + ")";
        if (soff.count(m)) return "(stages + (GTOP ? " + std::to_string(soff.at(m)) + " : " + std::to_string(stage_off.at(m)) + "))";
        return "(stages + " + std::to_string(stage_off.at(m)) + ")";
    }
    std::string stage_h(int m) {
        const std::string ty = m <= h16 ? "__half" : "typename P::st_t";
        return "((" + ty + "*)((unsigned char*)" + (goff.count(m) ? "gst" : "stages") + " + " + std::to_string(hoff.at(m)) + "))";
    }

    // Emit one statement; stage placeholders (stage(), space()) are resolved per layout by emit_raw.
    // in the stage arrays.
    std::string last_op;
    // Warp-0 regions (latency variant, XW): a CTA-level node of size <= XW is decoded by warp 0
    // alone -- stage loops with 32 threads, __syncwarp instead of CTA barriers -- and the other
    // warps wait at one barrier after the region.  In the throughput variant (T = 32) the
    // rewrite is the identity.
    int XW = 0;
    bool in_region = false;
    static std::string region(std::string x) {
        for (size_t q; (q = x.find("<P, T, ")) != std::string::npos;) x.replace(q, 7, "<P, 32, ");
        for (size_t q; (q = x.find("<T, ")) != std::string::npos;) x.replace(q, 4, "<32, ");
        if (x == "sync();" || x == "sync.comb();" || x == "sync.sub();") x = "__syncwarp();";
        return x;
    }
    void emit(const std::string& stmt0) {
        const std::string stmt = in_region ? region(stmt0) : stmt0;
        if ((stmt == "sync();" || stmt == "sync.comb();" || stmt == "sync.sub();" || stmt == "__syncwarp();") && g_marks) {
            emit_raw(stmt);
            std::string lab = last_op.rfind("if (gtid", 0) == 0 ? std::string("subtree") : last_op.substr(0, last_op.find('('));
            emit_raw(g_marks->mark("cta:" + lab));
            return;
        }
        if (stmt.rfind("sync.", 0) != 0) last_op = stmt;
        emit_raw(stmt);
    }
    void emit_raw(const std::string& stmt) {
        if (stmt.find('@') == std::string::npos) {
            body << "        " << stmt << "\n";
            return;
        }
        // layout: 0 latency (WF32: the W stage is the f32 `wst`), 1 H16, 2 default
        auto subst = [&](int layout) {
            std::string r = stmt;
            for (size_t q; (q = r.find('@')) != std::string::npos;) {
                const size_t e = r.find('@', q + 1);
                const char kind = r[q + 1];
                const int m = std::atoi(r.substr(q + 2, e - q - 2).c_str());
                std::string by;
                if (kind == 'S') by = layout == 0 && m == W ? "wst" : layout == 1 ? stage_h(m) : stage_s(m);
                else by = layout == 1 ? (goff.count(m) ? "0" : "1") : (goff.count(m) ? "(GTOP ? 0 : 1)" : "1");
                r.replace(q, e - q + 1, by);
            }
            return r;
        };
        body << "        if constexpr (WF32) { " << subst(0) << " }";
        if (h16 > 0) body << " else if constexpr (H16) { " << subst(1) << " }";
        body << " else { " << subst(2) << " }\n";
    }

    // The warp subtree is emitted twice when small subtrees are shared (DEDUP): with the
    // shared noinline functions for the throughput variant (smaller code, measured +11% at
    // N = 32768) and fully inlined for the latency variant (the calls cost ~6 us of batch-1
    // latency), profiles/r1_history.md.
    SharedFns* sh_lat = nullptr;
    bool helper = false;                  // HELPER: instruction run-ahead warp (latency variant)
    bool latni = false;                   // latency-copy subtrees non-inlined
    std::vector<std::string> lat_subs;    // latency-copy subtree functions, in call order
    int comb_req = 0, comb_req_id = -1;   // a Combine the next subtree call (node comb_req_id) performs
    bool comb_done = false;
    void sub_call(int id, const std::string& src) {
        std::string fname = "sub" + std::to_string(n_subs++);
        const int comb = (comb_req && comb_req_id == id) ? comb_req : 0;
        if (comb) comb_done = true;
        if ((sh && !sh->sizes.empty() && sh_lat) || helper || latni) {
            TraceMarks* keep = g_marks;
            g_marks = nullptr;  // trace marks only in the latency copy
            emit_warp_sub(subs, t, id, fname + "_tp", sh, false, false, comb);
            g_marks = keep;
            emit_warp_sub(subs, t, id, fname + "_lat", sh_lat ? sh_lat : sh, false, helper || latni, comb);
            lat_subs.push_back(fname + "_lat");
            emit("if constexpr (T == 32) { " + fname + "_tp<P>(" + src + ", beta); } else { if (w0) " +
                 fname + "_lat<P>(" + src + ", beta); }");
        } else {
            emit_warp_sub(subs, t, id, fname, sh, false, false, comb);
            emit("if (w0) " + fname + "<P>(" + src + ", beta);");
        }
        emit("sync.sub();");
    }

    // State space (SP_GLOBAL 0 / SP_SHARED 1) of a stage, as a placeholder (see stage()).
    std::string space(int m) { return "@P" + std::to_string(m) + "@"; }

    void child(int id, const std::string& src, int done = 0) {
        const Node& v = t.nodes[id];
        if (v.kind == Kind::Rate0) return;  // beta zeroed at frame start
        if (v.n > W && v.n <= XW && !in_region) {
            emit_raw("if (w0) {  // warp-0 region");
            in_region = true;
            cta(id, src);
            in_region = false;
            emit_raw("}");
            emit("sync();");
            return;
        }
        if (v.n > W) cta(id, src, done);
        else sub_call(id, src);
    }

    // Fused descents (decoder.cuh cXY): X<n> of a node and the first op of its child c (F, or
    // G_0R when c's left child is Rate-0) as one op, when c is a CTA-level split node outside a
    // warp-0 region.  Returns the child's first-op kind (OP_F 0, OP_G0R 2) or -1.
    bool fuse = false;
    int fuse_depth = 3;  // FUSE=2: pairs only
    bool fuse_comb = false;  // FCOMB=1 (spec option): subtree right children perform their parent's Combine
    int fuse_kind(int cid) {
        if (!fuse) return -1;
        const Node& c = t.nodes[cid];
        if (c.kind != Kind::Split || c.n <= W || (c.n <= XW && !in_region)) return -1;
        return t.nodes[c.left].kind == Kind::Rate0 ? 2 : 0;
    }
    // X<n> of node id (XK: 0 F, 1 G, 2 G_0R) from src into D, then the child cid (fused when
    // fuse_kind allows)
    void xop_child(int id, int XK, const std::string& src, const std::string& D, const std::string& B, int cid) {
        const Node& v = t.nodes[id];
        const int n = v.n, h = n / 2;
        const std::string N_ = std::to_string(n);
        const std::string SS = src == "chan" ? "CHS" : space(n);
        const std::string CL = src == "chan" ? "true" : "false";  // int8 channel: clamp -128
        const int YK = fuse_kind(cid);
        if (YK < 0) {
            if (XK == 0) emit("cF<P, T, " + N_ + ", " + CL + ", " + SS + ", " + space(h) + ", NI>(" + src + ", " + D + ");");
            else if (XK == 1)
                emit("cG<P, T, " + N_ + ", " + CL + ", false, " + SS + ", " + space(h) + ", NI>(" + src + ", " + D + ", " + B + ");");
            else emit("cG0R<P, T, " + N_ + ", " + CL + ", " + SS + ", " + space(h) + ", NI>(" + src + ", " + D + ");");
            emit("sync();");
            emit("PD_DUMPS(" + D + ", " + std::to_string(h) + ");");
            if (id == 0 && XK != 0) emit("sync.root_g_done();");
            child(cid, D);
            return;
        }
        const std::string D2 = stage(h / 2);
        const std::string BB = XK == 1 ? B : std::string("beta");
        const Node& c = t.nodes[cid];
        const int gcid = YK == 0 ? c.left : c.right;
        const int ZK = fuse_depth >= 3 ? fuse_kind(gcid) : -1;
        if (ZK >= 0) {
            const std::string D3 = stage(h / 4);
            emit("cXYZ<P, T, " + N_ + ", " + CL + ", " + std::to_string(XK) + ", " + std::to_string(YK) + ", " +
                 std::to_string(ZK) + ", " + SS + ", " + space(h) + ", " + space(h / 2) + ", " + space(h / 4) + ", NI>(" + src +
                 ", " + D + ", " + D2 + ", " + D3 + ", " + BB + ");");
            emit("sync();");
            emit("PD_DUMPS(" + D + ", " + std::to_string(h) + ");");
            emit("PD_DUMPS(" + D2 + ", " + std::to_string(h / 2) + ");");
            emit("PD_DUMPS(" + D3 + ", " + std::to_string(h / 4) + ");");
            if (id == 0 && XK != 0) emit("sync.root_g_done();");
            child(cid, D, 2);
            return;
        }
        emit("cXY<P, T, " + N_ + ", " + CL + ", " + std::to_string(XK) + ", " + std::to_string(YK) + ", " + SS + ", " +
             space(h) + ", " + space(h / 2) + ", NI>(" + src + ", " + D + ", " + D2 + ", " + BB + ");");
        emit("sync();");
        emit("PD_DUMPS(" + D + ", " + std::to_string(h) + ");");
        emit("PD_DUMPS(" + D2 + ", " + std::to_string(h / 2) + ");");
        if (id == 0 && XK != 0) emit("sync.root_g_done();");
        child(cid, D, 1);
    }

    void cta(int id, const std::string& src, int done = 0) {
        const std::string SS = src == "chan" ? "CHS" : space(t.nodes[id].n);
        const Node& v = t.nodes[id];
        const int n = v.n;
        const std::string N_ = std::to_string(n);
        const std::string B = "(beta + " + std::to_string(v.off / 32) + ")";
        const std::string CL = src == "chan" ? "true" : "false";  // int8 channel: clamp -128
        switch (v.kind) {
            case Kind::Rate0:
                return;
            case Kind::Rate1:
                emit("cR1<P, T, " + N_ + ">(" + src + ", " + B + ");");
                emit("sync();");
                return;
            case Kind::Rep:
                emit("cRep<P, T, " + N_ + ">(" + src + ", " + stage(n / 2) + ", " + B + ");");
                emit("sync();");
                return;
            case Kind::Spc:
                emit("cSPC<P, T, " + N_ + ">(" + src + ", " + B + ");");
                emit("sync();");
                return;
            case Kind::Split:
                break;
        }
        const int h = n / 2;
        const std::string D = stage(h);
        const Node& l = t.nodes[v.left];
        const Node& r = t.nodes[v.right];
        // done > 0: this node's first op (G_0R or F) ran fused into an ancestor's op, and so did the
        // first ops of done - 1 further nodes down its first-child chain
        // HELPER: one arrive per subtree call, just before the stage op that produces its input
        // a right child that is a warp subtree performs this node's Combine itself (fuse_comb)
        auto want_comb = [&](int kind) {
            comb_req = (fuse_comb && r.kind != Kind::Rate0 && r.n <= W && h >= 64 && h <= 512) ? kind : 0;
            comb_req_id = v.right;
            comb_done = false;
        };
        auto comb_tail = [&](const std::string& op) {
            const bool fused = comb_req && comb_done;
            comb_req = 0;
            comb_req_id = -1;
            comb_done = false;
            if (fused) return;
            emit(op + "<T, " + N_ + ">(" + B + ");");
            emit("sync.comb();");
        };
        if (l.kind == Kind::Rate0) {
            want_comb(2);
            if (done > 0) {
                child(v.right, D, done - 1);
            } else {
                if (helper && h == W && r.kind != Kind::Rate0) emit("if (gtid<T>() < 32) sync.helper_arrive();");
                xop_child(id, 2, src, D, B, v.right);
            }
            comb_tail("cComb0R");
            return;
        }
        if (done > 0) {
            child(v.left, D, done - 1);
        } else {
            if (helper && h == W) emit("if (gtid<T>() < 32) sync.helper_arrive();");
            xop_child(id, 0, src, D, B, v.left);
        }
        if (r.kind == Kind::Rate0) return;
        if (helper && h == W) emit("if (gtid<T>() < 32) sync.helper_arrive();");
        want_comb(1);
        xop_child(id, 1, src, D, B, v.right);
        comb_tail("cComb");
    }
};

// Frame-interleaved decoder (xframe.cuh): the same Fast-SSC traversal, emitted as per-lane
// code, one frame per lane.  Nodes of N_v >= 64 are stage ops on interleaved int8 stages
// (shared memory, or the warp's global scratch slot for the largest ones); a node of N_v = 64
// feeds its two 32-value children straight into f32 registers, where the subtree runs as
// compile-time-indexed scalar code (lF/lG/lR1/lRep/lSPC of decoder.cuh).
struct XEmitter {
    const Tree& t;
    std::ostringstream& o;
    std::map<int, std::pair<std::string, int>> stage;  // child size -> (space, byte offset per warp)
    int nm = 0;
    std::string ind = "        ";

    std::string fresh(const char* p) { return std::string(p) + std::to_string(nm++); }
    const std::vector<uint8_t>* mask = nullptr;
    std::map<std::string, std::string>* fns = nullptr;  // frozen pattern of a 64-node -> function
    std::ostringstream* defs = nullptr;

    // A split 64-node whose two 32-value children run in registers, as a __noinline__ function
    // of its parent pointer and beta words (one per distinct frozen pattern: less code to fetch
    // and to compile).
    std::string pair_fn(int id) {
        const Node& v = t.nodes[id];
        std::string key;
        for (int i = v.off; i < v.off + v.n; ++i) key += (*mask)[i] ? '1' : '0';
        auto it = fns->find(key);
        if (it != fns->end()) return it->second;
        const std::string fn = "xp" + std::to_string(fns->size());
        (*fns)[key] = fn;
        std::ostringstream body;
        XEmitter e{t, body};
        e.ind = "    ";
        const Node& l = t.nodes[v.left];
        const Node& r = t.nodes[v.right];
        body << "    float q[32];\n";
        if (l.kind == Kind::Rate0) {
            body << "    xf::rG0R<S>(p, q);\n";
            const std::string mr = e.reg(v.right, "q");
            body << "    bp[0] = " << mr << ";\n    bp[32] = " << mr << ";\n";
        } else {
            body << "    xf::rF<S>(p, q);\n";
            const std::string ml = e.reg(v.left, "q");
            if (r.kind == Kind::Rate0) {
                body << "    bp[0] = " << ml << ";\n    bp[32] = 0u;\n";
            } else {
                body << "    xf::rG<S>(p, q, " << ml << ");\n";
                const std::string mr = e.reg(v.right, "q");
                body << "    bp[0] = " << ml << " ^ " << mr << ";\n    bp[32] = " << mr << ";\n";
            }
        }
        *defs << "template <int S>\n__device__ __noinline__ void " << fn << "(const int8_t* p, uint32_t* bp) {\n"
              << body.str() << "}\n\n";
        return fn;
    }

    // Register node (n <= 32) whose values are in array `arr`; returns its beta mask name.
    std::string reg(int id, const std::string& arr) {
        const Node& v = t.nodes[id];
        const int n = v.n;
        const std::string N_ = std::to_string(n);
        std::string m;
        switch (v.kind) {
            case Kind::Rate0: return "0u";
            case Kind::Rate1: m = fresh("m"); o << ind << "const uint32_t " << m << " = lR1<PI8, " << N_ << ">(" << arr << ");\n"; return m;
            case Kind::Rep: m = fresh("m"); o << ind << "const uint32_t " << m << " = lRep<PI8, " << N_ << ">(" << arr << ");\n"; return m;
            case Kind::Spc: m = fresh("m"); o << ind << "const uint32_t " << m << " = lSPC<PI8, " << N_ << ">(" << arr << ");\n"; return m;
            case Kind::Split: break;
        }
        const int h = n / 2;
        const std::string H = std::to_string(h);
        const std::string c = fresh("q");
        o << ind << "float " << c << "[" << h << "];\n";
        const Node& l = t.nodes[v.left];
        const Node& r = t.nodes[v.right];
        if (l.kind == Kind::Rate0) {
            o << ind << "lG0R<PI8, " << N_ << ">(" << arr << ", " << c << ");\n";
            const std::string mr = reg(v.right, c);
            m = fresh("m");
            o << ind << "const uint32_t " << m << " = " << mr << " | (" << mr << " << " << H << ");\n";
            return m;
        }
        o << ind << "lF<PI8, " << N_ << ">(" << arr << ", " << c << ");\n";
        const std::string ml = reg(v.left, c);
        if (r.kind == Kind::Rate0) return ml;
        o << ind << "lG<PI8, " << N_ << ">(" << arr << ", " << c << ", " << ml << ");\n";
        const std::string mr = reg(v.right, c);
        m = fresh("m");
        o << ind << "const uint32_t " << m << " = (" << ml << " ^ " << mr << ") | (" << mr << " << " << H << ");\n";
        return m;
    }

    // Memory node (n >= 64) whose values are the stage `S` at byte offset SO ("CH": channel).
    void mem(int id, const std::string& S, int SO) {
        const Node& v = t.nodes[id];
        const int n = v.n, b = v.off;
        const std::string N_ = std::to_string(n), B = std::to_string(b);
        const std::string src = S + ", " + std::to_string(SO);
        switch (v.kind) {
            case Kind::Rate0: return;
            case Kind::Rate1: o << ind << "xf::lvR1<" << N_ << ", " << src << ">(x, " << B << ");\n"; return;
            case Kind::Rep: o << ind << "xf::lvRep<" << N_ << ", " << src << ">(x, " << B << ");\n"; return;
            case Kind::Spc: o << ind << "xf::lvSPC<" << N_ << ", " << src << ">(x, " << B << ");\n"; return;
            case Kind::Split: break;
        }
        const int h = n / 2;
        const Node& l = t.nodes[v.left];
        const Node& r = t.nodes[v.right];
        if (h == 32) {  // both children in registers: one shared function per frozen pattern
            const std::string fn = pair_fn(id);
            o << ind << "xfn::" << fn << "<" << S << ">(xf::cptr<" << src << ">(x, 0), xf::bword(x, " << b / 32 << "));\n";
            return;
        }
        const auto& d = stage.at(h);
        const std::string dst = d.first + ", " + std::to_string(d.second);
        const std::string targs = N_ + ", " + src + ", " + dst;
        if (l.kind == Kind::Rate0) {
            o << ind << "xf::sG0R<" << targs << ">(x);\n";
            mem(v.right, d.first, d.second);
            o << ind << "xf::bComb0R<" << N_ << ">(x, " << B << ");\n";
            return;
        }
        o << ind << "xf::sF<" << targs << ">(x);\n";
        mem(v.left, d.first, d.second);
        if (r.kind == Kind::Rate0) {
            o << ind << "xf::bZero<" << h / 32 << ">(x, " << (b + h) / 32 << ");\n";
            return;
        }
        o << ind << "xf::sG<" << targs << ">(x, " << B << ");\n";
        mem(v.right, d.first, d.second);
        o << ind << "xf::bComb<" << N_ << ">(x, " << B << ");\n";
    }
};

// Emit struct XCode (frame-interleaved int8 decoder).  Stages of size >= xg live in the
// warp's global scratch slot (L2), smaller ones in shared memory; beta in shared memory when
// its 4N bytes per warp fit under the budget, else in the global slot.
void emit_xcode(std::ostringstream& o, const Tree& t, const Spec& sp, int xg, bool beta_gl) {
    XEmitter e{t, o};
    int sacc = 0, gacc = 0;
    for (int m = sp.N / 2; m >= 64; m /= 2) {
        if (m >= xg) {
            e.stage[m] = {"xf::GL", gacc};
            gacc += 32 * m;
        } else {
            e.stage[m] = {"xf::SM", sacc};
            sacc += 32 * m;
        }
    }
    const int beta = 4 * 32 * std::max(1, sp.N / 32);
    std::ostringstream body, defs;
    std::map<std::string, std::string> fns;
    XEmitter eb{t, body};
    eb.stage = e.stage;
    eb.mask = &sp.mask;
    eb.fns = &fns;
    eb.defs = &defs;
    if (sp.N <= 32) {
        body << "        float q[" << sp.N << "];\n        xf::rChan<" << sp.N << ">(x, q);\n";
        const std::string m = eb.reg(0, "q");
        body << "        xf::stB(x, 0, " << m << ");\n";
    } else {
        eb.mem(0, "xf::CH", 0);
    }
    o << "namespace xfn {\nusing namespace pd;\n" << defs.str() << "}  // namespace xfn\n\n";
    o << "struct XCode {\n"
      << "    static constexpr int N = " << sp.N << ";\n"
      << "    static constexpr int K = " << sp.K << ";\n"
      << "    static constexpr int SSTAGE = " << sacc << ";  // shared stage bytes per warp\n"
      << "    static constexpr int GSTAGE = " << gacc << ";  // global stage bytes per warp slot\n"
      << "    static constexpr bool BETA_GL = " << (beta_gl ? "true" : "false") << ";\n"
      << "    static constexpr int SMEM_WARP = SSTAGE + (BETA_GL ? 0 : " << beta << ");\n"
      << "    static constexpr int GSLOT = GSTAGE + (BETA_GL ? " << beta << " : 0);\n"
      << "    static PD_INLINE void decode(const xf::Ctx& x) {\n"
      << body.str() << "    }\n};\n\n";
}

std::string mask_string(const std::vector<uint8_t>& m) {
    std::string s;
    for (uint8_t b : m) s += b ? '1' : '0';
    return s;
}

// jit != nullptr: run-time specialisation -- the source and the variants go to *jit, no files.
void emit_code(const Spec& sp, const std::string& outdir, std::ostringstream& reg_decl,
               std::ostringstream& reg_entries, JitCode* jit = nullptr) {
    Tree t = build_tree(sp.N, sp.mask.data(), sp.nodes);
    std::vector<std::string> ops = schedule(t);
    const int W = std::min(sp.N, sp.W);
    const bool cta_phase = sp.N > W;
    SharedFns sh{sp.mask, sp.dedup, {}, {}};
    TraceMarks marks;
    g_marks = &marks;
    g_ll = sp.ll;
    g_repspc = sp.repspc;
    marks.mark("start");
    std::ostringstream o;
    // One struct per warp-subtree size: "Code" (throughput variants) and, when WLAT differs,
    // "CodeLat" (latency variants).
    auto emit_struct = [&](const std::string& sname, int Wv) {
    const int W = Wv;
    const bool cta_phase = sp.N > W;
    o << "struct " << sname << " {\n"
      << "    static constexpr int N = " << sp.N << ";\n"
      << "    static constexpr int K = " << sp.K << ";\n"
      << "    static constexpr int W = " << W << ";\n";
    if (!cta_phase) {
        o << "    static constexpr int STAGE_ELEMS = 0;\n    static constexpr int STAGE_ELEMS_SMEM = 0;\n"
          << "    static constexpr int GSTAGE_ELEMS = 0;\n    static constexpr int WST = 0;\n"
          << "    static constexpr int STAGE_BYTES_SMEM_H = 0;\n    static constexpr int GSTAGE_BYTES_H = 0;\n"
          << "    static constexpr bool GBETA = false;\n    static constexpr int HELPER = 0;\n"
          << "    template <class P, class SyncT>\n"
          << "    static PD_INLINE void helper(const float*, uint32_t*, const SyncT&) {}\n";
        emit_warp_sub(o, t, 0, "decode_root", &sh, true);  // reads the channel
        o << "    template <class P, int T, bool GTOP, bool WF32, int CHS, bool H16, class ChanT, class SyncT>\n"
          << "    static PD_INLINE void decode(const ChanT* chan, typename P::st_t*, typename P::st_t*, typename P::v_t*,\n"
          << "                                 uint32_t* beta, const SyncT&) {\n"
          << "        if (gtid<T>() < 32) decode_root<P>(chan, beta);\n    }\n";
    } else {
        std::ostringstream body, subs;
        CtaEmitter ce{t, body, subs, W, sp.T, sp.N, {}, {}, {}, 0, &sh};
        SharedFns sh_none{sp.mask, {}, {}, {}};
        ce.sh_lat = &sh_none;
        ce.XW = sp.xw;
        ce.helper = sp.helper > 0;
        ce.latni = sp.latni;
        ce.fuse = sp.fuse >= 2 && !ce.helper;
        ce.fuse_depth = sp.fuse;
        ce.fuse_comb = sp.fcomb && !ce.helper;
        int acc = 0, sacc = 0, gacc = 0, hs = 0, hg = 0;
        const int gs = sp.gs > 0 ? sp.gs : (sp.N >= 16384 ? sp.N / 4 : sp.N + 1);
        ce.h16 = sp.h16;
        for (int m = sp.N / 2; m >= W; m /= 2) {
            ce.stage_off[m] = acc;
            acc += m;
            const int hb = m * (m <= sp.h16 ? 2 : 1);  // H16 layout bytes (int8 profile)
            if (m >= gs) {
                ce.goff[m] = gacc;
                gacc += m;
                ce.hoff[m] = hg;
                hg += hb;
            } else {
                ce.soff[m] = sacc;
                sacc += m;
                ce.hoff[m] = hs;
                hs += hb;
            }
        }
        ce.cta(0, "chan");
        o << "    static constexpr int STAGE_ELEMS = " << acc << ";\n"
          << "    static constexpr int STAGE_ELEMS_SMEM = " << sacc << ";  // GTOP layout\n"
          << "    static constexpr int GSTAGE_ELEMS = " << gacc << ";\n"
          << "    static constexpr int STAGE_BYTES_SMEM_H = " << hs << ";  // H16 layout (int8 throughput)\n"
          << "    static constexpr int GSTAGE_BYTES_H = " << hg << ";\n"
          << "    static constexpr int WST = " << W << ";  // f32 stage feeding the register subtrees\n"
          << "    static constexpr bool GBETA = " << (sp.gbeta && gacc > 0 ? "true" : "false") << ";\n"
          << "    static constexpr int HELPER = " << (ce.helper ? sp.helper : 0) << ";  // helper warp on scheduler HELPER-1\n";
        o << subs.str();
        // the helper warp's run-ahead sequence: the latency copies of the subtrees, in call order
        o << "    template <class P, class SyncT>\n"
          << "    static PD_INLINE void helper(const float* dsrc, uint32_t* dbeta, const SyncT& sync) {\n";
        if (ce.helper)
            for (auto& f : ce.lat_subs) o << "        sync.helper_wait();\n        " << f << "<P>(dsrc, dbeta);\n";
        o << "    }\n";
        o << "    template <class P, int T, bool GTOP, bool WF32, int CHS, bool H16, class ChanT, class SyncT>\n"
          << "    static PD_INLINE void decode(const ChanT* chan, typename P::st_t* stages, typename P::st_t* gst,\n"
          << "                                 typename P::v_t* wst, uint32_t* beta, const SyncT& sync) {\n"
          << "        constexpr bool NI = T == 32 && N >= 8192;  // shared non-inlined stage ops\n"
          << "        // warp 0 of the group, as a value the compiler knows is warp-uniform (a shuffle from\n"
          << "        // lane 0): the subtree code it guards then needs no WARPSYNC.COLLECTIVE wrappers\n"
          << "        // around its shuffles/votes (threadIdx.x < 32 would, measured in the SASS)\n"
          << "        const bool w0 = T == 32 || __shfl_sync(FULL, threadIdx.x >> 5, 0) == 0;\n"
          << "        (void)w0;\n"
          << "        PTRACE(0);\n"
          << body.str() << "    }\n";
    }
    o << "};\n\n";
    };
    const int WL = std::min(sp.N, sp.wlat > 0 ? sp.wlat : W);
    const bool two = WL != W;
    // WF: the f32 throughput variant may want another subtree size than the int8 one (its
    // stages are 4x larger: (2048,1723) int8 is fastest at W = 512, f32 at W = 2048)
    const int WF = std::min(sp.N, sp.wf > 0 ? sp.wf : W);
    const bool three = WF != W && WF != WL;
    if (two) {
        g_marks = nullptr;  // trace marks belong to the latency variant's code
        emit_struct("Code", W);
        g_marks = &marks;
        emit_struct("CodeLat", WL);
    } else {
        emit_struct("Code", W);
    }
    if (three) {
        TraceMarks* keep = g_marks;
        g_marks = nullptr;
        emit_struct("CodeF", WF);
        g_marks = keep;
    }
    // frame-interleaved variant: the largest stages go to the global slot until the shared
    // stages (and beta, unless it is global too) fit the per-warp budget
    int xg = sp.N;  // stages of size >= xg are global
    const int xbeta = 4 * 32 * std::max(1, sp.N / 32);
    const bool xbeta_gl = xbeta > sp.xsm / 2;
    auto xsmem = [&](int g) {
        int s = xbeta_gl ? 0 : xbeta;
        for (int m = sp.N / 2; m >= 64; m /= 2)
            if (m < g) s += 32 * m;
        return s;
    };
    while (xg > 64 && xsmem(xg) > sp.xsm) xg /= 2;
    emit_xcode(o, t, sp, xg, xbeta_gl);
    o << "}  // namespace code_" << sp.name << "\n}  // namespace pd\n\n";
    {
        std::ostringstream head;
        head << "// Generated by codegen.cpp for code " << sp.name << " (N=" << sp.N << ", K=" << sp.K << ", "
             << ops.size() << " Fast-SSC ops, W=" << W << ", " << sh.by_key.size()
             << " shared subtree functions). Do not edit.\n"
             << "#include \"kernels.cuh\"\n#include \"xframe.cuh\"\n\nnamespace pd {\nnamespace code_" << sp.name << " {\n\n"
             << sh.defs.str();
        const std::string rest = o.str();
        o.str("");
        o << head.str() << rest;
    }
    const std::string C = "pd::code_" + sp.name + "::Code";
    const std::string CL = "pd::code_" + sp.name + (two ? "::CodeLat" : "::Code");
    const std::string CF = "pd::code_" + sp.name + (WF == W ? "::Code" : WF == WL ? "::CodeLat" : "::CodeF");
    const int t_lat = sp.N > WL ? sp.T : 32;
    struct V {
        const char* tag;
        const char* prof;
        int T;
        bool chan_smem;
        int fpc;
        bool gtop;
        int minb;
        bool lat;
        bool h16;
    };
    auto bytes = [&](const char* prof) { return sp.N * (std::string(prof) == "PF32" ? 4 : 1); };
    // Throughput variant: as many lockstep warps (frames) per CTA as the shared memory of one
    // SM holds, at most 16 (same formula as FrameLayout::PER_FRAME).
    auto a16 = [](int x) { return (x + 15) & ~15; };
    // stage element counts of a struct with warp-subtree size Wv (as emit_struct computes them)
    struct SL {
        bool cta;
        int g_elems = 0, h_smem = 0, h_glob = 0;  // global stage elements; H16 layout bytes
    };
    auto layout_of = [&](int Wv) {
        SL l{sp.N > Wv};
        if (l.cta) {
            const int gs = sp.gs > 0 ? sp.gs : (sp.N >= 16384 ? sp.N / 4 : sp.N + 1);
            for (int m = sp.N / 2; m >= Wv; m /= 2) {
                const int hb = m * (m <= sp.h16 ? 2 : 1);
                if (m >= gs) l.g_elems += m, l.h_glob += hb;
                else l.h_smem += hb;
            }
        }
        return l;
    };
    const SL lw = layout_of(W), lf = layout_of(WF);
    const int g_elems = lw.g_elems, h_glob = lw.h_glob;
    const bool h16 = cta_phase && sp.h16 > 0;
    auto fpc = [&](const char* prof, bool chan_smem) {
        const int s = std::string(prof) == "PF32" ? 4 : 1;
        const SL& l = s == 4 ? lf : lw;
        const int Wv = s == 4 ? WF : W;
        const int stages = (h16 && s == 1) ? a16(l.h_smem) : a16(std::max(0, l.cta ? sp.N - Wv - l.g_elems : 0) * s);
        const int outw = a16((sp.K + 31) / 32 * 4);
        const bool gb = sp.gbeta && l.g_elems > 0;
        const int per = (chan_smem ? 2 * a16(sp.N * s) : 0) + stages + (gb ? 0 : a16(std::max(1, sp.N / 32) * 4)) +
                        (stages >= outw ? 0 : outw) + 16;
        return std::max(1, std::min(sp.fpc_max, (220 * 1024) / per));
    };
    const bool cs_f = 2 * bytes("PF32") <= 16384, cs_i = 2 * bytes("PI8") <= 16384;
    const bool gt = g_elems > 0;
    std::vector<V> vars = {
        {"tp_f32", "PF32", 32, cs_f, fpc("PF32", cs_f), lf.g_elems > 0, 1, false, false},
        {"tp_i8", "PI8", 32, cs_i, fpc("PI8", cs_i), gt, sp.cps, false, h16},
        {"lat_f32", "PF32", t_lat, bytes("PF32") <= 32768, 1, false, 1, true, false},
        {"lat_i8", "PI8", t_lat, bytes("PI8") <= 32768, 1, false, 1, true, false},
    };
    // the host-side registry symbols exist only in the build-time (nvcc) compilation
    o << "#ifndef __CUDACC_RTC__\n";
    auto gscratch_of = [&](const V& v) {
        const bool f = std::string(v.prof) == "PF32" && !v.lat;
        return v.gtop ? (v.h16 ? a16(h_glob) : a16((f ? lf.g_elems : g_elems) * (std::string(v.prof) == "PF32" ? 4 : 1))) +
                            (sp.gbeta ? a16(std::max(1, sp.N / 32) * 4) : 0)
                      : 0;
    };
    int vi = 0;
    for (auto& v : vars) {
        const std::string cs = v.lat ? CL : std::string(v.prof) == "PF32" ? CF : C;
        const std::string targs = std::string("pd::") + v.prof + ", " + cs + ", " + std::to_string(v.T) + ", " +
                                  std::to_string(v.fpc) + ", " + (v.chan_smem ? "true" : "false") + ", " +
                                  (v.gtop ? "true" : "false") + ", " + (v.h16 ? "true" : "false");
        const std::string kargs = targs + ", " + std::to_string(v.minb);
        if (jit) {
            jit->vars[vi++] = JitVariant{"&pd::k_frame<" + kargs + ">", "pd::FrameLayout<" + targs + ">::SMEM", (uint32_t)v.T,
                                         (uint32_t)v.fpc, (uint32_t)gscratch_of(v),
                                         (uint32_t)(v.lat && sp.helper && sp.N > WL ? 32 * sp.helper : 0)};
        }
        o << "extern const void* const polar_kern_" << sp.name << "_" << v.tag << " = (const void*)&pd::k_frame<"
          << kargs << ">;\n"
          << "extern const unsigned polar_smem_" << sp.name << "_" << v.tag << " = pd::FrameLayout<" << targs
          << ">::SMEM;\n";
        reg_decl << "extern const void* const polar_kern_" << sp.name << "_" << v.tag << ";\n"
                 << "extern const unsigned polar_smem_" << sp.name << "_" << v.tag << ";\n";
    }
    {
        const std::string XC = "pd::code_" + sp.name + "::XCode";
        const std::string kx = "pd::k_xf<" + XC + ", " + std::to_string(sp.xwpc) + ", 1>";
        o << "extern const void* const polar_kern_" << sp.name << "_xf_i8 = (const void*)&" << kx << ";\n"
          << "extern const unsigned polar_smem_" << sp.name << "_xf_i8 = " << sp.xwpc << " * " << XC << "::SMEM_WARP;\n"
          << "extern const unsigned polar_gslot_" << sp.name << "_xf_i8 = " << XC << "::GSLOT;\n";
        reg_decl << "extern const void* const polar_kern_" << sp.name << "_xf_i8;\n"
                 << "extern const unsigned polar_smem_" << sp.name << "_xf_i8;\n"
                 << "extern const unsigned polar_gslot_" << sp.name << "_xf_i8;\n";
    }
    const bool mbox = sp.mailbox && sp.N >= 64 && sp.N > WL;
    if (mbox) {
        const std::string km = "pd::k_mailbox<pd::PI8, " + CL + ", " + std::to_string(t_lat) + ">";
        o << "extern const void* const polar_kern_" << sp.name << "_mbox_i8 = (const void*)&" << km << ";\n"
          << "extern const unsigned polar_smem_" << sp.name << "_mbox_i8 = pd::FrameLayout<pd::PI8, " << CL << ", "
          << t_lat << ", 1, true, false, false>::SMEM;\n";
        reg_decl << "extern const void* const polar_kern_" << sp.name << "_mbox_i8;\n"
                 << "extern const unsigned polar_smem_" << sp.name << "_mbox_i8;\n";
    }
    o << "#else\n";
    // NVRTC: the shared-memory sizes, read back by polar_api.cu (cudaLibraryGetGlobal)
    if (jit) {
        o << "extern \"C\" __device__ unsigned polar_jit_smem[4] = {";
        for (int i = 0; i < 4; ++i) o << (i ? ", " : "") << jit->vars[i].smem;
        o << "};\n";
    }
    o << "#endif\n";
    std::string sched;
    for (auto& s : ops) sched += s + ";";
    if (jit) {
        jit->source = o.str();
        jit->n_ops = (uint32_t)ops.size();
        jit->warp_root = (uint32_t)W;
        jit->schedule = sched;
        g_marks = nullptr;
        return;
    }
    std::ofstream(outdir + "/code_" + sp.name + ".cu") << o.str();
    {
        std::ofstream tl(outdir + "/trace_" + sp.name + ".txt");
        for (auto& l : marks.labels) tl << l << "\n";
    }
    g_marks = nullptr;

    reg_decl << "static const uint8_t mask_" << sp.name << "[" << sp.N << "] = {";
    for (int i = 0; i < sp.N; ++i) reg_decl << (i ? "," : "") << int(sp.mask[i]);
    reg_decl << "};\n";
    reg_entries << "    {\"" << sp.name << "\", " << sp.N << ", " << sp.K << ", mask_" << sp.name << ", "
                << code_hash(sp.N, sp.K, sp.mask.data()) << "ull, " << ops.size() << ", " << W;
    for (auto& v : vars)
        reg_entries << ", {&polar_kern_" << sp.name << "_" << v.tag << ", &polar_smem_" << sp.name << "_" << v.tag
                    << ", " << v.T << ", " << v.fpc << ", " << gscratch_of(v)
                    << ", " << (v.lat && sp.helper && sp.N > WL ? 32 * sp.helper : 0) << "}";
    reg_entries << ", {&polar_kern_" << sp.name << "_xf_i8, &polar_smem_" << sp.name << "_xf_i8, 32, " << sp.xwpc
                << ", 0, 0}, &polar_gslot_" << sp.name << "_xf_i8";
    if (mbox)
        reg_entries << ", {&polar_kern_" << sp.name << "_mbox_i8, &polar_smem_" << sp.name << "_mbox_i8, " << t_lat
                    << ", 1, 0, 0}";
    else
        reg_entries << ", {nullptr, nullptr, 0, 0, 0, 0}";
    reg_entries << ", \"" << sched << "\"},\n";
}

}  // namespace

namespace {
void parse_options(Spec& sp, std::istream& ls);
}

#ifndef POLAR_CODEGEN_LIB
int main(int argc, char** argv) {
    if (argc != 3) {
        std::cerr << "usage: polar_codegen <spec file> <output dir>\n";
        return 1;
    }
    std::ifstream in(argv[1]);
    if (!in) {
        std::cerr << "codegen: cannot read " << argv[1] << "\n";
        return 1;
    }
    std::vector<Spec> specs;
    std::string line;
    while (std::getline(in, line)) {
        auto hash = line.find('#');
        if (hash != std::string::npos) line = line.substr(0, hash);
        std::istringstream ls(line);
        Spec sp;
        std::string how;
        if (!(ls >> sp.name >> sp.N >> sp.K >> how)) continue;
        if (sp.N < 2 || (sp.N & (sp.N - 1)) || sp.N > 32768 || sp.K < 1 || sp.K > sp.N) {
            std::cerr << "codegen: bad (N, K) for " << sp.name << "\n";
            return 2;
        }
        sp.mask.assign(sp.N, 0);
        if (how == "ga") {
            double ebn0;
            ls >> ebn0;
            construct_ga(sp.N, sp.K, ebn0, sp.mask.data());
        } else if (how == "mask") {
            std::string bits;
            ls >> bits;
            if ((int)bits.size() != sp.N) {
                std::cerr << "codegen: mask length of " << sp.name << "\n";
                return 2;
            }
            int nf = 0;
            for (int i = 0; i < sp.N; ++i) nf += (sp.mask[i] = bits[i] == '1');
            if (nf != sp.N - sp.K) {
                std::cerr << "codegen: mask of " << sp.name << " has " << nf << " frozen bits\n";
                return 2;
            }
        } else {
            std::cerr << "codegen: unknown construction " << how << "\n";
            return 2;
        }
        parse_options(sp, ls);
        specs.push_back(sp);
    }
    std::ostringstream decl, entries;
    for (auto& sp : specs) emit_code(sp, argv[2], decl, entries);
    std::ostringstream reg;
    reg << "// Generated by codegen.cpp. Do not edit.\n#include \"registry.hpp\"\n\n" << decl.str()
        << "\nnamespace polar {\nconst RegistryEntry kRegistry[] = {\n" << entries.str() << "};\n"
        << "const uint32_t kRegistrySize = " << specs.size() << ";\n}  // namespace polar\n";
    std::ofstream(std::string(argv[2]) + "/registry.cpp") << reg.str();
    return 0;
}
#endif  // POLAR_CODEGEN_LIB

namespace {
void parse_options(Spec& sp, std::istream& ls) {
        std::string opt;
        while (ls >> opt) {
            if (opt.rfind("W=", 0) == 0) sp.W = std::atoi(opt.c_str() + 2);
            else if (opt.rfind("T=", 0) == 0) sp.T = std::atoi(opt.c_str() + 2);
            else if (opt.rfind("FPC=", 0) == 0) sp.fpc_max = std::atoi(opt.c_str() + 4);
            else if (opt.rfind("GS=", 0) == 0) sp.gs = std::atoi(opt.c_str() + 3);
            else if (opt.rfind("H16=", 0) == 0) sp.h16 = std::atoi(opt.c_str() + 4);
            else if (opt.rfind("REPSPC=", 0) == 0) sp.repspc = std::atoi(opt.c_str() + 7) != 0;
            else if (opt.rfind("NODES=", 0) == 0) {
                const std::string v = opt.substr(6);
                sp.nodes = v == "sc" ? NodeSet::SC : v == "ssc" ? NodeSet::SSC : v == "nospc" ? NodeSet::NoSPC : NodeSet::FastSSC;
            }
            else if (opt.rfind("LL=", 0) == 0) sp.ll = std::atoi(opt.c_str() + 3);
            else if (opt.rfind("CPS=", 0) == 0) sp.cps = std::atoi(opt.c_str() + 4);
            else if (opt.rfind("WLAT=", 0) == 0) sp.wlat = std::atoi(opt.c_str() + 5);
            else if (opt.rfind("WF=", 0) == 0) sp.wf = std::atoi(opt.c_str() + 3);
            else if (opt.rfind("XW=", 0) == 0) sp.xw = std::atoi(opt.c_str() + 3);
            else if (opt.rfind("HELPER=", 0) == 0) sp.helper = std::atoi(opt.c_str() + 7);
            else if (opt.rfind("LATNI=", 0) == 0) sp.latni = std::atoi(opt.c_str() + 6) != 0;
            else if (opt.rfind("MAILBOX=", 0) == 0) sp.mailbox = std::atoi(opt.c_str() + 8) != 0;
            else if (opt.rfind("XSM=", 0) == 0) sp.xsm = std::atoi(opt.c_str() + 4);
            else if (opt.rfind("XWPC=", 0) == 0) sp.xwpc = std::atoi(opt.c_str() + 5);
            else if (opt.rfind("GBETA=", 0) == 0) sp.gbeta = std::atoi(opt.c_str() + 6) != 0;
            else if (opt.rfind("FUSE=", 0) == 0) sp.fuse = std::atoi(opt.c_str() + 5);
            else if (opt.rfind("FCOMB=", 0) == 0) sp.fcomb = std::atoi(opt.c_str() + 6) != 0;
            else if (opt.rfind("DEDUP=", 0) == 0) {  // comma-separated sizes, or "none"
                sp.dedup.clear();
                std::stringstream ds(opt.substr(6));
                std::string tok;
                while (std::getline(ds, tok, ','))
                    if (tok != "none") sp.dedup.insert(std::atoi(tok.c_str()));
            }
        }
}
}  // namespace

namespace polar {
// Default options by code length: those of the registered codes in codes.txt.
bool codegen_jit(int N, int K, const uint8_t* frozen, JitCode* out, std::string* err) {
    if (N < 2 || (N & (N - 1)) || N > 32768 || K < 1 || K > N) {
        if (err) *err = "bad (N, K)";
        return false;
    }
    Spec sp;
    sp.name = "jit";
    sp.N = N;
    sp.K = K;
    sp.mask.assign(frozen, frozen + N);
    std::istringstream opts(N >= 16384 ? "W=512 FPC=6 CPS=3 DEDUP=32"
                            : N == 8192 ? "W=512 T=512 GS=2048 DEDUP=16,32,64"
                            : N == 4096 ? "W=1024 T=256"
                            : N == 2048 ? "W=256 WF=2048 WLAT=1024 FPC=8 CPS=2"
                                        : "");
    parse_options(sp, opts);
    std::ostringstream decl, entries;
    emit_code(sp, "", decl, entries, out);
    return true;
}
}  // namespace polar
