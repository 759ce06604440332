// tree.hpp -- the Fast-SSC decoder tree of a polar code (host side, product code).
//
// Giard et al., arXiv:1504.00353: SC decoding is a depth-first traversal of the binary tree
// of constituent codes; Fast-SSC stops the traversal at Rate-0 and
// Rate-1 nodes, repetition nodes and single-parity-check nodes
// (P:442-459).  The unrolled decoder is the list of operations met on that traversal
// (Listing 1).  Node priority and the N_v = 2 rule follow reading C14 of
// Rate-0 > Rate-1 > Rep > SPC > split.
//
// Used by the schedule emitter (codegen.cpp, build time) and by polar_code_create (to
// validate the mask and report the op count).  Shares nothing with oracle/.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace polar {

enum class Kind : int { Rate0 = 0, Rate1 = 1, Rep = 2, Spc = 3, Split = 4 };

struct Node {
    Kind kind;
    int n;     // N_v, the node size
    int off;   // index of the node's first bit in the codeword
    int left;  // child indices into Tree::nodes (-1 for leaves)
    int right;
};

struct Tree {
    int N = 0;
    std::vector<Node> nodes;  // nodes[0] is the root
};

// Node sets of the decoder generator (the paper's algorithm ablation, tab:impl:tp:algo-unroll
// P:948-963): Fast-SSC (default: Rate-0, Rate-1, Rep, SPC), the paper's
// GPU set without SPC nodes, SSC (Rate-0 and Rate-1 nodes of any size)
// and plain SC (no node specialisation: the traversal reaches every bit).
enum class NodeSet : int { FastSSC = 0, NoSPC = 1, SSC = 2, SC = 3 };

// Classify the constituent code frozen[off .. off+n): counts of frozen bits decide.
inline Kind classify(const uint8_t* frozen, int off, int n, NodeSet set = NodeSet::FastSSC) {
    int n_frozen = 0;
    for (int i = off; i < off + n; ++i) n_frozen += frozen[i] != 0;
    if (set == NodeSet::SC && n > 1) return Kind::Split;
    if (n_frozen == n) return Kind::Rate0;
    if (n_frozen == 0) return Kind::Rate1;
    if (set == NodeSet::SSC) return Kind::Split;
    if (n_frozen == n - 1 && frozen[off + n - 1] == 0) return Kind::Rep;
    if (set == NodeSet::NoSPC) return Kind::Split;
    if (n_frozen == 1 && frozen[off] != 0) return Kind::Spc;
    return Kind::Split;
}

inline int build_node(Tree& t, const uint8_t* frozen, int off, int n, NodeSet set) {
    int id = (int)t.nodes.size();
    t.nodes.push_back(Node{classify(frozen, off, n, set), n, off, -1, -1});
    if (t.nodes[id].kind == Kind::Split) {
        int l = build_node(t, frozen, off, n / 2, set);
        int r = build_node(t, frozen, off + n / 2, n / 2, set);
        t.nodes[id].left = l;
        t.nodes[id].right = r;
    }
    return id;
}

inline Tree build_tree(int N, const uint8_t* frozen, NodeSet set = NodeSet::FastSSC) {
    Tree t;
    t.N = N;
    build_node(t, frozen, 0, N, set);
    return t;
}

// The unfused op list of the traversal, in Listing 1's vocabulary:
// a split node whose left child is Rate-0 runs G_0R, its right subtree and Combine_0R;
// any other split node runs F and its left subtree, then -- unless its right child is
// Rate-0, where the right half of beta stays 0 (reading C16) -- G, its right subtree and
// Combine.  Leaves emit Info (Rate-1), Repetition or SPC; Rate-0 leaves emit nothing.
inline void schedule_rec(const Tree& t, int id, std::vector<std::string>& ops) {
    const Node& v = t.nodes[id];
    auto op = [&](const char* name) { ops.push_back(std::string(name) + "<" + std::to_string(v.n) + ">"); };
    switch (v.kind) {
        case Kind::Rate0: return;
        case Kind::Rate1: op("Info"); return;
        case Kind::Rep: op("Repetition"); return;
        case Kind::Spc: op("SPC"); return;
        case Kind::Split: break;
    }
    const Node& l = t.nodes[v.left];
    const Node& r = t.nodes[v.right];
    if (l.kind == Kind::Rate0) {
        op("G_0R");
        schedule_rec(t, v.right, ops);
        op("Combine_0R");
        return;
    }
    op("F");
    schedule_rec(t, v.left, ops);
    if (r.kind == Kind::Rate0) {
        op("Combine_R0");
        return;
    }
    op("G");
    schedule_rec(t, v.right, ops);
    op("Combine");
}

inline std::vector<std::string> schedule(const Tree& t) {
    std::vector<std::string> ops;
    schedule_rec(t, 0, ops);
    return ops;
}

// The same traversal as a compact program for the generic (interpreted) decoder, the GPU
// analogue of the paper's instruction-based decoder: one uint32 per
// op = opcode | log2(N_v) << 4 | node offset << 9.  Combine_R0 needs no instruction (the
// right half of beta is already zero).
enum : uint32_t { OP_F = 0, OP_G = 1, OP_G0R = 2, OP_R1 = 3, OP_REP = 4, OP_SPC = 5, OP_COMB = 6, OP_COMB0R = 7 };

inline uint32_t encode_op(uint32_t op, int n, int off) {
    int k = 0;
    while ((1 << k) < n) ++k;
    return op | (uint32_t)k << 4 | (uint32_t)off << 9;
}

inline void program_rec(const Tree& t, int id, std::vector<uint32_t>& p) {
    const Node& v = t.nodes[id];
    switch (v.kind) {
        case Kind::Rate0: return;
        case Kind::Rate1: p.push_back(encode_op(OP_R1, v.n, v.off)); return;
        case Kind::Rep: p.push_back(encode_op(OP_REP, v.n, v.off)); return;
        case Kind::Spc: p.push_back(encode_op(OP_SPC, v.n, v.off)); return;
        case Kind::Split: break;
    }
    const Node& l = t.nodes[v.left];
    const Node& r = t.nodes[v.right];
    if (l.kind == Kind::Rate0) {
        p.push_back(encode_op(OP_G0R, v.n, v.off));
        program_rec(t, v.right, p);
        p.push_back(encode_op(OP_COMB0R, v.n, v.off));
        return;
    }
    p.push_back(encode_op(OP_F, v.n, v.off));
    program_rec(t, v.left, p);
    if (r.kind == Kind::Rate0) return;
    p.push_back(encode_op(OP_G, v.n, v.off));
    program_rec(t, v.right, p);
    p.push_back(encode_op(OP_COMB, v.n, v.off));
}

inline std::vector<uint32_t> program(const Tree& t) {
    std::vector<uint32_t> p;
    program_rec(t, 0, p);
    return p;
}

// Information set closed under bit-superset: i in A implies i | 2^b in A for every b.
// Required by the two-pass systematic encoder (reading C4).
inline bool superset_closed(int N, const uint8_t* frozen) {
    for (int i = 0; i < N; ++i) {
        if (frozen[i]) continue;
        for (int b = 1; b < N; b <<= 1)
            if (!(i & b) && frozen[i | b]) return false;
    }
    return true;
}

// FNV-1a over (N, K, mask bytes): the registry key of a specialised decoder.
inline uint64_t code_hash(int N, int K, const uint8_t* frozen) {
    uint64_t h = 1469598103934665603ull;
    auto mix = [&](uint8_t b) { h ^= b; h *= 1099511628211ull; };
    for (int s = 0; s < 32; s += 8) mix((uint8_t)(N >> s));
    for (int s = 0; s < 32; s += 8) mix((uint8_t)(K >> s));
    for (int i = 0; i < N; ++i) mix(frozen[i] ? 1 : 0);
    return h;
}

}  // namespace polar
