// registry.hpp -- table of the codes whose decoders were specialised at build time.
// Entries are emitted by codegen.cpp into build/gen/registry.cpp; each points at the
// kernels instantiated in build/gen/code_<name>.cu.
#pragma once

#include <cstdint>

namespace polar {

// One compiled kernel: __global__ (const void* llr, long long n, uint32_t* out, const uint32_t* gtab,
// void* gscratch).
// Held through pointers to per-code constants so the table is constant-initialised.
struct Variant {
    const void* const* kern;
    const unsigned* smem;  // dynamic shared memory per CTA
    uint32_t threads;      // threads per frame group
    uint32_t frames;       // frame groups (frames decoded concurrently) per CTA
    uint32_t gscratch;     // bytes of global stage scratch per frame group (0: none)
    uint32_t extra;        // extra threads per CTA (the latency variant's run-ahead helper warp)
};

struct RegistryEntry {
    const char* name;
    uint32_t N, K;
    const uint8_t* mask;   // N bytes, 1 = frozen
    uint64_t hash;         // code_hash(N, K, mask)
    uint32_t n_ops;        // Listing-1 op count of the schedule
    uint32_t warp_root;    // W: size of the subtrees decoded by one warp in registers
    Variant tp_f32, tp_i8;    // throughput: one warp per frame
    Variant lat_f32, lat_i8;  // latency: one CTA of threads per frame
    Variant xf_i8;            // frame-interleaved throughput: one lane per frame (frames = warps per CTA)
    const unsigned* xf_gslot; // its global scratch bytes per warp
    Variant mbox_i8;          // batch-1 mailbox kernel (kern == nullptr: not built for this code)
    const char* schedule;     // ';'-separated Listing-1 op list
};

extern const RegistryEntry kRegistry[];
extern const uint32_t kRegistrySize;

}  // namespace polar
