// registry.hpp -- table of the codes whose decoders were specialised at build time.
// Entries are emitted by codegen.cpp into build/gen/registry.cpp; each points at the
// kernels instantiated in build/gen/code_<name>.cu.
#pragma once

#include <cstdint>

namespace polar {

enum : uint32_t { MODE_WARP = 0, MODE_CTA = 1 };

struct RegistryEntry {
    const char* name;
    uint32_t N, K;
    const uint8_t* mask;   // N bytes, 1 = frozen
    uint64_t hash;         // code_hash(N, K, mask)
    uint32_t n_ops;        // Listing-1 op count of the schedule
    uint32_t mode;         // MODE_WARP: one warp per frame; MODE_CTA: one CTA per frame
    uint32_t warp_root;    // W: size of the subtrees decoded by one warp in registers
    uint32_t threads;      // threads per CTA
    // Addresses of the per-code constants (kept as pointers so the table is constant-
    // initialised): kernel = __global__ (const void*, long long, uint32_t*, const uint16_t*).
    const void* const* kern_f32;
    const void* const* kern_i8;
    const unsigned* smem_f32;  // dynamic shared memory per CTA
    const unsigned* smem_i8;
    uint32_t frames_per_cta;     // WARPS for MODE_WARP, 1 for MODE_CTA
    const char* schedule;        // ';'-separated Listing-1 op list
};

extern const RegistryEntry kRegistry[];
extern const uint32_t kRegistrySize;

}  // namespace polar
