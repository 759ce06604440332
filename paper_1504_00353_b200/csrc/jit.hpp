// jit.hpp -- run-time specialisation of an unregistered code (the paper
// generates its unrolled decoders per code, and its instruction-based decoder covers
// codes without one).  codegen.cpp emits the same source it writes at build time;
// polar_api.cu compiles it with NVRTC for sm_100a, caches the cubin by a hash of the source, and
// binds the kernels like a registry entry.
#pragma once

#include <cstdint>
#include <string>

namespace polar {

struct JitVariant {
    std::string kernel;  // C++ name expression of the k_frame instantiation ("&pd::k_frame<...>")
    std::string smem;    // its dynamic shared memory, a constant expression
    uint32_t threads, frames, gscratch, extra;
};

struct JitCode {
    std::string source;  // the generated translation unit (includes kernels.cuh, xframe.cuh)
    JitVariant vars[4];  // tp_f32, tp_i8, lat_f32, lat_i8 (the registry order)
    uint32_t n_ops = 0, warp_root = 0;
    std::string schedule;
};

// Emit the unrolled decoder of (N, K, frozen mask) with the default build options for its
// length (those of codes.txt).  false + *err on an invalid code.
bool codegen_jit(int N, int K, const uint8_t* frozen, JitCode* out, std::string* err);

// The headers the generated source includes, embedded at build time (build.py).
extern const int kJitHeaderCount;
extern const char* const kJitHeaderNames[];
extern const char* const kJitHeaderText[];

}  // namespace polar
