// mm_common.cuh — device helpers shared by the sm_100a kernels of libmm_b200.
// (Independent of oracle/: nothing here is shared with the CPU oracle.)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mm.h"

namespace mm {

// ---------------------------------------------------------------- MUFU wrappers
// .approx.ftz forms map 1:1 onto MUFU.RCP / MUFU.RSQ / MUFU.LG2 / MUFU.EX2.
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rsqrt_approx(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float lg2_approx(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Softening added to r^2 before the reciprocal (reading Q6): 1e-36 is a
// normal float, so an exactly coincident pair gives 0 * rcp(1e-36) = 0 and
// any pair with r > ~4e-15 is unaffected after rounding.
constexpr float kEps2 = 1e-36f;
// Clamp of the exponent for q > 0 so that ex2 stays finite for coincident
// (masked) pairs: 2^126 < FLT_MAX.
constexpr float kExpClamp = 126.0f;

// |d|^-(q+2) from r2 = |d|^2 (+eps): q = 0 -> rcp(r2); q > 0 -> 2^(c * lg2 r2),
// c = -(q+2)/2, clamped to stay finite.
template <bool QPOW>
__device__ __forceinline__ float inv_pow(float r2, float c) {
    if constexpr (!QPOW) {
        return rcp_approx(r2);
    } else {
        return ex2_approx(fminf(c * lg2_approx(r2), kExpClamp));
    }
}

// ---------------------------------------------------------------- counter RNG (Q18)
// SplitMix64 output function; the CUDA path's own copy (the oracle has its own).
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
constexpr uint64_t kTagInit = 0x494e4954ULL;    // "INIT"
constexpr uint64_t kTagJitter = 0x4a495454ULL;  // "JITT"
constexpr uint64_t kTagMatch = 0x4d415443ULL;   // "MATC"

__device__ __forceinline__ float uniform24(uint64_t key) {
    return (float)(uint32_t)(key >> 40) * (1.0f / 16777216.0f);
}

// ---------------------------------------------------------------- coordinates
template <int DIM>
struct Vec;
template <>
struct Vec<2> {
    using T = float2;
};
template <>
struct Vec<3> {
    using T = float4;
};

template <int DIM>
__device__ __forceinline__ float4 load_x(const float* __restrict__ x, int64_t i) {
    if constexpr (DIM == 2) {
        float2 v = __ldg(reinterpret_cast<const float2*>(x) + i);
        return make_float4(v.x, v.y, 0.f, 0.f);
    } else {
        float4 v = __ldg(reinterpret_cast<const float4*>(x) + i);
        v.w = 0.f;
        return v;
    }
}
template <int DIM>
__device__ __forceinline__ void store_x(float* __restrict__ x, int64_t i, float4 v) {
    if constexpr (DIM == 2) {
        reinterpret_cast<float2*>(x)[i] = make_float2(v.x, v.y);
    } else {
        v.w = 0.f;
        reinterpret_cast<float4*>(x)[i] = v;
    }
}

// ---------------------------------------------------------------- launch bookkeeping
// Implemented in api.cu: counts launches and (optionally) brackets them with events.
struct LaunchScope {
    const char* name;
    cudaStream_t stream;
    int slot;
    LaunchScope(const char* name, cudaStream_t s);
    ~LaunchScope();
};

}  // namespace mm
