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

// Softening added to r^2 before the reciprocal (reading Q6): an exactly
// coincident pair gives 0 * rcp(eps) = 0.  1e-18 keeps the product of two
// softened r^2 (batched reciprocal, k_repulse.cu) a normal float; it changes
// r^2 by < 1e-6 relative for every pair with r > 1e-6.
constexpr float kEps2 = 1e-18f;
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

// ---------------------------------------------------------------- packed FP32 pairs
// A pair of floats held in one 64-bit register (PTX .b64) so that ptxas keeps
// it in an aligned register pair and emits FADD2/FFMA2/FMUL2 without MOVs.
typedef uint64_t f2x;
__device__ __forceinline__ f2x pk(float a, float b) {
    f2x r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void upk(f2x r, float& a, float& b) {
    asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
// a - (s, s): FADD2 with a broadcast scalar operand
__device__ __forceinline__ f2x sub_bc(f2x a, float s) {
    f2x d;
    asm("{.reg .b64 t; mov.b64 t, {%2,%2}; sub.rn.f32x2 %0, %1, t;}" : "=l"(d) : "l"(a), "f"(s));
    return d;
}
// a * (s, s): FMUL2 with a broadcast scalar operand
__device__ __forceinline__ f2x mul_bc(f2x a, float s) {
    f2x d;
    asm("{.reg .b64 t; mov.b64 t, {%2,%2}; mul.rn.f32x2 %0, %1, t;}" : "=l"(d) : "l"(a), "f"(s));
    return d;
}
__device__ __forceinline__ f2x add2(f2x a, f2x b) {
    f2x d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f2x fma2(f2x a, f2x b, f2x c) {
    f2x d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ f2x mul2(f2x a, f2x b) {
    f2x d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
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
constexpr uint64_t kTagDisc = 0x44495343ULL;    // "DISC"

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
