// k_repulse.cu — kernels (b) exact all-pairs repulsion, (c) coarse-
// representative repulsion, and the all-pairs entropy sum of mm_energy.
//
// (b) computes, for every target i, R_i^all = sum_{j != i} (x_i - x_j)/|x_i - x_j|^(q+2)
//     over ALL vertices (the second term of Eq.(2), with the
//     exponent q of BASELINE.json's north_star).  Kernel (a) afterwards
//     subtracts the S_i pairs, so the net sum runs over j notin S_i.
// (c) computes sum_{v' != H(i)} nu(v') (x_i - x'_v')/|x_i - x'_v'|^(q+2), the
//     representative term of Eq.(3), over the k coarse
//     representatives {x', nu} of the approximation level.
//
// Design (B200, sm_100a): n-body tiling.  A CTA owns BLOCK*T targets (T per
// thread, packed pairwise into float2 registers so every FP32 op is an
// FADD2/FFMA2/FMUL2) and one chunk of the sources; sources are staged through
// shared memory one BLOCK-sized tile at a time and read back as broadcast
// LDS.128.  Per pair: 1 FADD2 per axis, 1 FFMA2 per axis for r^2, one MUFU
// (rcp for q = 0; lg2+ex2 for q > 0), 1 FFMA2 per axis for the accumulation.
// The inner loop is MUFU-bound (16 MUFU/clk/SM), not HBM-bound: one 8-16 B
// source feeds BLOCK*T pairs.  Source chunks (grid.y) give the grid enough
// CTAs to fill 148 SMs; partial sums part[p][i] are reduced by kernel (a) in
// the fixed order p = 0..P-1, so the result does not depend on scheduling.
#include "k_repulse.cuh"

namespace mm {

namespace {

template <int DIM, bool COARSE>
struct SrcT {
    using T = float4;
};
template <>
struct SrcT<2, false> {
    using T = float2;
};

template <int DIM, bool QPOW, bool COARSE, int BLOCK, int T>
__global__ void __launch_bounds__(BLOCK) k_repulse(int32_t n_tgt, const float* __restrict__ x,
                                                   int32_t n_src, const float4* __restrict__ reps,
                                                   const int32_t* __restrict__ anc, float cexp,
                                                   int32_t chunk, float* __restrict__ part) {
    static_assert(T % 2 == 0, "targets are processed in packed pairs");
    constexpr int G = T / 2;
    using S = typename SrcT<DIM, COARSE>::T;
    __shared__ S sm[BLOCK];

    const int tid = threadIdx.x;
    const int64_t base = (int64_t)blockIdx.x * BLOCK * T;
    float2 X[G], Y[G], Z[G], AX[G], AY[G], AZ[G];
    int32_t hi[T];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        float4 a, b;
        int64_t ia = base + (2 * g) * BLOCK + tid, ib = base + (2 * g + 1) * BLOCK + tid;
        int64_t ca = ia < n_tgt ? ia : n_tgt - 1, cb = ib < n_tgt ? ib : n_tgt - 1;
        a = load_x<DIM>(x, ca);
        b = load_x<DIM>(x, cb);
        X[g] = make_float2(a.x, b.x);
        Y[g] = make_float2(a.y, b.y);
        Z[g] = make_float2(a.z, b.z);
        AX[g] = AY[g] = AZ[g] = make_float2(0.f, 0.f);
        if constexpr (COARSE) {
            hi[2 * g] = __ldg(anc + ca);
            hi[2 * g + 1] = __ldg(anc + cb);
        }
    }
    (void)hi;
    const float2 eps2 = make_float2(kEps2, kEps2);

    const int64_t s_begin = (int64_t)blockIdx.y * chunk;
    const int64_t s_end = min((int64_t)n_src, s_begin + chunk);
    for (int64_t t0 = s_begin; t0 < s_end; t0 += BLOCK) {
        const int cnt = (int)min((int64_t)BLOCK, s_end - t0);
        __syncthreads();
        if (tid < cnt) {
            if constexpr (COARSE) {
                sm[tid] = __ldg(reps + t0 + tid);
            } else if constexpr (DIM == 2) {
                sm[tid] = __ldg(reinterpret_cast<const float2*>(x) + t0 + tid);
            } else {
                sm[tid] = __ldg(reinterpret_cast<const float4*>(x) + t0 + tid);
            }
        }
        __syncthreads();
#pragma unroll 4
        for (int jj = 0; jj < cnt; ++jj) {
            const S s = sm[jj];
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const float2 dx = __fadd2_rn(X[g], make_float2(-s.x, -s.x));
                const float2 dy = __fadd2_rn(Y[g], make_float2(-s.y, -s.y));
                float2 r2 = __ffma2_rn(dx, dx, eps2);
                r2 = __ffma2_rn(dy, dy, r2);
                float2 dz;
                if constexpr (DIM == 3) {
                    dz = __fadd2_rn(Z[g], make_float2(-s.z, -s.z));
                    r2 = __ffma2_rn(dz, dz, r2);
                }
                float2 inv = make_float2(inv_pow<QPOW>(r2.x, cexp), inv_pow<QPOW>(r2.y, cexp));
                if constexpr (COARSE) {
                    const int32_t j = (int32_t)(t0 + jj);
                    const float nu = s.w;
                    inv = __fmul2_rn(inv, make_float2(j == hi[2 * g] ? 0.f : nu, j == hi[2 * g + 1] ? 0.f : nu));
                }
                AX[g] = __ffma2_rn(dx, inv, AX[g]);
                AY[g] = __ffma2_rn(dy, inv, AY[g]);
                if constexpr (DIM == 3) AZ[g] = __ffma2_rn(dz, inv, AZ[g]);
            }
        }
    }
    float* out = part + (int64_t)blockIdx.y * n_tgt * (DIM == 2 ? 2 : 4);
#pragma unroll
    for (int g = 0; g < G; ++g) {
        int64_t ia = base + (2 * g) * BLOCK + tid, ib = base + (2 * g + 1) * BLOCK + tid;
        if (ia < n_tgt) store_x<DIM>(out, ia, make_float4(AX[g].x, AY[g].x, AZ[g].x, 0.f));
        if (ib < n_tgt) store_x<DIM>(out, ib, make_float4(AX[g].y, AY[g].y, AZ[g].y, 0.f));
    }
}

// All-pairs entropy for mm_energy: per target, sum over j != i of phi_q(r)
// in the form  q = 0: sum lg2(r^2 + eps)   (phi_0 = -ln r = -(ln 2 / 2) lg2 r^2)
//              q > 0: sum 2^(-q/2 lg2(r^2 + eps))   (phi_q = r^-q / q)
// plus a count of exactly coincident pairs (j != i).  FP32 per thread, FP64
// per CTA, written to partials[blockIdx.y * gridDim.x + blockIdx.x].
template <int DIM, bool QPOW, int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_entropy_all(int32_t n, const float* __restrict__ x, float cq,
                                                       int32_t chunk, double* __restrict__ partial,
                                                       int32_t* __restrict__ coinc) {
    using S = typename SrcT<DIM, false>::T;
    __shared__ S sm[BLOCK];
    __shared__ double red[BLOCK / 32];
    __shared__ int32_t redc[BLOCK / 32];
    const int tid = threadIdx.x;
    const int64_t i = (int64_t)blockIdx.x * BLOCK + tid;
    const int64_t ci = i < n ? i : n - 1;
    const float4 xi = load_x<DIM>(x, ci);
    float acc = 0.f;
    int32_t zc = 0;
    const int64_t s_begin = (int64_t)blockIdx.y * chunk;
    const int64_t s_end = min((int64_t)n, s_begin + chunk);
    for (int64_t t0 = s_begin; t0 < s_end; t0 += BLOCK) {
        const int cnt = (int)min((int64_t)BLOCK, s_end - t0);
        __syncthreads();
        if (tid < cnt) {
            if constexpr (DIM == 2) sm[tid] = __ldg(reinterpret_cast<const float2*>(x) + t0 + tid);
            else sm[tid] = __ldg(reinterpret_cast<const float4*>(x) + t0 + tid);
        }
        __syncthreads();
#pragma unroll 4
        for (int jj = 0; jj < cnt; ++jj) {
            const S s = sm[jj];
            const float dx = xi.x - s.x, dy = xi.y - s.y;
            float r2 = fmaf(dx, dx, 0.f);
            r2 = fmaf(dy, dy, r2);
            if constexpr (DIM == 3) {
                const float dz = xi.z - s.z;
                r2 = fmaf(dz, dz, r2);
            }
            const bool self = (t0 + jj) == i;
            zc += (r2 == 0.f && !self) ? 1 : 0;
            const float l = lg2_approx(r2 + kEps2);
            float v;
            if constexpr (!QPOW) v = l;
            else v = ex2_approx(fminf(cq * l, kExpClamp));
            acc += self ? 0.f : v;
        }
    }
    double dacc = (i < n) ? (double)acc : 0.0;
    if (i >= n) zc = 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        dacc += __shfl_xor_sync(0xffffffffu, dacc, o);
        zc += __shfl_xor_sync(0xffffffffu, zc, o);
    }
    if ((tid & 31) == 0) {
        red[tid >> 5] = dacc;
        redc[tid >> 5] = zc;
    }
    __syncthreads();
    if (tid == 0) {
        double s = 0.0;
        int32_t c = 0;
        for (int w = 0; w < BLOCK / 32; ++w) {
            s += red[w];
            c += redc[w];
        }
        partial[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = s;
        if (c) atomicAdd(coinc, c);
    }
}

constexpr int kBlock = 256;

template <int DIM, int T>
int num_target_blocks(int32_t n_tgt) {
    return (int)((n_tgt + (int64_t)kBlock * T - 1) / ((int64_t)kBlock * T));
}

}  // namespace

// ---------------------------------------------------------------- host launchers

RepulsePlan plan_repulse(int32_t n_tgt, int32_t n_src, int dim) {
    RepulsePlan p;
    const int T = (dim == 2) ? 4 : 2;
    p.tblocks = (int)((n_tgt + (int64_t)kBlock * T - 1) / ((int64_t)kBlock * T));
    // Aim for about one full wave of resident CTAs (148 SMs x 6 CTAs of 256
    // threads) of equal size, with chunks of at least 2 tiles.
    const int target_ctas = 148 * 6;
    int P = (target_ctas + p.tblocks - 1) / p.tblocks;
    const int max_p = (int)std::max<int64_t>(1, (int64_t)n_src / (2 * kBlock));
    P = std::max(1, std::min(P, max_p));
    int64_t chunk = ((int64_t)n_src + P - 1) / P;
    chunk = ((chunk + kBlock - 1) / kBlock) * kBlock;
    p.chunk = (int32_t)std::max<int64_t>(chunk, kBlock);
    p.P = (int)(((int64_t)n_src + p.chunk - 1) / p.chunk);
    if (p.P < 1) p.P = 1;
    return p;
}

cudaError_t launch_repulse(int dim, bool qpow, bool coarse, float q, int32_t n_tgt, const float* x,
                           int32_t n_src, const float4* reps, const int32_t* anc, const RepulsePlan& p,
                           float* part, cudaStream_t st) {
    const float cexp = -(q + 2.0f) * 0.5f;
    dim3 grid(p.tblocks, p.P);
    LaunchScope ls(coarse ? "repulse_coarse" : "repulse_exact", st);
#define MM_LAUNCH(D, Q, C, T) \
    k_repulse<D, Q, C, kBlock, T><<<grid, kBlock, 0, st>>>(n_tgt, x, n_src, reps, anc, cexp, p.chunk, part)
    if (dim == 2) {
        if (!qpow && !coarse) MM_LAUNCH(2, false, false, 4);
        else if (!qpow && coarse) MM_LAUNCH(2, false, true, 4);
        else if (qpow && !coarse) MM_LAUNCH(2, true, false, 4);
        else MM_LAUNCH(2, true, true, 4);
    } else {
        if (!qpow && !coarse) MM_LAUNCH(3, false, false, 2);
        else if (!qpow && coarse) MM_LAUNCH(3, false, true, 2);
        else if (qpow && !coarse) MM_LAUNCH(3, true, false, 2);
        else MM_LAUNCH(3, true, true, 2);
    }
#undef MM_LAUNCH
    return cudaGetLastError();
}

EntropyPlan plan_entropy(int32_t n) {
    EntropyPlan p;
    p.tblocks = (n + kBlock - 1) / kBlock;
    int P = (148 * 6 + p.tblocks - 1) / p.tblocks;
    P = std::max(1, std::min(P, std::max(1, n / (2 * kBlock))));
    int64_t chunk = ((int64_t)n + P - 1) / P;
    chunk = ((chunk + kBlock - 1) / kBlock) * kBlock;
    p.chunk = (int32_t)std::max<int64_t>(chunk, kBlock);
    p.P = (int)(((int64_t)n + p.chunk - 1) / p.chunk);
    return p;
}

cudaError_t launch_entropy_all(int dim, double q, int32_t n, const float* x, const EntropyPlan& p,
                               double* partial, int32_t* coinc, cudaStream_t st) {
    dim3 grid(p.tblocks, p.P);
    const float cq = (float)(-q * 0.5);
    LaunchScope ls("entropy_all", st);
    const bool qpow = q != 0.0;
    if (dim == 2) {
        if (qpow) k_entropy_all<2, true, kBlock><<<grid, kBlock, 0, st>>>(n, x, cq, p.chunk, partial, coinc);
        else k_entropy_all<2, false, kBlock><<<grid, kBlock, 0, st>>>(n, x, cq, p.chunk, partial, coinc);
    } else {
        if (qpow) k_entropy_all<3, true, kBlock><<<grid, kBlock, 0, st>>>(n, x, cq, p.chunk, partial, coinc);
        else k_entropy_all<3, false, kBlock><<<grid, kBlock, 0, st>>>(n, x, cq, p.chunk, partial, coinc);
    }
    return cudaGetLastError();
}

}  // namespace mm
