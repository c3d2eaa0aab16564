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
// Design (B200, sm_100a): n-body tiling.  A work item is (target block of
// 256*T targets, source tile of 256 sources); targets live in registers (T per
// thread, packed pairwise into float2 so every FP32 op is FADD2/FFMA2/FMUL2),
// sources are staged through shared memory and read back as broadcast LDS.
// The inner loop is bound by the MUFU (XU) pipe, 16 ops/clk/SM, not by HBM:
// one 8-32 B source feeds 256*T pairs.
//   * q = 0 uses batched reciprocals in half of the target groups:
//     1/a = b * rcp(a*b), 1/b = a * rcp(a*b)  (one MUFU for two pairs, three
//     FMUL lanes), which balances the MUFU and FMA pipes.
//   * Schedule: a persistent grid of G = 148 x (resident CTAs per SM) CTAs;
//     the linearised (target block, source tile) space is split into G equal
//     contiguous ranges, so every SM gets the same number of pairs (no tail
//     wave).  A CTA whose range crosses target blocks writes one partial per
//     block into slot (g - first CTA of that block); kernel (a) sums the
//     slots of a vertex in slot order.  The split is static, so the result is
//     bitwise independent of scheduling.
//   * Coarse representatives are stored as FP64-accurate hi + lo float pairs
//     and differenced as (x_i - hi) - lo: a target near a foreign centroid
//     then keeps full relative precision in x_i - x'.
#include "k_repulse.cuh"

namespace mm {

namespace {

constexpr int kBlock = 256;   // threads per CTA = sources per shared-memory tile

// 1/|d|^(q+2) for a packed pair of r^2.  q = 0 batched: one MUFU for both,
// 1/a = b * rcp(a*b), 1/b = a * rcp(a*b) (FMUL + MUFU + FMUL2 with swapped halves).
template <bool QPOW, bool BATCH>
__device__ __forceinline__ f2x inv_pair(f2x r2, float cexp) {
    float r0, r1;
    upk(r2, r0, r1);
    if constexpr (!QPOW && BATCH) {
        const float ip = rcp_approx(r0 * r1);
        return mul2(pk(r1, r0), pk(ip, ip));
    } else {
        return pk(inv_pow<QPOW>(r0, cexp), inv_pow<QPOW>(r1, cexp));
    }
}

template <int DIM, bool QPOW, bool COARSE, int T>
__global__ void __launch_bounds__(kBlock) k_repulse(int32_t n_tgt, const float* __restrict__ x, int32_t n_src,
                                                    const float4* __restrict__ rep_hi,
                                                    const float4* __restrict__ rep_lo,
                                                    const int32_t* __restrict__ anc, float cexp, Sched sch,
                                                    float* __restrict__ part) {
    static_assert(T % 2 == 0, "targets are processed in packed pairs");
    constexpr int G = T / 2;
    constexpr int TPB = kBlock * T;
    constexpr int stride = DIM == 2 ? 2 : 4;
    // shared source tile: exact 2-D -> float2; exact 3-D -> float4; coarse -> hi/lo float4 pairs
    __shared__ float4 sm_a[kBlock];
    __shared__ float4 sm_b[COARSE ? kBlock : 1];
    float2* sm2 = reinterpret_cast<float2*>(sm_a);

    const int tid = threadIdx.x;
    const int32_t g = blockIdx.x;
    const int64_t u0 = (int64_t)g * sch.U / sch.G, u1 = (int64_t)(g + 1) * sch.U / sch.G;
    const f2x eps2 = pk(kEps2, kEps2);

    for (int64_t u = u0; u < u1;) {
        const int32_t tb = (int32_t)(u / sch.Ub);
        const int64_t seg_end = min(u1, (int64_t)(tb + 1) * sch.Ub);
        const int32_t tile0 = (int32_t)(u - (int64_t)tb * sch.Ub), tile1 = (int32_t)(seg_end - (int64_t)tb * sch.Ub);
        // targets of this block (registers), packed pairwise
        f2x X[G], Y[G], Z[G], AX[G], AY[G], AZ[G];
        int32_t hi[T];
        const int64_t base = (int64_t)tb * TPB;
#pragma unroll
        for (int gg = 0; gg < G; ++gg) {
            const int64_t ia = base + (2 * gg) * kBlock + tid, ib = base + (2 * gg + 1) * kBlock + tid;
            const int64_t ca = ia < n_tgt ? ia : n_tgt - 1, cb = ib < n_tgt ? ib : n_tgt - 1;
            // scalar loads, so that ptxas can place (x_a, x_b) in one aligned
            // register pair for the whole loop (vector loads would interleave
            // the halves and force MOVs to re-form the pair at every use)
            const float* pa = x + ca * stride;
            const float* pb = x + cb * stride;
            X[gg] = pk(__ldg(pa), __ldg(pb));
            Y[gg] = pk(__ldg(pa + 1), __ldg(pb + 1));
            Z[gg] = (DIM == 3) ? pk(__ldg(pa + 2), __ldg(pb + 2)) : 0ull;
            AX[gg] = AY[gg] = AZ[gg] = 0ull;
            if constexpr (COARSE) {
                hi[2 * gg] = __ldg(anc + ca);
                hi[2 * gg + 1] = __ldg(anc + cb);
            }
        }
        (void)hi;
        for (int32_t tile = tile0; tile < tile1; ++tile) {
            const int64_t t0 = (int64_t)tile * kBlock;
            const int cnt = (int)min((int64_t)kBlock, (int64_t)n_src - t0);
            __syncthreads();
            if (tid < cnt) {
                if constexpr (COARSE) {
                    sm_a[tid] = __ldg(rep_hi + t0 + tid);
                    sm_b[tid] = __ldg(rep_lo + t0 + tid);
                } else if constexpr (DIM == 2) {
                    sm2[tid] = __ldg(reinterpret_cast<const float2*>(x) + t0 + tid);
                } else {
                    sm_a[tid] = __ldg(reinterpret_cast<const float4*>(x) + t0 + tid);
                }
            }
            __syncthreads();
            // per-tile FP32 accumulators, folded into the running sums after the tile
            f2x TX[G], TY[G], TZ[G];
#pragma unroll
            for (int gg = 0; gg < G; ++gg) TX[gg] = TY[gg] = TZ[gg] = 0ull;
#pragma unroll 4
            for (int jj = 0; jj < cnt; ++jj) {
                float sx, sy, sz = 0.f, lx = 0.f, ly = 0.f, lz = 0.f, nu = 1.f;
                if constexpr (COARSE) {
                    const float4 a = sm_a[jj], b = sm_b[jj];
                    sx = a.x; sy = a.y; sz = a.z; nu = a.w;
                    lx = b.x; ly = b.y; lz = b.z;
                } else if constexpr (DIM == 2) {
                    const float2 a = sm2[jj];
                    sx = a.x; sy = a.y;
                } else {
                    const float4 a = sm_a[jj];
                    sx = a.x; sy = a.y; sz = a.z;
                }
#pragma unroll
                for (int gg = 0; gg < G; ++gg) {
                    f2x dx = sub_bc(X[gg], sx);
                    f2x dy = sub_bc(Y[gg], sy);
                    if constexpr (COARSE) {
                        dx = sub_bc(dx, lx);
                        dy = sub_bc(dy, ly);
                    }
                    f2x r2 = fma2(dx, dx, eps2);
                    r2 = fma2(dy, dy, r2);
                    f2x dz = 0ull;
                    if constexpr (DIM == 3) {
                        dz = sub_bc(Z[gg], sz);
                        if constexpr (COARSE) dz = sub_bc(dz, lz);
                        r2 = fma2(dz, dz, r2);
                    }
                    f2x inv = (gg % 2 == 0) ? inv_pair<QPOW, true>(r2, cexp) : inv_pair<QPOW, false>(r2, cexp);
                    if constexpr (COARSE) {
                        const int32_t j = (int32_t)(t0 + jj);
                        inv = mul2(inv, pk(j == hi[2 * gg] ? 0.f : nu, j == hi[2 * gg + 1] ? 0.f : nu));
                    }
                    TX[gg] = fma2(dx, inv, TX[gg]);
                    TY[gg] = fma2(dy, inv, TY[gg]);
                    if constexpr (DIM == 3) TZ[gg] = fma2(dz, inv, TZ[gg]);
                }
            }
#pragma unroll
            for (int gg = 0; gg < G; ++gg) {
                AX[gg] = add2(AX[gg], TX[gg]);
                AY[gg] = add2(AY[gg], TY[gg]);
                if constexpr (DIM == 3) AZ[gg] = add2(AZ[gg], TZ[gg]);
            }
        }
        // partial of this (target block, CTA) pair -> slot g - first CTA of the block
        const int32_t slot = g - sched_first_cta((int64_t)tb * sch.Ub, sch);
        float* out = part + (int64_t)slot * n_tgt * stride;
#pragma unroll
        for (int gg = 0; gg < G; ++gg) {
            const int64_t ia = base + (2 * gg) * kBlock + tid, ib = base + (2 * gg + 1) * kBlock + tid;
            float ax0, ax1, ay0, ay1, az0 = 0.f, az1 = 0.f;
            upk(AX[gg], ax0, ax1);
            upk(AY[gg], ay0, ay1);
            if constexpr (DIM == 3) upk(AZ[gg], az0, az1);
            if (ia < n_tgt) store_x<DIM>(out, ia, make_float4(ax0, ay0, az0, 0.f));
            if (ib < n_tgt) store_x<DIM>(out, ib, make_float4(ax1, ay1, az1, 0.f));
        }
        u = seg_end;
    }
}

// All-pairs entropy for mm_energy: per target, sum over j != i of phi_q(r)
// in the form  q = 0: sum lg2(r^2 + eps)   (phi_0 = -ln r = -(ln 2 / 2) lg2 r^2)
//              q > 0: sum 2^(-q/2 lg2(r^2 + eps))   (phi_q = r^-q / q)
// plus a count of exactly coincident pairs (j != i).  FP32 per thread and
// tile, FP64 across tiles and threads, written per CTA.
template <int DIM, bool QPOW>
__global__ void __launch_bounds__(kBlock) k_entropy_all(int32_t n, const float* __restrict__ x, float cq,
                                                        int32_t chunk, double* __restrict__ partial,
                                                        int32_t* __restrict__ coinc) {
    __shared__ float4 sm[kBlock];
    __shared__ double red[kBlock / 32];
    __shared__ int32_t redc[kBlock / 32];
    const int tid = threadIdx.x;
    const int64_t i = (int64_t)blockIdx.x * kBlock + tid;
    const int64_t ci = i < n ? i : n - 1;
    const float4 xi = load_x<DIM>(x, ci);
    double dacc = 0.0;
    int32_t zc = 0;
    const int64_t s_begin = (int64_t)blockIdx.y * chunk;
    const int64_t s_end = min((int64_t)n, s_begin + chunk);
    for (int64_t t0 = s_begin; t0 < s_end; t0 += kBlock) {
        const int cnt = (int)min((int64_t)kBlock, s_end - t0);
        __syncthreads();
        if (tid < cnt) sm[tid] = load_x<DIM>(x, t0 + tid);
        __syncthreads();
        float acc = 0.f;
#pragma unroll 4
        for (int jj = 0; jj < cnt; ++jj) {
            const float4 s = sm[jj];
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
        dacc += (double)acc;
    }
    if (i >= n) {
        dacc = 0.0;
        zc = 0;
    }
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
        for (int w = 0; w < kBlock / 32; ++w) {
            s += red[w];
            c += redc[w];
        }
        partial[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = s;
        if (c) atomicAdd(coinc, c);
    }
}

template <int DIM, bool QPOW, bool COARSE, int T>
int resident_ctas() {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_repulse<DIM, QPOW, COARSE, T>, kBlock, 0);
    return occ > 0 ? occ : 1;
}

int sm_count() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
    }
    return sms;
}

int targets_per_thread(int dim) { return dim == 2 ? 4 : 2; }

}  // namespace

// ---------------------------------------------------------------- host launchers

RepulsePlan plan_repulse(int32_t n_tgt, int32_t n_src, int dim, bool coarse, bool qpow) {
    RepulsePlan p;
    const int T = targets_per_thread(dim);
    const int64_t TPB = (int64_t)kBlock * T;
    Sched& s = p.sch;
    s.TB = (int32_t)((n_tgt + TPB - 1) / TPB);
    s.Ub = (int32_t)((n_src + kBlock - 1) / kBlock);
    s.U = (int64_t)s.TB * s.Ub;
    int occ;
    if (dim == 2) {
        occ = coarse ? (qpow ? resident_ctas<2, true, true, 4>() : resident_ctas<2, false, true, 4>())
                     : (qpow ? resident_ctas<2, true, false, 4>() : resident_ctas<2, false, false, 4>());
    } else {
        occ = coarse ? (qpow ? resident_ctas<3, true, true, 2>() : resident_ctas<3, false, true, 2>())
                     : (qpow ? resident_ctas<3, true, false, 2>() : resident_ctas<3, false, false, 2>());
    }
    s.G = (int32_t)std::max<int64_t>(1, std::min<int64_t>((int64_t)sm_count() * occ, s.U));
    // slots: max over target blocks of (CTAs touching the block)
    int32_t ms = 1;
    for (int32_t tb = 0; tb < s.TB; ++tb) {
        const int32_t a = sched_first_cta((int64_t)tb * s.Ub, s);
        const int32_t b = sched_first_cta((int64_t)(tb + 1) * s.Ub - 1, s);
        ms = std::max(ms, b - a + 1);
    }
    p.slots = ms;
    return p;
}

cudaError_t launch_repulse(int dim, bool qpow, bool coarse, float q, int32_t n_tgt, const float* x,
                           int32_t n_src, const float4* rep_hi, const float4* rep_lo, const int32_t* anc,
                           const RepulsePlan& p, float* part, cudaStream_t st) {
    const float cexp = -(q + 2.0f) * 0.5f;
    LaunchScope ls(coarse ? "repulse_coarse" : "repulse_exact", st);
#define MM_LAUNCH(D, Q, C, T) \
    k_repulse<D, Q, C, T><<<p.sch.G, kBlock, 0, st>>>(n_tgt, x, n_src, rep_hi, rep_lo, anc, cexp, p.sch, part)
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

int repulse_targets_per_block(int dim) { return kBlock * targets_per_thread(dim); }

EntropyPlan plan_entropy(int32_t n) {
    EntropyPlan p;
    p.tblocks = (n + kBlock - 1) / kBlock;
    int P = (sm_count() * 6 + p.tblocks - 1) / p.tblocks;
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
        if (qpow) k_entropy_all<2, true><<<grid, kBlock, 0, st>>>(n, x, cq, p.chunk, partial, coinc);
        else k_entropy_all<2, false><<<grid, kBlock, 0, st>>>(n, x, cq, p.chunk, partial, coinc);
    } else {
        if (qpow) k_entropy_all<3, true><<<grid, kBlock, 0, st>>>(n, x, cq, p.chunk, partial, coinc);
        else k_entropy_all<3, false><<<grid, kBlock, 0, st>>>(n, x, cq, p.chunk, partial, coinc);
    }
    return cudaGetLastError();
}

}  // namespace mm
