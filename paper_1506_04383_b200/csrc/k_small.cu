// k_small.cu — all the sweeps of one SMALL level in one persistent kernel.
//
// A coarse level (n up to a few 10^4, k up to a few 10^3 representatives)
// needs only microseconds of arithmetic per sweep, but a sweep of the tiled
// path is 3-4 kernel launches (centroids, repulsion, gather, schedule
// decision) whose latency dominates: the paper's schedule runs up
// to ~200 sweeps per level.  This kernel runs them all in one cooperative
// launch (one CTA per SM, all co-resident) with grid barriers between phases:
//
//   per sweep  (x_in -> x_out, Jacobi)
//   [Eq.(3) only] representatives x'_v' = member means (FP64, hi/lo, Q11/Q24),
//                 one warp per representative                               -> grid barrier
//   every CTA stages the sources in shared memory: the k representatives
//   {hi, lo, nu} (Eq.(3)) or all n coordinates (Eq.(2))
//   one warp per target i (lanes stride the sources, the S row, the siblings):
//     R_i = sum over all sources (x_i - s)/|x_i - s|^(q+2)   [Eq.(3): nu-weighted, (x_i - hi) - lo]
//           - own representative (Eq.(3), Q25) + siblings under P(i) (Eq.(3))
//     S_i gather: rho_i, A_i, C_i (S-pair r-values, subtracted), stress
//     x'_i = (A_i + alpha (R_i - C_i)) / rho_i
//   per-CTA FP64 partials of (|x'-x|^2, |x|^2, stress, non-finite)            -> grid barrier
//   every CTA sums the partials in CTA order (identical in every CTA) and makes
//   the same decision: fixed K sweeps (mm_layout) or the schedule's rules in
//   double arithmetic (mm_layout_schedule, exactly as the host runner)
//
// The pair term, the S-pair subtraction and the own-representative
// subtraction use the same FP32 formulas as kernels (a)-(c); only the
// summation order differs (one thread sums all sources of its target).
#include <cooperative_groups.h>

#include "k_small.cuh"

namespace mm {

namespace {

constexpr int kSmallBlock = 256;

struct SmallState {
    unsigned bar_count;
    unsigned bar_gen;
};
__device__ SmallState g_small;

// grid-wide barrier for a cooperative launch (all CTAs resident)
__device__ __forceinline__ void grid_barrier(unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* gen = &g_small.bar_gen;
        const unsigned g = *gen;
        __threadfence();
        if (atomicAdd(&g_small.bar_count, 1u) == nblocks - 1) {
            g_small.bar_count = 0;
            __threadfence();
            atomicAdd(&g_small.bar_gen, 1u);
        } else {
            while (*gen == g) __nanosleep(40);
        }
        __threadfence();
    }
    __syncthreads();
}

// coordinates written inside this launch are read through L2 (ld.global.cg):
// the non-coherent path (__ldg) could return a line cached two sweeps ago
template <int DIM>
__device__ __forceinline__ float4 load_xc(const float* x, int64_t i) {
    if constexpr (DIM == 2) {
        const float2 v = __ldcg(reinterpret_cast<const float2*>(x) + i);
        return make_float4(v.x, v.y, 0.f, 0.f);
    } else {
        float4 v = __ldcg(reinterpret_cast<const float4*>(x) + i);
        v.w = 0.f;
        return v;
    }
}

template <int DIM>
__device__ __forceinline__ void pair_term(const float4& xi, float sx, float sy, float sz, float w, float cexp,
                                          bool qpow, float4& acc) {
    const float dx = xi.x - sx, dy = xi.y - sy;
    float r2 = fmaf(dx, dx, kEps2);
    r2 = fmaf(dy, dy, r2);
    float dz = 0.f;
    if constexpr (DIM == 3) {
        dz = xi.z - sz;
        r2 = fmaf(dz, dz, r2);
    }
    const float inv = (qpow ? inv_pow<true>(r2, cexp) : inv_pow<false>(r2, cexp)) * w;
    acc.x = fmaf(dx, inv, acc.x);
    acc.y = fmaf(dy, inv, acc.y);
    if constexpr (DIM == 3) acc.z = fmaf(dz, inv, acc.z);
}

template <int DIM, bool APPROX, int G>
__global__ void __launch_bounds__(kSmallBlock, 1) k_small_level(SmallArgs a) {
    extern __shared__ float4 sm[];  // APPROX: [k] hi, [k] lo ; exact: [n] coordinates
    __shared__ double red[4][kSmallBlock / 32];
    const unsigned NB = gridDim.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int lg = tid & (G - 1);  // lane within the target's group of G lanes
    const float cexp = -(a.q + 2.0f) * 0.5f;
    const bool qpow = a.q != 0.0f;
    const float* xin = a.x0;
    float* xout = a.x1;
    // schedule state (identical in every CTA)
    double alpha = a.alpha0;
    int32_t it = 0, count = 0, err = 0;
    bool fin = alpha <= a.alpha_min;
    int32_t max_it = fin ? a.max_final : a.rounds;
    double last[3] = {0.0, 0.0, 0.0};
    for (;;) {
        // ---- representatives of x_in (Eq.(3))
        if constexpr (APPROX) {
            const int32_t gw = (int32_t)(blockIdx.x * (kSmallBlock / 32) + warp), nw = (int32_t)(NB * (kSmallBlock / 32));
            for (int32_t v = gw; v < a.k; v += nw) {
                const int32_t b = __ldg(a.mptr + v), e = __ldg(a.mptr + v + 1);
                double sx = 0.0, sy = 0.0, sz = 0.0;
                for (int32_t t = b + lane; t < e; t += 32) {
                    const float4 p = load_xc<DIM>(xin, __ldg(a.mem + t));
                    sx += p.x;
                    sy += p.y;
                    sz += p.z;
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    sx += __shfl_xor_sync(0xffffffffu, sx, o);
                    sy += __shfl_xor_sync(0xffffffffu, sy, o);
                    sz += __shfl_xor_sync(0xffffffffu, sz, o);
                }
                if (lane == 0) {
                    const double nu = (double)(e - b);
                    const double mx = sx / nu, my = sy / nu, mz = DIM == 3 ? sz / nu : 0.0;
                    const float hx = (float)mx, hy = (float)my, hz = (float)mz;
                    a.rep_hi[v] = make_float4(hx, hy, hz, (float)nu);
                    a.rep_lo[v] = make_float4((float)(mx - hx), (float)(my - hy), (float)(mz - hz), 0.f);
                }
            }
            grid_barrier(NB);
            for (int32_t v = tid; v < a.k; v += kSmallBlock) {
                sm[v] = __ldcg(a.rep_hi + v);
                sm[a.k + v] = __ldcg(a.rep_lo + v);
            }
        } else {
            for (int32_t v = tid; v < a.n; v += kSmallBlock) sm[v] = load_xc<DIM>(xin, v);
        }
        __syncthreads();
        // ---- one warp per target: lanes stride the sources, the S row and the
        //      siblings; a fixed xor tree combines the lanes
        double v_dx2 = 0.0, v_x2 = 0.0, v_st = 0.0;
        int32_t bad = 0;
        const float alpha_f = (float)alpha;
        const int32_t gg = (int32_t)((blockIdx.x * kSmallBlock + tid) / G), ng = (int32_t)(NB * (kSmallBlock / G));
        // all lanes of a warp run the same number of iterations (the shuffles need them)
        const int32_t iters = (a.n + ng - 1) / ng;
        for (int32_t r = 0; r < iters; ++r) {
            const int32_t i0 = gg + r * ng;
            const bool valid = i0 < a.n;
            const int32_t i = valid ? i0 : a.n - 1;
            const float4 xi = load_xc<DIM>(xin, i);
            float4 R = make_float4(0.f, 0.f, 0.f, 0.f), C = R, A = R;
            if constexpr (APPROX) {
                for (int32_t v = lg; v < a.k; v += G) {
                    const float4 h = sm[v], l = sm[a.k + v];
                    const float4 d4 = make_float4((xi.x - h.x) - l.x, (xi.y - h.y) - l.y, (xi.z - h.z) - l.z, 0.f);
                    pair_term<DIM>(d4, 0.f, 0.f, 0.f, h.w, cexp, qpow, R);
                }
                if (lg == 0) {  // own representative (Q25): into C, i.e. subtracted
                    const int32_t hv = __ldg(a.anc + i);
                    const float4 h = sm[hv], l = sm[a.k + hv];
                    const float4 d4 = make_float4((xi.x - h.x) - l.x, (xi.y - h.y) - l.y, (xi.z - h.z) - l.z, 0.f);
                    pair_term<DIM>(d4, 0.f, 0.f, 0.f, h.w, cexp, qpow, C);
                }
                const int32_t p = __ldg(a.parent + i);
                const int32_t c1 = __ldg(a.cptr + p + 1);
                for (int32_t c = __ldg(a.cptr + p) + lg; c < c1; c += G) {  // siblings under P(i)
                    const int32_t j = __ldg(a.child + c);
                    if (j == i) continue;
                    const float4 xj = load_xc<DIM>(xin, j);
                    pair_term<DIM>(xi, xj.x, xj.y, xj.z, 1.f, cexp, qpow, R);
                }
            } else {
                for (int32_t j = lg; j < a.n; j += G) {
                    const float4 sv = sm[j];
                    pair_term<DIM>(xi, sv.x, sv.y, sv.z, 1.f, cexp, qpow, R);  // j = i: dx = 0 -> 0
                }
            }
            // S_i: attraction, S-pair r-values (subtracted), stress
            float rho = 0.f, st = 0.f;
            const int64_t e0 = __ldg(a.rp + i), e1 = __ldg(a.rp + i + 1);
            for (int64_t e = e0 + lg; e < e1; e += G) {
                const int32_t j = __ldg(a.col + e);
                const float dd = __ldg(a.d + e), ww = __ldg(a.w + e);
                const float4 xj = load_xc<DIM>(xin, j);
                const float dx = xi.x - xj.x, dy = xi.y - xj.y;
                float r2 = fmaf(dx, dx, kEps2);
                r2 = fmaf(dy, dy, r2);
                float dz = 0.f;
                if constexpr (DIM == 3) {
                    dz = xi.z - xj.z;
                    r2 = fmaf(dz, dz, r2);
                }
                const float inv = qpow ? inv_pow<true>(r2, cexp) : inv_pow<false>(r2, cexp);
                C.x = fmaf(dx, inv, C.x);
                C.y = fmaf(dy, inv, C.y);
                if constexpr (DIM == 3) C.z = fmaf(dz, inv, C.z);
                const float rinv = rsqrt_approx(r2);
                const float dist = r2 * rinv;
                const float sc = dd * rinv;
                rho += ww;
                A.x = fmaf(ww, fmaf(sc, dx, xj.x), A.x);
                A.y = fmaf(ww, fmaf(sc, dy, xj.y), A.y);
                if constexpr (DIM == 3) A.z = fmaf(ww, fmaf(sc, dz, xj.z), A.z);
                const float dev = dist - dd;
                st = fmaf(ww * dev, dev, st);
            }
#pragma unroll
            for (int o = G / 2; o > 0; o >>= 1) {
                R.x += __shfl_xor_sync(0xffffffffu, R.x, o, G);
                R.y += __shfl_xor_sync(0xffffffffu, R.y, o, G);
                C.x += __shfl_xor_sync(0xffffffffu, C.x, o, G);
                C.y += __shfl_xor_sync(0xffffffffu, C.y, o, G);
                A.x += __shfl_xor_sync(0xffffffffu, A.x, o, G);
                A.y += __shfl_xor_sync(0xffffffffu, A.y, o, G);
                rho += __shfl_xor_sync(0xffffffffu, rho, o, G);
                st += __shfl_xor_sync(0xffffffffu, st, o, G);
                if constexpr (DIM == 3) {
                    R.z += __shfl_xor_sync(0xffffffffu, R.z, o, G);
                    C.z += __shfl_xor_sync(0xffffffffu, C.z, o, G);
                    A.z += __shfl_xor_sync(0xffffffffu, A.z, o, G);
                }
            }
            if (lg == 0 && valid) {
                R.x -= C.x;
                R.y -= C.y;
                R.z -= C.z;
                float4 xn;
                xn.x = fmaf(alpha_f, R.x, A.x) / rho;
                xn.y = fmaf(alpha_f, R.y, A.y) / rho;
                xn.z = (DIM == 3) ? fmaf(alpha_f, R.z, A.z) / rho : 0.f;
                xn.w = 0.f;
                store_x<DIM>(xout, i, xn);
                if (!(isfinite(xn.x) && isfinite(xn.y) && isfinite(xn.z))) bad = 1;
                const double ex = (double)xn.x - xi.x, ey = (double)xn.y - xi.y, ez = (double)xn.z - xi.z;
                v_dx2 += ex * ex + ey * ey + ez * ez;
                v_x2 += (double)xi.x * xi.x + (double)xi.y * xi.y + (double)xi.z * xi.z;
                v_st += (double)st;
            }
        }
        // ---- per-CTA partials (fixed order), then every CTA reduces all of them
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            v_dx2 += __shfl_xor_sync(0xffffffffu, v_dx2, o);
            v_x2 += __shfl_xor_sync(0xffffffffu, v_x2, o);
            v_st += __shfl_xor_sync(0xffffffffu, v_st, o);
        }
        bad = __reduce_or_sync(0xffffffffu, bad);
        if (lane == 0) {
            red[0][warp] = v_dx2;
            red[1][warp] = v_x2;
            red[2][warp] = v_st;
            red[3][warp] = (double)bad;
        }
        __syncthreads();
        // partials double-buffered by sweep parity: a CTA that runs ahead into the
        // next sweep cannot overwrite what a slower CTA is still summing
        double* part = a.partial + (int64_t)(count & 1) * NB * 4;
        if (tid < 4) {
            double s = 0.0;
            for (int w = 0; w < kSmallBlock / 32; ++w) s = (tid == 3) ? fmax(s, red[3][w]) : s + red[tid][w];
            part[(int64_t)blockIdx.x * 4 + tid] = s;
        }
        grid_barrier(NB);
        // warp 0 sums the CTA partials (lane l: CTAs l, l+32, ..., then a fixed
        // xor tree): the same order in every CTA; broadcast via shared memory
        __shared__ double s_tot[4];
        if (warp == 0) {
            double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
            for (unsigned b = lane; b < NB; b += 32) {
                const double2 u = __ldcg(reinterpret_cast<const double2*>(part + (int64_t)b * 4));
                const double2 v = __ldcg(reinterpret_cast<const double2*>(part + (int64_t)b * 4 + 2));
                t0 += u.x;
                t1 += u.y;
                t2 += v.x;
                t3 = fmax(t3, v.y);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                t0 += __shfl_xor_sync(0xffffffffu, t0, o);
                t1 += __shfl_xor_sync(0xffffffffu, t1, o);
                t2 += __shfl_xor_sync(0xffffffffu, t2, o);
                t3 = fmax(t3, __shfl_xor_sync(0xffffffffu, t3, o));
            }
            if (lane == 0) {
                s_tot[0] = t0;
                s_tot[1] = t1;
                s_tot[2] = t2;
                s_tot[3] = t3;
            }
        }
        __syncthreads();
        const double tot[4] = {s_tot[0], s_tot[1], s_tot[2], s_tot[3]};
        ++count;
        last[0] = tot[0];
        last[1] = tot[1];
        last[2] = tot[2];
        const float* t = xin;
        xin = xout;
        xout = const_cast<float*>(t);
        bool done;
        if (tot[3] != 0.0) {
            err = 1;
            done = true;
        } else if (a.mode == 0) {
            done = count >= a.K;
        } else {
            const double rel = tot[1] > 0 ? sqrt(tot[0]) / sqrt(tot[1]) : INFINITY;
            ++it;
            done = false;
            if (rel < a.eps || it >= max_it) {
                if (fin) {
                    done = true;
                } else {
                    alpha = fmax(alpha * a.factor, a.alpha_min);
                    it = 0;
                    fin = alpha <= a.alpha_min;
                    max_it = fin ? a.max_final : a.rounds;
                }
            }
        }
        if (done) break;
        // no barrier here: x_out of this sweep is complete (barrier above), the
        // shared-memory sources are per-CTA, the partials alternate buffers, and
        // the next sweep's writes to the other coordinate buffer come after every
        // CTA has passed the barrier above (it was this sweep's input)
        __syncthreads();
    }
    if (blockIdx.x == 0 && tid == 0) {
        a.result[0] = count;
        a.result[1] = err;
        a.result[2] = (count & 1) ? 1 : 0;  // 1: the result is in x1
        if (a.stats) {
            a.stats->dx2 = last[0];
            a.stats->x2 = last[1];
            a.stats->stress = 0.5 * last[2];
            a.stats->flags = err;
            a.stats->pad = 0;
        }
    }
}

template <int DIM, bool APPROX, int G>
cudaError_t launch_small_t(const SmallArgs& a, int grid, size_t smem, cudaStream_t st) {
    auto* fn = k_small_level<DIM, APPROX, G>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    SmallArgs args = a;
    void* params[] = {&args};
    return cudaLaunchCooperativeKernel((const void*)fn, dim3(grid), dim3(kSmallBlock), params, smem, st);
}

}  // namespace

size_t small_level_smem(int dim, int32_t n, int32_t k, bool approx) {
    (void)dim;
    return approx ? (size_t)k * 2 * sizeof(float4) : (size_t)n * sizeof(float4);
}

int small_level_grid(int32_t n) {
    static const int sms = [] {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
        return v;
    }();
    const int need = (int)((n + kSmallBlock / 32 - 1) / (kSmallBlock / 32));  // >= one warp per target
    return std::max(1, std::min(need, sms));
}

bool small_level_ok(int dim, int32_t n, int32_t k, bool approx) {
    // measured crossover with the tiled path (profiles/README.md): ~25-40K targets
    static const int64_t max_n = [] {
        const char* e = getenv("MM_SMALL_N");  // 0 disables the persistent small-level path
        return e ? (int64_t)atoll(e) : (int64_t)32768;
    }();
    if (max_n <= 0 || n > max_n) return false;
    if (!approx && n > 4096) return false;                    // all n sources in shared memory
    if (approx && k > 3072) return false;                     // 2 k float4 in shared memory
    return small_level_smem(dim, n, k, approx) <= 100 * 1024;
}

cudaError_t launch_small_level(int dim, bool approx, const SmallArgs& a, cudaStream_t st) {
    const int grid = small_level_grid(a.n);
    const size_t smem = small_level_smem(dim, a.n, a.k, approx);
    LaunchScope ls("small_level", st);
    // lanes per target: one or two targets per group per sweep
    const int64_t lanes = (int64_t)grid * kSmallBlock;
    const int G = (a.n * 32 <= 2 * lanes) ? 32 : (a.n * 16 <= 2 * lanes) ? 16 : 8;
#define MM_S(D, AP)                                                              \
    switch (G) {                                                                 \
        case 32: return launch_small_t<D, AP, 32>(a, grid, smem, st);            \
        case 16: return launch_small_t<D, AP, 16>(a, grid, smem, st);            \
        default: return launch_small_t<D, AP, 8>(a, grid, smem, st);            \
    }
    if (dim == 2) {
        if (approx) { MM_S(2, true) } else { MM_S(2, false) }
    } else {
        if (approx) { MM_S(3, true) } else { MM_S(3, false) }
    }
#undef MM_S
}

int small_level_partials(int32_t n) { return 2 * small_level_grid(n); }

}  // namespace mm
