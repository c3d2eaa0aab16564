// k_gather.cu — kernel (a): S_i gather + position update, with the fused
// convergence/stress reduction (e); and the S-part of mm_energy.
//
// For every vertex i (Eq.(2); Eq.(3)):
//   rho_i = sum_{j in S_i} w_ij
//   A_i   = sum_{j in S_i} w_ij (x_j + d_ij (x_i - x_j)/|x_i - x_j|)
//   C_i   = sum_{j in S_i} r(i,j)            (removed from the all-pairs /
//                                             representative sum: "subtracts
//                                             values of r for {u,v} in E that
//                                             have been added in good faith")
//   Sib_i = sum_{j != i, P(j) = P(i)} r(i,j)  (Eq.(3) same-cluster term; approx only)
//   R_i   = sum_p part[p][i] + Sib_i - C_i     (fixed order p = 0..P-1)
//   x'_i  = (A_i + alpha R_i) / rho_i
// with r(i,j) = (x_i - x_j)/|x_i - x_j|^(q+2) evaluated with exactly the same
// FP32 operation sequence as kernels (b)/(c) so that the S-pair terms cancel
// to rounding.  Synchronous (Jacobi): reads x, writes x_out.
//
// Mapping: a group of G lanes (G in {4,8,16,32}, chosen from the mean row
// length) owns one vertex; lanes stride the CSR row so the col/d/w loads of a
// group are contiguous; neighbour coordinates are 8/16-byte gathers (L2
// resident for every config: x is at most 32 MB).  Group results are combined
// with shuffles; per-CTA FP64 partials of |x'-x|^2, |x|^2 and the stress are
// written for a fixed-order final reduction (relative change).
#include "k_repulse.cuh"

namespace mm {

namespace {

constexpr int kGBlock = 256;

template <int G>
__device__ __forceinline__ float group_sum(float v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, G);
    return v;
}

template <int DIM, bool QPOW>
__device__ __forceinline__ void r_value(const float4& xi, const float4& xj, float cexp, float4& acc, float sgn) {
    const float dx = xi.x - xj.x, dy = xi.y - xj.y;
    float r2 = fmaf(dx, dx, kEps2);
    r2 = fmaf(dy, dy, r2);
    float dz = 0.f;
    if constexpr (DIM == 3) {
        dz = xi.z - xj.z;
        r2 = fmaf(dz, dz, r2);
    }
    const float inv = inv_pow<QPOW>(r2, cexp) * sgn;
    acc.x = fmaf(dx, inv, acc.x);
    acc.y = fmaf(dy, inv, acc.y);
    if constexpr (DIM == 3) acc.z = fmaf(dz, inv, acc.z);
}

#ifndef MM_GATHER_MINB
#define MM_GATHER_MINB 4
#endif
#ifndef MM_GATHER_PREFETCH
#define MM_GATHER_PREFETCH 1  // first-level indices of the next vertex loaded one iteration ahead
#endif
#ifndef MM_GATHER_UNROLL
#define MM_GATHER_UNROLL 4
#endif
constexpr int kGatherUnroll = MM_GATHER_UNROLL;
#ifndef MM_GATHER_SLOAD
#define MM_GATHER_SLOAD 1  // S rows through the normal (L2-retaining) path; 0: evict-first streaming (measured slower: cfg5 0.105 vs 0.093 ms, cfg3 0.036 vs 0.031 ms; tools/gpu_session89.sh)
#endif
#ifndef MM_GATHER_CHUNK
#define MM_GATHER_CHUNK 0  // > 0: one-lane-per-vertex rows in two-phase chunks of this many entries
#endif
#ifndef MM_GATHER_UNROLL_G1
#define MM_GATHER_UNROLL_G1 2  // one lane per vertex (short rows, e.g. cfg5's 6): unroll 2 measured +10% there (tools/gpu_session87.sh)
#endif
// fixed-order block reduction of (dx2, x2, stress); the last CTA to finish
// reduces the per-CTA partials in CTA order and re-arms the ticket and flags
__device__ __forceinline__ void gather_finish_stats(const GatherArgs& a, double v_dx2, double v_x2, double v_st) {
    __shared__ double red[3][kGBlock / 32];
    __shared__ bool last;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v_dx2 += __shfl_xor_sync(0xffffffffu, v_dx2, o);
        v_x2 += __shfl_xor_sync(0xffffffffu, v_x2, o);
        v_st += __shfl_xor_sync(0xffffffffu, v_st, o);
    }
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = v_dx2;
        red[1][threadIdx.x >> 5] = v_x2;
        red[2][threadIdx.x >> 5] = v_st;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        double s = 0.0;
        for (int w = 0; w < kGBlock / 32; ++w) s += red[threadIdx.x][w];
        a.stat_partial[(int64_t)blockIdx.x * 3 + threadIdx.x] = s;
        __threadfence();  // each writer publishes its own partial before the ticket
    }
    __syncthreads();
    // last CTA to finish reduces the per-CTA partials in CTA order (the order
    // does not depend on which CTA is last) and re-arms the ticket and flags
    if (threadIdx.x == 0) last = atomicAdd(a.ticket, 1) == (int)gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    double t[3] = {0.0, 0.0, 0.0};
    for (int b = threadIdx.x; b < (int)gridDim.x; b += kGBlock)
        for (int k = 0; k < 3; ++k) t[k] += __ldcg(a.stat_partial + (int64_t)b * 3 + k);
    for (int k = 0; k < 3; ++k) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t[k] += __shfl_xor_sync(0xffffffffu, t[k], o);
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0)
        for (int k = 0; k < 3; ++k) red[k][threadIdx.x >> 5] = t[k];
    __syncthreads();
    if (threadIdx.x == 0) {
        double tot[3] = {0.0, 0.0, 0.0};
        for (int w = 0; w < kGBlock / 32; ++w)
            for (int k = 0; k < 3; ++k) tot[k] += red[k][w];
        const int32_t fl = atomicExch(a.flags, 0);
        if (a.stats) {
            a.stats->dx2 = tot[0];
            a.stats->x2 = tot[1];
            a.stats->stress = 0.5 * tot[2];
            a.stats->flags = fl;
            a.stats->pad = 0;
        }
        *a.ticket = 0;
    }
}

template <int DIM, bool QPOW, int G>
__global__ void __launch_bounds__(kGBlock, MM_GATHER_MINB) k_gather(GatherArgs a, float cexp) {
    if (a.alpha_dev) a.alpha = (float)*a.alpha_dev;  // same rounding as the host path's (float)alpha
    const int lg = threadIdx.x & (G - 1);
    constexpr int VPB = kGBlock / G;  // vertices per block iteration
    double v_dx2 = 0.0, v_x2 = 0.0, v_st = 0.0;
    // software pipeline over the grid-stride loop: the row bounds and the
    // map entries of the NEXT vertex are loaded while this one is processed,
    // which takes one level off each dependent chain (rp -> col -> x[col],
    // parent -> child_ptr -> child -> x, anc -> rpos -> rep, tpos -> partials)
    int64_t nx_e0 = 0, nx_e1 = 0;
    int32_t nx_tp = 0, nx_par = 0, nx_anc = 0, nx_sib = -1;
    auto prefetch = [&](int64_t vb2) {
        const int64_t i2 = vb2 + threadIdx.x / G;
        if (MM_GATHER_PREFETCH && i2 < a.n) {
            nx_e0 = a.rp[i2];
            nx_e1 = a.rp[i2 + 1];
            if (a.tpos != nullptr) nx_tp = __ldg(a.tpos + i2);
            if (a.sib != nullptr) nx_sib = __ldg(a.sib + i2);
            else if (a.parent != nullptr) nx_par = __ldg(a.parent + i2);
            if (a.anc != nullptr) nx_anc = __ldg(a.anc + i2);
        }
    };
    prefetch((int64_t)blockIdx.x * VPB);
    // grid-stride over vertex chunks: a fixed number of CTAs -> a fixed,
    // small number of FP64 partials, each accumulated in a fixed order
    for (int64_t vb = (int64_t)blockIdx.x * VPB; vb < a.n; vb += (int64_t)gridDim.x * VPB) {
        const int64_t i = vb + threadIdx.x / G;
        const bool valid = i < a.n;
        const int64_t cur_e0 = nx_e0, cur_e1 = nx_e1;
        const int32_t cur_tp = nx_tp, cur_par = nx_par, cur_anc = nx_anc, cur_sib = nx_sib;
        prefetch(vb + (int64_t)gridDim.x * VPB);
        float4 xi = make_float4(0.f, 0.f, 0.f, 0.f);
        float rho = 0.f, st = 0.f;
        float4 A = make_float4(0.f, 0.f, 0.f, 0.f), C = A;
        float4 R = make_float4(0.f, 0.f, 0.f, 0.f);
        if (valid) {
            xi = load_x<DIM>(a.x, i);
            {
                // repulsion partials of this vertex (static schedule slots), fetched
                // first so that their latency overlaps the S-row loads; the slots
                // and j-side rows are split over the group's lanes (lane lg takes
                // every G-th, in increasing order) and combined by the group sum below
                const int stride = DIM == 2 ? 2 : 4;
                // kernel (c) processes targets by slot (spatial order, Q27): the slot
                // count follows the slot's block; the partials sit at the vertex id
                const int64_t pi = a.tpos != nullptr ? (int64_t)(MM_GATHER_PREFETCH ? cur_tp : __ldg(a.tpos + i)) : i;
                const int64_t tb = (int32_t)pi / a.tpb;  // pi < n < 2^31: 32-bit division
                const int32_t nslot =
                    a.jpart ? sched_first_cta_tri(tri_prefix((int32_t)tb + 1, a.tri) - 1, a.tri) -
                                  sched_first_cta_tri(tri_prefix((int32_t)tb, a.tri), a.tri) + 1
                            : sched_first_cta((tb + 1) * a.sch.Ub - 1, a.sch) -
                                  sched_first_cta(tb * a.sch.Ub, a.sch) + 1;
                for (int p = lg; p < nslot; p += G) {
                    const float4 v = load_x<DIM>(a.part + (int64_t)p * a.n * stride, i);
                    R.x += v.x;
                    R.y += v.y;
                    R.z += v.z;
                }
                // symmetric mode: j-side sums of the block pairs (I, tb), I < tb
                if (a.jpart) {
                    for (int64_t I = lg; I < tb; I += G) {
                        const float4 v = load_x<DIM>(a.jpart + I * a.n * stride, i);
                        R.x += v.x;
                        R.y += v.y;
                        R.z += v.z;
                    }
                }
            }
            // row i: 64-bit base, 32-bit offsets; the S arrays are read once per
            // sweep through the normal cached path (what fits of them stays in
            // the 126 MB L2 for the next sweep: cfg3's 60 MB, most of cfg5's 150 MB)
            const int64_t e0 = MM_GATHER_PREFETCH ? cur_e0 : a.rp[i];
            const int len = (int)((MM_GATHER_PREFETCH ? cur_e1 : a.rp[i + 1]) - e0);
            const int32_t* __restrict__ colr = a.col + e0;
            const float* __restrict__ dr = a.d + e0;
            const float* __restrict__ wr = a.w + e0;
            // one S entry: the S-pair r-value (removed from the all-pairs / representative
            // sum) and the attraction term
            auto s_entry = [&](const float4& xj, float dd, float ww) {
                const float dx = xi.x - xj.x, dy = xi.y - xj.y;
                float r2 = fmaf(dx, dx, kEps2);
                r2 = fmaf(dy, dy, r2);
                float dz = 0.f;
                if constexpr (DIM == 3) {
                    dz = xi.z - xj.z;
                    r2 = fmaf(dz, dz, r2);
                }
                const float inv = inv_pow<QPOW>(r2, cexp);
                C.x = fmaf(dx, inv, C.x);
                C.y = fmaf(dy, inv, C.y);
                if constexpr (DIM == 3) C.z = fmaf(dz, inv, C.z);
                // attraction: w (x_j + d (x_i - x_j)/|x_i - x_j|)
                const float rinv = rsqrt_approx(r2);
                const float dist = r2 * rinv;
                const float s = dd * rinv;
                rho += ww;
                A.x = fmaf(ww, fmaf(s, dx, xj.x), A.x);
                A.y = fmaf(ww, fmaf(s, dy, xj.y), A.y);
                if constexpr (DIM == 3) A.z = fmaf(ww, fmaf(s, dz, xj.z), A.z);
                const float dev = dist - dd;
                st = fmaf(ww * dev, dev, st);
            };
            if constexpr (G == 1 && MM_GATHER_CHUNK > 0) {
                // one lane per vertex (short rows): chunks of MM_GATHER_CHUNK entries in two
                // phases (all index / d / w loads, then all coordinate gathers), so a row of
                // <= CHUNK entries costs one round trip per level of the col -> x[col] chain.
                // Slots past the row end are the pair (i, i) with w = d = 0: they add exact
                // zeros (0 * rcp(eps) = 0), so the sums equal the entry-by-entry loop's bit for bit.
                constexpr int CH = MM_GATHER_CHUNK;
                for (int k0 = 0; k0 < len; k0 += CH) {
                    int32_t jj[CH];
                    float dd[CH], ww[CH];
#pragma unroll
                    for (int u = 0; u < CH; ++u) {
                        const bool in = k0 + u < len;
                        jj[u] = in ? __ldg(colr + k0 + u) : (int32_t)i;
                        dd[u] = in ? __ldg(dr + k0 + u) : 0.f;
                        ww[u] = in ? __ldg(wr + k0 + u) : 0.f;
                    }
                    float4 xj[CH];
#pragma unroll
                    for (int u = 0; u < CH; ++u) xj[u] = load_x<DIM>(a.x, jj[u]);
#pragma unroll
                    for (int u = 0; u < CH; ++u) s_entry(xj[u], dd[u], ww[u]);
                }
            } else {
                constexpr int kUnr = G == 1 ? MM_GATHER_UNROLL_G1 : kGatherUnroll;
#pragma unroll kUnr
                for (int k = lg; k < len; k += G) {
#if MM_GATHER_SLOAD
                    const int32_t j = __ldg(colr + k);
                    const float dd = __ldg(dr + k), ww = __ldg(wr + k);
#else
                    const int32_t j = __ldcs(colr + k);
                    const float dd = __ldcs(dr + k), ww = __ldcs(wr + k);
#endif
                    s_entry(load_x<DIM>(a.x, j), dd, ww);
                }
            }
            if (a.anc != nullptr && lg == 0) {
                // Eq.(3) excludes the own representative H(i); kernel (c)
                // summed all k, so its term goes into C (subtracted), computed with
                // kernel (c)'s hi/lo differencing (Q25)
                int32_t h = MM_GATHER_PREFETCH ? cur_anc : __ldg(a.anc + i);
                if (a.rpos != nullptr) h = __ldg(a.rpos + h);
                const float4 rh = __ldg(a.rep_hi + h), rl = __ldg(a.rep_lo + h);
                const float4 fr = a.frame != nullptr ? __ldg(a.frame) : make_float4(0.f, 0.f, 0.f, 0.f);
                const float dx = ((xi.x - fr.x) - rh.x) - rl.x, dy = ((xi.y - fr.y) - rh.y) - rl.y;
                float r2 = fmaf(dx, dx, kEps2);
                r2 = fmaf(dy, dy, r2);
                float dz = 0.f;
                if constexpr (DIM == 3) {
                    dz = ((xi.z - fr.z) - rh.z) - rl.z;
                    r2 = fmaf(dz, dz, r2);
                }
                const float inv = inv_pow<QPOW>(r2, cexp) * rh.w;
                C.x = fmaf(dx, inv, C.x);
                C.y = fmaf(dy, inv, C.y);
                if constexpr (DIM == 3) C.z = fmaf(dz, inv, C.z);
            }
            int32_t sb = -2;
            if (a.sib != nullptr) {
                sb = MM_GATHER_PREFETCH ? cur_sib : __ldg(a.sib + i);
                // the only sibling (matching hierarchies): one term, as the child walk below
                if (sb >= 0 && lg == 0) r_value<DIM, QPOW>(xi, load_x<DIM>(a.x, sb), cexp, C, -1.f);
            }
            if (a.parent != nullptr && sb == -2) {  // Eq.(3): same-cluster exact r-values (added: sign -1 on C)
                const int32_t p = (MM_GATHER_PREFETCH && a.sib == nullptr) ? cur_par : __ldg(a.parent + i);
                const int32_t c0 = __ldg(a.child_ptr + p), c1 = __ldg(a.child_ptr + p + 1);
                for (int32_t c = c0 + lg; c < c1; c += G) {
                    const int32_t j = __ldg(a.child + c);
                    if (j != i) r_value<DIM, QPOW>(xi, load_x<DIM>(a.x, j), cexp, C, -1.f);
                }
            }
        }
        // all lanes of the warp take part in the shuffles
        rho = group_sum<G>(rho);
        st = group_sum<G>(st);
        A.x = group_sum<G>(A.x);
        A.y = group_sum<G>(A.y);
        C.x = group_sum<G>(C.x);
        C.y = group_sum<G>(C.y);
        R.x = group_sum<G>(R.x);
        R.y = group_sum<G>(R.y);
        if constexpr (DIM == 3) {
            A.z = group_sum<G>(A.z);
            C.z = group_sum<G>(C.z);
            R.z = group_sum<G>(R.z);
        }
        if (valid && lg == 0) {
            R.x -= C.x;
            R.y -= C.y;
            R.z -= C.z;
            float4 xn;
            xn.x = fmaf(a.alpha, R.x, A.x) / rho;
            xn.y = fmaf(a.alpha, R.y, A.y) / rho;
            xn.z = (DIM == 3) ? fmaf(a.alpha, R.z, A.z) / rho : 0.f;
            xn.w = 0.f;
            store_x<DIM>(a.x_out, i, xn);
            const bool fin = isfinite(xn.x) && isfinite(xn.y) && isfinite(xn.z);
            if (!fin) atomicOr(a.flags, 1);
            const double ex = (double)xn.x - xi.x, ey = (double)xn.y - xi.y, ez = (double)xn.z - xi.z;
            v_dx2 += ex * ex + ey * ey + ez * ez;
            v_x2 += (double)xi.x * xi.x + (double)xi.y * xi.y + (double)xi.z * xi.z;
            v_st += (double)st;
        }
    }
    gather_finish_stats(a, v_dx2, v_x2, v_st);
}

__global__ void k_stats_final(const double* __restrict__ partial, int nblocks, const int32_t* __restrict__ flags,
                              mm_sweep_stats* __restrict__ out) {
    __shared__ double red[3][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;  // 1 block of 1024 threads
    double s[3] = {0.0, 0.0, 0.0};
    for (int b = threadIdx.x; b < nblocks; b += blockDim.x)
        for (int k = 0; k < 3; ++k) s[k] += partial[(int64_t)b * 3 + k];
    for (int k = 0; k < 3; ++k) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s[k] += __shfl_xor_sync(0xffffffffu, s[k], o);
        if (lane == 0) red[k][wid] = s[k];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t[3] = {0.0, 0.0, 0.0};
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
            for (int k = 0; k < 3; ++k) t[k] += red[k][w];
        out->dx2 = t[0];
        out->x2 = t[1];
        out->stress = 0.5 * t[2];
        out->flags = *flags;
        out->pad = 0;
    }
}

// S part of mm_energy: per row, stress_i and sum_{j in S_i} of the same
// per-pair transform as k_entropy_all (so the subtraction is consistent).
template <int DIM, bool QPOW, int G>
__global__ void __launch_bounds__(kGBlock) k_energy_s(int32_t n, const int64_t* __restrict__ rp,
                                                      const int32_t* __restrict__ col, const float* __restrict__ d,
                                                      const float* __restrict__ w, const float* __restrict__ x,
                                                      float cq, double* __restrict__ partial,
                                                      int32_t* __restrict__ coinc) {
    const int lg = threadIdx.x & (G - 1);
    constexpr int VPB = kGBlock / G;
    double a0 = 0.0, a1 = 0.0;  // FP64 across vertices, FP32 within a row
    int32_t zc = 0;
    for (int64_t vb = (int64_t)blockIdx.x * VPB; vb < n; vb += (int64_t)gridDim.x * VPB) {
        const int64_t i = vb + threadIdx.x / G;
        if (i >= n) continue;
        float st = 0.f, ph = 0.f;
        const float4 xi = load_x<DIM>(x, i);
        for (int64_t e = rp[i] + lg; e < rp[i + 1]; e += G) {
            const float4 xj = load_x<DIM>(x, __ldg(col + e));
            const float dx = xi.x - xj.x, dy = xi.y - xj.y;
            float r2 = fmaf(dx, dx, 0.f);
            r2 = fmaf(dy, dy, r2);
            if constexpr (DIM == 3) {
                const float dz = xi.z - xj.z;
                r2 = fmaf(dz, dz, r2);
            }
            const float dist = sqrtf(r2);
            const float dev = dist - __ldg(d + e);
            st = fmaf(__ldg(w + e) * dev, dev, st);
            // same per-pair transform as k_entropy_tri; coincident pairs skipped and counted
            if (r2 == 0.f) {
                ++zc;
            } else {
                const float l = lg2_approx(fmaxf(r2, 1e-18f));  // same r^2 floor as k_entropy_tri
                if constexpr (!QPOW) ph += l;
                else ph += ex2_approx(fminf(cq * l, kExpClamp));
            }
        }
        a0 += (double)st;
        a1 += (double)ph;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a0 += __shfl_xor_sync(0xffffffffu, a0, o);
        a1 += __shfl_xor_sync(0xffffffffu, a1, o);
        zc += __shfl_xor_sync(0xffffffffu, zc, o);
    }
    __shared__ double red[2][kGBlock / 32];
    __shared__ int32_t redc[kGBlock / 32];
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = a0;
        red[1][threadIdx.x >> 5] = a1;
        redc[threadIdx.x >> 5] = zc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s0 = 0.0, s1 = 0.0;
        int32_t c = 0;
        for (int k = 0; k < kGBlock / 32; ++k) {
            s0 += red[0][k];
            s1 += red[1][k];
            c += redc[k];
        }
        partial[(int64_t)blockIdx.x * 2] = s0;
        partial[(int64_t)blockIdx.x * 2 + 1] = s1;
        if (c) atomicAdd(coinc, c);
    }
}

int pick_group(double mean_row) {
    static const int forced = [] {
        const char* e = getenv("MM_GATHER_G");  // experiments: 1, 2, 4, 8, 16, 32
        return e ? atoi(e) : 0;
    }();
    if (forced == 1 || forced == 2 || forced == 4 || forced == 8 || forced == 16 || forced == 32) return forced;
    // about 8 row entries per lane: more independent loads in flight per lane
    // beat wider groups (tools/bench_gather.py sweep, profiles/r01_gather_groups.txt)
    int g = 1;
    while (g < 32 && 8.0 * (2 * g) <= mean_row) g *= 2;
    return g;
}

}  // namespace

#ifndef MM_GATHER_SYM_GMIN
#define MM_GATHER_SYM_GMIN 1  // lanes per vertex at least, after the symmetric kernel (b); 4 / 8 / 16 measured slower at cfg2 (tools/gpu_session85.sh)
#endif

static int gather_blocks_g(int32_t n, int G) {
    const int64_t need = ((int64_t)n * G + kGBlock - 1) / kGBlock;
    static const int cap = [] {
        int dev = 0, sms = 148, occ = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_gather<2, false, 8>, kGBlock, 0);
        if (occ <= 0) occ = MM_GATHER_MINB;
        const char* e = getenv("MM_GATHER_WAVES");  // experiments
        const int waves = e ? std::max(1, atoi(e)) : 1;
        return sms * occ * waves;  // one resident wave of grid-stride CTAs (measured best: r01_gather_groups.txt)
    }();
    return (int)std::max<int64_t>(1, std::min<int64_t>(need, cap));
}

int gather_blocks(int32_t n, double mean_row) { return gather_blocks_g(n, pick_group(mean_row)); }

cudaError_t launch_gather(int dim, const GatherArgs& a, double mean_row, cudaStream_t st) {
    int G = pick_group(mean_row);
    // after the symmetric exact kernel a vertex of block b sums b j-side rows
    // (about n / 2048 on average) besides its slots: spread them over more lanes
    if (a.jpart != nullptr) G = std::max(G, MM_GATHER_SYM_GMIN);
    const int nb = gather_blocks_g(a.n, G);
    const float cexp = -(a.q + 2.0f) * 0.5f;
    const bool qpow = a.q != 0.0f;
    LaunchScope ls("gather_update", st);
#define MM_G(D, Q)                                                                  \
    switch (G) {                                                                    \
        case 1: k_gather<D, Q, 1><<<nb, kGBlock, 0, st>>>(a, cexp); break;          \
        case 2: k_gather<D, Q, 2><<<nb, kGBlock, 0, st>>>(a, cexp); break;          \
        case 4: k_gather<D, Q, 4><<<nb, kGBlock, 0, st>>>(a, cexp); break;          \
        case 8: k_gather<D, Q, 8><<<nb, kGBlock, 0, st>>>(a, cexp); break;          \
        case 16: k_gather<D, Q, 16><<<nb, kGBlock, 0, st>>>(a, cexp); break;        \
        default: k_gather<D, Q, 32><<<nb, kGBlock, 0, st>>>(a, cexp); break;        \
    }
    if (dim == 2) {
        if (qpow) { MM_G(2, true) } else { MM_G(2, false) }
    } else {
        if (qpow) { MM_G(3, true) } else { MM_G(3, false) }
    }
#undef MM_G
    return cudaGetLastError();
}

cudaError_t launch_stats_final(const double* partial, int nblocks, const int32_t* flags, mm_sweep_stats* out,
                               cudaStream_t st) {
    LaunchScope ls("stats_final", st);
    k_stats_final<<<1, 1024, 0, st>>>(partial, nblocks, flags, out);
    return cudaGetLastError();
}

cudaError_t launch_energy_s(int dim, double q, int32_t n, const int64_t* rp, const int32_t* col, const float* d,
                            const float* w, const float* x, double mean_row, double* partial, int32_t* coinc,
                            cudaStream_t st) {
    const int G = pick_group(mean_row);
    const int nb = gather_blocks(n, mean_row);
    const float cq = (float)(-q * 0.5);
    const bool qpow = q != 0.0;
    LaunchScope ls("energy_s", st);
#define MM_E(D, Q)                                                                                  \
    switch (G) {                                                                                    \
        case 1: k_energy_s<D, Q, 1><<<nb, kGBlock, 0, st>>>(n, rp, col, d, w, x, cq, partial, coinc); break;   \
        case 2: k_energy_s<D, Q, 2><<<nb, kGBlock, 0, st>>>(n, rp, col, d, w, x, cq, partial, coinc); break;   \
        case 4: k_energy_s<D, Q, 4><<<nb, kGBlock, 0, st>>>(n, rp, col, d, w, x, cq, partial, coinc); break;   \
        case 8: k_energy_s<D, Q, 8><<<nb, kGBlock, 0, st>>>(n, rp, col, d, w, x, cq, partial, coinc); break;   \
        case 16: k_energy_s<D, Q, 16><<<nb, kGBlock, 0, st>>>(n, rp, col, d, w, x, cq, partial, coinc); break; \
        default: k_energy_s<D, Q, 32><<<nb, kGBlock, 0, st>>>(n, rp, col, d, w, x, cq, partial, coinc); break; \
    }
    if (dim == 2) {
        if (qpow) { MM_E(2, true) } else { MM_E(2, false) }
    } else {
        if (qpow) { MM_E(3, true) } else { MM_E(3, false) }
    }
#undef MM_E
    return cudaGetLastError();
}

}  // namespace mm

namespace mm {
namespace {
// S-set validation: per row i, row_ptr monotone, 0 <= col < n, col != i,
// d > 0 finite, w >= 0 finite, rho_i = sum w > 0.  bad[0] = first bad row + 1
// (atomicMin on a 1-based row, 0 = none), bad[1] = OR of the reason bits.
__global__ void k_validate_sset(int32_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                const float* __restrict__ d, const float* __restrict__ w, int64_t nnz,
                                int32_t* __restrict__ bad) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int reason = 0;
    const int64_t b = rp[i], e = rp[i + 1];
    if (b < 0 || e < b || e > nnz) reason |= 1;
    double rho = 0.0;
    if (!(reason & 1)) {
        for (int64_t t = b; t < e; ++t) {
            const int32_t j = col[t];
            if (j < 0 || j >= n) reason |= 2;
            if (j == i) reason |= 4;
            if (!(d[t] > 0.f) || !isfinite(d[t])) reason |= 8;
            if (!(w[t] >= 0.f) || !isfinite(w[t])) reason |= 16;
            rho += w[t];
        }
        if (!(rho > 0.0)) reason |= 32;
    }
    if (reason) {
        atomicMin(bad, i + 1);
        atomicOr(bad + 1, reason);
    }
}
}  // namespace

cudaError_t launch_validate_sset(int32_t n, const int64_t* rp, const int32_t* col, const float* d, const float* w,
                                 int64_t nnz, int32_t* bad, cudaStream_t st) {
    LaunchScope ls("validate_sset", st);
    k_validate_sset<<<(n + 255) / 256, 256, 0, st>>>(n, rp, col, d, w, nnz, bad);
    return cudaGetLastError();
}
}  // namespace mm
