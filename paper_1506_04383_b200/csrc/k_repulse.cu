// k_repulse.cu — kernels (b) exact all-pairs repulsion, (c) coarse-
// representative repulsion, and the all-pairs entropy sum of mm_energy.
//
// (b) computes, for every target i, R_i^all = sum_{j != i} (x_i - x_j)/|x_i - x_j|^(q+2)
//     over ALL vertices (the second term of Eq.(2), with the
//     exponent q of BASELINE.json's north_star).  Kernel (a) afterwards
//     subtracts the S_i pairs, so the net sum runs over j notin S_i.
// (c) computes sum_{v'} nu(v') (x_i - x'_v')/|x_i - x'_v'|^(q+2) over ALL k
//     coarse representatives {x', nu} of the approximation level; kernel (a)
//     subtracts the own representative's term, so the net sum is Eq.(3)'s
//     sum over v' != H(i) (Q25).
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
static_assert(kBlock == kCoarseTile, "tile_nu granularity");
#ifndef MM_T2
#define MM_T2 4  // targets per thread, 2-D (experiments: tools/gvar builds)
#endif
#ifndef MM_T3
#define MM_T3 2
#endif
#ifndef MM_REP_UNR
#define MM_REP_UNR 4
#endif

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

#ifndef MM_COARSE_BMASK_FAST
#define MM_COARSE_BMASK_FAST 1  // batched reciprocals in these target groups of kernel (c)'s no-lo tiles
#endif
constexpr float kFarRel2 = 1.0f / 16384.f;  // Q27: a tile is far from a warp when sep^2 >= (2^-7 X)^2
// 2^y for a packed pair on the FMA and ALU pipes (no MUFU): y = n + f with n the
// nearest integer (round-to-nearest through the 1.5 * 2^23 shifter), 2^f by a
// degree-5 relative-error fit on [-1/2, 1/2] (max error 2.2e-7 in FP32, about
// the 2 ulp of ex2.approx), 2^n added to the exponent field.  y is clamped to
// [-125, 126] (below, ex2.approx.ftz would flush to 0; the difference is < 2^-125).
__device__ __forceinline__ f2x ex2_poly2(f2x y) {
    constexpr float kShift = 12582912.0f;
    float y0, y1;
    upk(y, y0, y1);
    y0 = fminf(fmaxf(y0, -125.f), kExpClamp);
    y1 = fminf(fmaxf(y1, -125.f), kExpClamp);
    const f2x yc = pk(y0, y1);
    const f2x t = add2(yc, pk(kShift, kShift));
    float t0, t1;
    upk(t, t0, t1);
    const f2x tm = add2(t, pk(-kShift, -kShift));
    const f2x f = fma2(tm, pk(-1.f, -1.f), yc);
    f2x p = pk(0.0013266970636323094f, 0.0013266970636323094f);
    p = fma2(p, f, pk(0.009675459936261177f, 0.009675459936261177f));
    p = fma2(p, f, pk(0.05550742521882057f, 0.05550742521882057f));
    p = fma2(p, f, pk(0.24022121727466583f, 0.24022121727466583f));
    p = fma2(p, f, pk(0.6931469440460205f, 0.6931469440460205f));
    p = fma2(p, f, pk(1.0000001192092896f, 1.0000001192092896f));
    float p0, p1;
    upk(p, p0, p1);
    const int n0 = __float_as_int(t0) - 0x4B400000, n1 = __float_as_int(t1) - 0x4B400000;
    return pk(__int_as_float(__float_as_int(p0) + (n0 << 23)), __int_as_float(__float_as_int(p1) + (n1 << 23)));
}

// 2^(c L) for a packed pair of L = lg2 r^2 on the FMA and ALU pipes, with the
// scale c folded into the range reduction (no separate multiply): L is clamped
// to [lmin, lmax] = [126/c, -125/c] (c < 0) so that c L stays in [-125, 126];
// t = c L + 1.5 2^23 rounds c L to the nearest integer n, f = c L - n by one
// FMA (exact product), then the degree-5 fit of ex2_poly2.
// CLAMP = false: the caller guarantees c L <= 126 (r^2 >= kEps2 and
// q <= kQNoClamp), so only the lower bound is applied.
template <bool CLAMP>
__device__ __forceinline__ f2x ex2_poly2_scaled(f2x L, float c, float lmin, float lmax) {
    constexpr float kShift = 12582912.0f;
    float l0, l1;
    upk(L, l0, l1);
    if constexpr (CLAMP) {
        l0 = fmaxf(l0, lmin);
        l1 = fmaxf(l1, lmin);
    }
    l0 = fminf(l0, lmax);
    l1 = fminf(l1, lmax);
    const f2x lc = pk(l0, l1);
    const f2x cc = pk(c, c);
    const f2x t = fma2(lc, cc, pk(kShift, kShift));
    float t0, t1;
    upk(t, t0, t1);
    const f2x nn = fma2(t, pk(-1.f, -1.f), pk(kShift, kShift));  // -n, exact
    const f2x f = fma2(lc, cc, nn);                               // c L - n
    f2x p = pk(0.0013266970636323094f, 0.0013266970636323094f);
    p = fma2(p, f, pk(0.009675459936261177f, 0.009675459936261177f));
    p = fma2(p, f, pk(0.05550742521882057f, 0.05550742521882057f));
    p = fma2(p, f, pk(0.24022121727466583f, 0.24022121727466583f));
    p = fma2(p, f, pk(0.6931469440460205f, 0.6931469440460205f));
    p = fma2(p, f, pk(1.0000001192092896f, 1.0000001192092896f));
    float p0, p1;
    upk(p, p0, p1);
    // (t_bits - 0x4B400000) << 23 == t_bits << 23 (mod 2^32): one LEA per value
    return pk(__int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23)),
              __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23)));
}

#ifndef MM_POLY_FUSED
#define MM_POLY_FUSED 1
#endif

#ifndef MM_POLY_MASK3
#define MM_POLY_MASK3 0x11  // 3-D q > 0: sources 0 and 4 of every 8 take the polynomial 2^y (Q29; measured best of 0x11, 0x25, 0x49, 0x55)
#endif
#ifndef MM_POLY_MASK2
#define MM_POLY_MASK2 0x11  // 2-D q > 0
#endif

// One source (shared-memory slot jj) against the thread's T = 2G targets:
// T* += the pair terms.  PAIR_NU: multiply every pair by its representative's
// mass nu (coarse tiles of mixed mass); otherwise the caller scales the tile
// sum.  LO: difference against the representative as (x_i - hi) - lo (Q24);
// without it (x_i - hi) only, for tiles far from every target of the warp
// (Q27).  POLY (q > 0): 2^y by ex2_poly2 instead of MUFU.EX2 (Q29).
template <int DIM, bool QPOW, bool COARSE, int G, int BMASK, bool PAIR_NU, bool LO, bool POLY, bool CLAMP>
__device__ __forceinline__ void source_pairs(int jj, const float4* sm_a, const float4* sm_b, const f2x (&X)[G],
                                             const f2x (&Y)[G], const f2x (&Z)[G], f2x (&TX)[G], f2x (&TY)[G],
                                             f2x (&TZ)[G], float cexp) {
    const f2x eps2 = pk(kEps2, kEps2);
    const float2* sm2 = reinterpret_cast<const float2*>(sm_a);
    float sx, sy, sz = 0.f, lx = 0.f, ly = 0.f, lz = 0.f, nu = 1.f;
    if constexpr (COARSE) {
        const float4 a = sm_a[jj];
        sx = a.x; sy = a.y; sz = a.z; nu = a.w;
        if constexpr (LO) {
            const float4 b = sm_b[jj];
            lx = b.x; ly = b.y; lz = b.z;
        }
    } else if constexpr (DIM == 2) {
        const float2 a = sm2[jj];
        sx = a.x; sy = a.y;
    } else {
        const float4 a = sm_a[jj];
        sx = a.x; sy = a.y; sz = a.z;
    }
    (void)nu;
    (void)lx; (void)ly; (void)lz;
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
        f2x dx = sub_bc(X[gg], sx);
        f2x dy = sub_bc(Y[gg], sy);
        if constexpr (COARSE && LO) {
            dx = sub_bc(dx, lx);
            dy = sub_bc(dy, ly);
        }
        f2x r2 = fma2(dx, dx, eps2);
        r2 = fma2(dy, dy, r2);
        f2x dz = 0ull;
        if constexpr (DIM == 3) {
            dz = sub_bc(Z[gg], sz);
            if constexpr (COARSE && LO) dz = sub_bc(dz, lz);
            r2 = fma2(dz, dz, r2);
        }
        // groups whose bit is set in BMASK use the batched reciprocal (q = 0)
        f2x inv;
        if constexpr (QPOW && POLY) {
            float r0, r1;
            upk(r2, r0, r1);
            if constexpr (MM_POLY_FUSED != 0)
                inv = ex2_poly2_scaled<CLAMP>(pk(lg2_approx(r0), lg2_approx(r1)), cexp, kExpClamp / cexp,
                                              -125.f / cexp);
            else
                inv = ex2_poly2(mul_bc(pk(lg2_approx(r0), lg2_approx(r1)), cexp));
            if constexpr (PAIR_NU) inv = mul_bc(inv, nu);
        } else if constexpr (QPOW && !CLAMP) {
            // 2^(c lg2 r^2) with c lg2 r^2 <= 126 guaranteed (no clamp); packed scale
            float r0, r1, y0, y1;
            upk(r2, r0, r1);
            upk(mul_bc(pk(lg2_approx(r0), lg2_approx(r1)), cexp), y0, y1);
            inv = pk(ex2_approx(y0), ex2_approx(y1));
            if constexpr (PAIR_NU) inv = mul_bc(inv, nu);
        } else if constexpr (PAIR_NU) {
            // all k representatives, the own one H(i) included: kernel (a)
            // subtracts that term (Q25); nu folded into the
            // batched reciprocal: nu/a = b * (nu * rcp(ab))
            if ((BMASK >> gg) & 1) {
                float r0, r1;
                upk(r2, r0, r1);
                const float ip = nu * rcp_approx(r0 * r1);
                inv = mul_bc(pk(r1, r0), ip);
            } else {
                inv = mul_bc(inv_pair<QPOW, false>(r2, cexp), nu);
            }
        } else {
            inv = ((BMASK >> gg) & 1) ? inv_pair<QPOW, true>(r2, cexp) : inv_pair<QPOW, false>(r2, cexp);
        }
        TX[gg] = fma2(dx, inv, TX[gg]);
        TY[gg] = fma2(dy, inv, TY[gg]);
        if constexpr (DIM == 3) TZ[gg] = fma2(dz, inv, TZ[gg]);
    }
}

// One shared-memory source tile (cnt sources) against the thread's targets.
template <int DIM, bool QPOW, bool COARSE, int G, int BMASK, int UNR, bool PAIR_NU, bool LO, bool CLAMP>
__device__ __forceinline__ void tile_pairs(int cnt, const float4* sm_a, const float4* sm_b, const f2x (&X)[G],
                                           const f2x (&Y)[G], const f2x (&Z)[G], f2x (&TX)[G], f2x (&TY)[G],
                                           f2x (&TZ)[G], float cexp) {
    constexpr int PM = (QPOW && COARSE) ? (DIM == 3 ? MM_POLY_MASK3 : MM_POLY_MASK2) : 0;
    int jj = 0;
    if constexpr (PM != 0) {
        // blocks of 8 sources with a fixed MUFU / polynomial split (Q29)
#define MM_SRC(u) \
    source_pairs<DIM, QPOW, COARSE, G, BMASK, PAIR_NU, LO, ((PM >> (u)) & 1) != 0, CLAMP>(jj + (u), sm_a, sm_b, X, Y, Z, TX, TY, TZ, cexp)
        for (; jj + 8 <= cnt; jj += 8) {
            MM_SRC(0); MM_SRC(1); MM_SRC(2); MM_SRC(3); MM_SRC(4); MM_SRC(5); MM_SRC(6); MM_SRC(7);
        }
#undef MM_SRC
    }
    if constexpr (G == 1 && DIM == 2 && !QPOW && (BMASK & 1)) {
        // one packed target pair per thread: batch the reciprocals of every other
        // SOURCE (instead of every other target group) to keep the FMA / MUFU balance
#pragma unroll 2
        for (; jj + 2 <= cnt; jj += 2) {
            source_pairs<DIM, QPOW, COARSE, G, 1, PAIR_NU, LO, false, CLAMP>(jj, sm_a, sm_b, X, Y, Z, TX, TY, TZ, cexp);
            source_pairs<DIM, QPOW, COARSE, G, 0, PAIR_NU, LO, false, CLAMP>(jj + 1, sm_a, sm_b, X, Y, Z, TX, TY, TZ,
                                                                            cexp);
        }
    }
#pragma unroll UNR
    for (; jj < cnt; ++jj)
        source_pairs<DIM, QPOW, COARSE, G, BMASK, PAIR_NU, LO, false, CLAMP>(jj, sm_a, sm_b, X, Y, Z, TX, TY, TZ, cexp);
}

template <int DIM, bool QPOW, bool COARSE, int T, int BMASK = 1, int MINB = 1, int UNR = 4, bool CLAMP = true>
__global__ void __launch_bounds__(kBlock, MINB) k_repulse(int32_t n_tgt, const float* __restrict__ x, int32_t n_src,
                                                    const float4* __restrict__ rep_hi,
                                                    const float4* __restrict__ rep_lo, CoarseOrder co, float cexp,
                                                    Sched sch, float* __restrict__ part) {
    static_assert(T % 2 == 0, "targets are processed in packed pairs");
    constexpr int G = T / 2;
    constexpr int TPB = kBlock * T;
    constexpr int stride = DIM == 2 ? 2 : 4;
    constexpr int kFastMask = (DIM == 2 && !QPOW) ? MM_COARSE_BMASK_FAST : 0;
    // shared source tile: exact 2-D -> float2; exact 3-D -> float4; coarse -> hi/lo float4 pairs
    __shared__ float4 sm_a[kBlock];
    __shared__ float4 sm_b[COARSE ? kBlock : 1];
    float2* sm2 = reinterpret_cast<float2*>(sm_a);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int32_t g = blockIdx.x;
    const int64_t u0 = (int64_t)g * sch.U / sch.G, u1 = (int64_t)(g + 1) * sch.U / sch.G;
    // target slot of (group gg, half h): each warp owns 32 T consecutive slots
    auto tslot = [&](int64_t base, int gg, int h) -> int64_t {
        return base + (int64_t)warp * (32 * T) + (2 * gg + h) * 32 + lane;
    };

    for (int64_t u = u0; u < u1;) {
        const int32_t tb = (int32_t)(u / sch.Ub);
        const int64_t seg_end = min(u1, (int64_t)(tb + 1) * sch.Ub);
        const int32_t tile0 = (int32_t)(u - (int64_t)tb * sch.Ub), tile1 = (int32_t)(seg_end - (int64_t)tb * sch.Ub);
        // targets of this block (registers), packed pairwise
        f2x X[G], Y[G], Z[G], AX[G], AY[G], AZ[G];
        const int64_t base = (int64_t)tb * TPB;
        float wlo[3] = {INFINITY, INFINITY, INFINITY}, whi[3] = {-INFINITY, -INFINITY, -INFINITY};
        const float4 fr = (COARSE && co.frame != nullptr) ? __ldg(co.frame) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int gg = 0; gg < G; ++gg) {
            const int64_t ia = tslot(base, gg, 0), ib = tslot(base, gg, 1);
            int64_t ca = ia < n_tgt ? ia : n_tgt - 1, cb = ib < n_tgt ? ib : n_tgt - 1;
            if (COARSE && co.tperm != nullptr) {
                ca = __ldg(co.tperm + ca);
                cb = __ldg(co.tperm + cb);
            }
            // scalar loads, so that ptxas can place (x_a, x_b) in one aligned
            // register pair for the whole loop (vector loads would interleave
            // the halves and force MOVs to re-form the pair at every use)
            const float* pa = x + ca * stride;
            const float* pb = x + cb * stride;
            // frame-relative targets: x - c is exact (c chosen by Sterbenz's rule, Q28)
            const float xa = __ldg(pa) - fr.x, xb = __ldg(pb) - fr.x, ya = __ldg(pa + 1) - fr.y,
                        yb = __ldg(pb + 1) - fr.y;
            const float za = DIM == 3 ? __ldg(pa + 2) - fr.z : 0.f, zb = DIM == 3 ? __ldg(pb + 2) - fr.z : 0.f;
            X[gg] = pk(xa, xb);
            Y[gg] = pk(ya, yb);
            Z[gg] = (DIM == 3) ? pk(za, zb) : 0ull;
            AX[gg] = AY[gg] = AZ[gg] = 0ull;
            if constexpr (COARSE) {
                wlo[0] = fminf(wlo[0], fminf(xa, xb));
                whi[0] = fmaxf(whi[0], fmaxf(xa, xb));
                wlo[1] = fminf(wlo[1], fminf(ya, yb));
                whi[1] = fmaxf(whi[1], fmaxf(ya, yb));
                wlo[2] = fminf(wlo[2], fminf(za, zb));
                whi[2] = fmaxf(whi[2], fmaxf(za, zb));
            }
        }
        // the warp's target box (Q27): lo-free tiles need every target of the warp far away
        float wX = 0.f;
        if constexpr (COARSE) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    wlo[c] = fminf(wlo[c], __shfl_xor_sync(0xffffffffu, wlo[c], o));
                    whi[c] = fmaxf(whi[c], __shfl_xor_sync(0xffffffffu, whi[c], o));
                }
                wX = fmaxf(wX, fmaxf(fabsf(wlo[c]), fabsf(whi[c])));
            }
        }
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
            // coarse tiles whose representatives all have the same mass nu
            // (representatives are stored in mass order, Q26) sum
            // (x_i - x')/|x_i - x'|^(q+2) and scale the tile sum by nu once
            const int tnu = (COARSE && co.tile_nu != nullptr) ? __ldg(co.tile_nu + tile) : 0;
            // far tile (Q27): every target of the warp is at least 2^-7 X from the
            // tile's box, so dropping lo perturbs each pair term by < 2^-17 (q+1) relative
            bool far = false;
            if (COARSE && co.tile_box != nullptr) {
                const float4 blo = __ldg(co.tile_box + 2 * tile), bhi = __ldg(co.tile_box + 2 * tile + 1);
                const float sx = fmaxf(0.f, fmaxf(blo.x - whi[0], wlo[0] - bhi.x));
                const float sy = fmaxf(0.f, fmaxf(blo.y - whi[1], wlo[1] - bhi.y));
                const float sz = fmaxf(0.f, fmaxf(blo.z - whi[2], wlo[2] - bhi.z));
                const float XX = fmaxf(wX, blo.w);
                far = sx * sx + sy * sy + sz * sz >= XX * XX * kFarRel2;
            }
            if (tnu > 0) {
                if (far)
                    tile_pairs<DIM, QPOW, COARSE, G, kFastMask, UNR, false, false, CLAMP>(cnt, sm_a, sm_b, X, Y, Z, TX, TY,
                                                                                 TZ, cexp);
                else
                    tile_pairs<DIM, QPOW, COARSE, G, BMASK, UNR, false, COARSE, CLAMP>(cnt, sm_a, sm_b, X, Y, Z, TX, TY, TZ,
                                                                               cexp);
                const f2x nu2 = pk((float)tnu, (float)tnu);
#pragma unroll
                for (int gg = 0; gg < G; ++gg) {
                    AX[gg] = fma2(TX[gg], nu2, AX[gg]);
                    AY[gg] = fma2(TY[gg], nu2, AY[gg]);
                    if constexpr (DIM == 3) AZ[gg] = fma2(TZ[gg], nu2, AZ[gg]);
                }
            } else {
                if (far)
                    tile_pairs<DIM, QPOW, COARSE, G, BMASK, UNR, COARSE, false, CLAMP>(cnt, sm_a, sm_b, X, Y, Z, TX, TY, TZ,
                                                                               cexp);
                else
                    tile_pairs<DIM, QPOW, COARSE, G, BMASK, UNR, COARSE, COARSE, CLAMP>(cnt, sm_a, sm_b, X, Y, Z, TX, TY,
                                                                                TZ, cexp);
#pragma unroll
                for (int gg = 0; gg < G; ++gg) {
                    AX[gg] = add2(AX[gg], TX[gg]);
                    AY[gg] = add2(AY[gg], TY[gg]);
                    if constexpr (DIM == 3) AZ[gg] = add2(AZ[gg], TZ[gg]);
                }
            }
        }
        // partial of this (target block, CTA) pair -> slot g - first CTA of the block
        const int32_t slot = g - sched_first_cta((int64_t)tb * sch.Ub, sch);
        float* out = part + (int64_t)slot * n_tgt * stride;
#pragma unroll
        for (int gg = 0; gg < G; ++gg) {
            const int64_t ia = tslot(base, gg, 0), ib = tslot(base, gg, 1);
            float ax0, ax1, ay0, ay1, az0 = 0.f, az1 = 0.f;
            upk(AX[gg], ax0, ax1);
            upk(AY[gg], ay0, ay1);
            if constexpr (DIM == 3) upk(AZ[gg], az0, az1);
            // stored at the vertex id (spatial order: tperm), so that kernel (a) reads
            // its slots coalesced
            if (ia < n_tgt) store_x<DIM>(out, (COARSE && co.tperm) ? (int64_t)__ldg(co.tperm + ia) : ia,
                                         make_float4(ax0, ay0, az0, 0.f));
            if (ib < n_tgt) store_x<DIM>(out, (COARSE && co.tperm) ? (int64_t)__ldg(co.tperm + ib) : ib,
                                         make_float4(ax1, ay1, az1, 0.f));
        }
        u = seg_end;
    }
}

// ---------------------------------------------------------------------------
// Symmetric exact repulsion (kernel (b), default for exact sweeps): every
// unordered pair is evaluated once and applied to both vertices, using the
// exact FP32 antisymmetry of the pair term (x_j - x_i = -(x_i - x_j) exactly,
// same r^2, same reciprocal).  Blocks of kSymTPB vertices; the work units are
// the block pairs (I, J >= I) of a triangular persistent schedule.
//  * I == J: every ordered pair inside the block on the target side only
//    (the plain loop; the self pair contributes exactly 0).
//  * I <  J: warp w owns 64*SG targets of I (2*SG per lane, in registers); the
//    sources of J are taken 32 at a time, one per lane, and rotated through
//    the lanes in 32 shuffle steps together with their own accumulators, so
//    each lane meets every source of the chunk; after the 32 steps every
//    source's j-side sum (over the warp's targets) is back in its home lane.
//    The warps' j-side sums are added in warp order in shared memory and
//    written to jpart[I][j]; target sums go to ipart[slot][i] as in k_repulse.
// Kernel (a) adds, for vertex i of block B, its i-side slots and jpart[I][i]
// for I < B, in that fixed order: the result is bitwise deterministic.
constexpr int kSymTPB = 1024;  // vertices per block (targets = sources)
#ifndef MM_SYM_BATCH
#define MM_SYM_BATCH 0  // measured: plain reciprocals +2.8% (the symmetric mix is FMA-bound, MUFU 60%)
#endif
constexpr bool kSymBatch = MM_SYM_BATCH != 0;  // batched reciprocal in every other target group

#ifndef MM_SYM_SRC
#define MM_SYM_SRC 256
#endif
constexpr int kSymSrc = MM_SYM_SRC;  // sources per shared-memory sub-tile
template <int DIM>
constexpr int sym_smem_bytes(int warps) {
    return kSymSrc * 16 + warps * kSymSrc * (DIM == 2 ? 2 : 3) * 4;
}

#ifndef MM_SYM_UNR
#define MM_SYM_UNR 8
#endif
constexpr int kSymUnroll = MM_SYM_UNR;
#ifndef MM_SYM_JPACK
#define MM_SYM_JPACK 0  // 1: j-side sums as packed per-step partials (FFMA2); measured 2% slower at cfg2
#endif
constexpr bool kSymJPack = MM_SYM_JPACK != 0;
// one 32-step rotation over a chunk of 32 sources; MASK: the chunk is the
// partial tail of the last block (lanes past the end carry weight 0)
template <int DIM, bool QPOW, int SG, bool MASK>
__device__ __forceinline__ void sym_chunk(const f2x (&X)[SG], const f2x (&Y)[SG], const f2x (&Z)[SG], f2x (&AX)[SG],
                                          f2x (&AY)[SG], f2x (&AZ)[SG], float4 sv, float sw, float cexp, int lane,
                                          float& bx_out, float& by_out, float& bz_out) {
    const f2x eps2 = pk(kEps2, kEps2);
    float sx = sv.x, sy = sv.y, sz = sv.z;
    float bx = 0.f, by = 0.f, bz = 0.f;
    const int nxt = (lane + 1) & 31;
#pragma unroll kSymUnroll
    for (int k = 0; k < 32; ++k) {
        f2x PX = 0ull, PY = 0ull, PZ = 0ull;
        (void)PX; (void)PY; (void)PZ;
#pragma unroll
        for (int gg = 0; gg < SG; ++gg) {
            const f2x dx = sub_bc(X[gg], sx), dy = sub_bc(Y[gg], sy);
            f2x r2 = fma2(dx, dx, eps2);
            r2 = fma2(dy, dy, r2);
            f2x dz = 0ull;
            if constexpr (DIM == 3) {
                dz = sub_bc(Z[gg], sz);
                r2 = fma2(dz, dz, r2);
            }
            f2x inv = (kSymBatch && (gg & 1) == 0) ? inv_pair<QPOW, true>(r2, cexp) : inv_pair<QPOW, false>(r2, cexp);
            if constexpr (MASK) inv = mul2(inv, pk(sw, sw));
            AX[gg] = fma2(dx, inv, AX[gg]);
            AY[gg] = fma2(dy, inv, AY[gg]);
            if constexpr (DIM == 3) AZ[gg] = fma2(dz, inv, AZ[gg]);
            // j side: sum_t (x_j - x_t) inv_t = -sum_t dx_t inv_t
            if constexpr (kSymJPack) {
                // packed per-step partials (one FFMA2 per component and packed pair),
                // folded into the rotating scalar sums after the step
                if (gg == 0) {
                    PX = mul2(dx, inv);
                    PY = mul2(dy, inv);
                    if constexpr (DIM == 3) PZ = mul2(dz, inv);
                } else {
                    PX = fma2(dx, inv, PX);
                    PY = fma2(dy, inv, PY);
                    if constexpr (DIM == 3) PZ = fma2(dz, inv, PZ);
                }
            } else {
                float i0, i1, a0, a1;
                upk(inv, i0, i1);
                upk(dx, a0, a1);
                bx = fmaf(-a0, i0, bx);
                bx = fmaf(-a1, i1, bx);
                upk(dy, a0, a1);
                by = fmaf(-a0, i0, by);
                by = fmaf(-a1, i1, by);
                if constexpr (DIM == 3) {
                    upk(dz, a0, a1);
                    bz = fmaf(-a0, i0, bz);
                    bz = fmaf(-a1, i1, bz);
                }
            }
        }
        if constexpr (kSymJPack) {
            float p0, p1;
            upk(PX, p0, p1);
            bx -= p0 + p1;
            upk(PY, p0, p1);
            by -= p0 + p1;
            if constexpr (DIM == 3) {
                upk(PZ, p0, p1);
                bz -= p0 + p1;
            }
        }
        // rotate the source and its accumulator: lane l takes lane l+1's
        sx = __shfl_sync(0xffffffffu, sx, nxt);
        sy = __shfl_sync(0xffffffffu, sy, nxt);
        bx = __shfl_sync(0xffffffffu, bx, nxt);
        by = __shfl_sync(0xffffffffu, by, nxt);
        if constexpr (DIM == 3) {
            sz = __shfl_sync(0xffffffffu, sz, nxt);
            bz = __shfl_sync(0xffffffffu, bz, nxt);
        }
        if constexpr (MASK) sw = __shfl_sync(0xffffffffu, sw, nxt);
    }
    bx_out = bx;
    by_out = by;
    bz_out = bz;
}

#ifndef MM_SYM_MINB
#define MM_SYM_MINB 6
#endif
template <int DIM, bool QPOW, int SG, int WARPS, int SRC>
__global__ void __launch_bounds__(WARPS * 32, MM_SYM_MINB) k_repulse_sym(int32_t n, const float* __restrict__ x, float cexp,
                                                            TriSched ts, float* __restrict__ ipart,
                                                            float* __restrict__ jpart) {
    static_assert(WARPS * 64 * SG == kSymTPB, "a block is one target set");
    constexpr int NT = WARPS * 32;
    constexpr int stride = DIM == 2 ? 2 : 4;
    constexpr int DC = DIM == 2 ? 2 : 3;
    extern __shared__ float4 sym_smem[];
    float4* src = sym_smem;                                 // [SRC]
    float* jacc = reinterpret_cast<float*>(sym_smem + SRC);  // [WARPS][SRC][DC]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int32_t g = blockIdx.x;
    const int64_t u0 = (int64_t)g * ts.U / ts.G, u1 = (int64_t)(g + 1) * ts.U / ts.G;
    const f2x eps2 = pk(kEps2, kEps2);
    for (int64_t u = u0; u < u1;) {
        int32_t lo = 0, hi = ts.TB - 1;
        while (lo < hi) {
            const int32_t mid = (lo + hi + 1) >> 1;
            if (tri_prefix(mid, ts) <= u) lo = mid; else hi = mid - 1;
        }
        const int32_t I = lo;
        const int64_t pre = tri_prefix(I, ts);
        const int64_t seg_end = min(u1, tri_prefix(I + 1, ts));
        const int64_t ibase = (int64_t)I * kSymTPB;
        // this warp's targets: ibase + warp*64*SG + 32*k + lane, k = 0..2SG-1
        f2x X[SG], Y[SG], Z[SG], AX[SG], AY[SG], AZ[SG];
#pragma unroll
        for (int gg = 0; gg < SG; ++gg) {
            const int64_t ia = ibase + warp * 64 * SG + (2 * gg) * 32 + lane, ib = ia + 32;
            const int64_t ca = ia < n ? ia : n - 1, cb = ib < n ? ib : n - 1;
            const float* pa = x + ca * stride;
            const float* pb = x + cb * stride;
            X[gg] = pk(__ldg(pa), __ldg(pb));
            Y[gg] = pk(__ldg(pa + 1), __ldg(pb + 1));
            Z[gg] = (DIM == 3) ? pk(__ldg(pa + 2), __ldg(pb + 2)) : 0ull;
            AX[gg] = AY[gg] = AZ[gg] = 0ull;
        }
        // units of row I: (J, source sub-tile s) for J = I..TB-1, s = 0..NS-1
        constexpr int NS = kSymTPB / SRC;
        for (; u < seg_end; ++u) {
            const int32_t J = I + (int32_t)((u - pre) / NS);
            const int s0 = (int)((u - pre) % NS) * SRC;
            const int64_t jblk = (int64_t)J * kSymTPB;
            const int jtot = (int)min((int64_t)kSymTPB, (int64_t)n - jblk);
            {
                const int64_t jbase = jblk + s0;
                const int jcnt = min(SRC, jtot - s0);
                if (jcnt <= 0) continue;  // sub-tiles past the end of the last block
                __syncthreads();
                for (int t = tid; t < SRC; t += NT)
                    src[t] = (t < jcnt) ? load_x<DIM>(x, jbase + t) : make_float4(0.f, 0.f, 0.f, 0.f);
                __syncthreads();
                if (J == I) {
                    // diagonal block: all ordered pairs on the target side (self -> 0)
#pragma unroll 4
                    for (int jj = 0; jj < jcnt; ++jj) {
                        const float4 sv = src[jj];
#pragma unroll
                        for (int gg = 0; gg < SG; ++gg) {
                            const f2x dx = sub_bc(X[gg], sv.x), dy = sub_bc(Y[gg], sv.y);
                            f2x r2 = fma2(dx, dx, eps2);
                            r2 = fma2(dy, dy, r2);
                            f2x dz = 0ull;
                            if constexpr (DIM == 3) {
                                dz = sub_bc(Z[gg], sv.z);
                                r2 = fma2(dz, dz, r2);
                            }
                            const f2x inv =
                                (kSymBatch && (gg & 1) == 0) ? inv_pair<QPOW, true>(r2, cexp) : inv_pair<QPOW, false>(r2, cexp);
                            AX[gg] = fma2(dx, inv, AX[gg]);
                            AY[gg] = fma2(dy, inv, AY[gg]);
                            if constexpr (DIM == 3) AZ[gg] = fma2(dz, inv, AZ[gg]);
                        }
                    }
                    continue;
                }
                // off-diagonal (I < J, so block I is full): rotation over 32-source chunks
                const int nfull = jcnt >> 5;
                for (int c = 0; c < nfull; ++c) {
                    float bx, by, bz;
                    sym_chunk<DIM, QPOW, SG, false>(X, Y, Z, AX, AY, AZ, src[c * 32 + lane], 1.f, cexp, lane, bx, by,
                                                    bz);
                    float* jw = jacc + ((int64_t)warp * SRC + c * 32 + lane) * DC;
                    jw[0] = bx;
                    jw[1] = by;
                    if constexpr (DIM == 3) jw[2] = bz;
                }
                if (jcnt & 31) {
                    const int c = nfull;
                    float bx, by, bz;
                    sym_chunk<DIM, QPOW, SG, true>(X, Y, Z, AX, AY, AZ, src[c * 32 + lane],
                                                   (c * 32 + lane) < jcnt ? 1.f : 0.f, cexp, lane, bx, by, bz);
                    float* jw = jacc + ((int64_t)warp * SRC + c * 32 + lane) * DC;
                    jw[0] = bx;
                    jw[1] = by;
                    if constexpr (DIM == 3) jw[2] = bz;
                }
                __syncthreads();
                // j-side partial of block pair (I, J): warps added in warp order
                float* jo = jpart + (int64_t)I * n * stride;
                for (int t = tid; t < jcnt; t += NT) {
                    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                    for (int w = 0; w < WARPS; ++w) {
                        const float* jr = jacc + ((int64_t)w * SRC + t) * DC;
                        v.x += jr[0];
                        v.y += jr[1];
                        if constexpr (DIM == 3) v.z += jr[2];
                    }
                    store_x<DIM>(jo, jbase + t, v);
                }
            }
        }
        // target side of row I handled by this CTA -> slot g - first CTA of the row
        const int32_t slot = g - sched_first_cta_tri(pre, ts);
        float* out = ipart + (int64_t)slot * n * stride;
#pragma unroll
        for (int gg = 0; gg < SG; ++gg) {
            const int64_t ia = ibase + warp * 64 * SG + (2 * gg) * 32 + lane, ib = ia + 32;
            float ax0, ax1, ay0, ay1, az0 = 0.f, az1 = 0.f;
            upk(AX[gg], ax0, ax1);
            upk(AY[gg], ay0, ay1);
            if constexpr (DIM == 3) upk(AZ[gg], az0, az1);
            if (ia < n) store_x<DIM>(out, ia, make_float4(ax0, ay0, az0, 0.f));
            if (ib < n) store_x<DIM>(out, ib, make_float4(ax1, ay1, az1, 0.f));
        }
    }
}

#ifndef MM_SYM_SG
#define MM_SYM_SG 4  // 8 targets per lane, 4 warps per CTA (measured best with plain reciprocals)
#endif
constexpr int kSymSG = MM_SYM_SG;
constexpr int kSymWarps = kSymTPB / (64 * kSymSG);

// All-pairs entropy for mm_energy over UNORDERED pairs i < j (the ordered sum
// of Eq.(1) in the S form is  1/2 sum_{i != j} phi - 1/2 sum_i sum_{S_i} phi
// = sum_{i<j} phi - 1/2 sum_S phi, valid for asymmetric S too):
//   q = 0: sum lg2(r^2), two pairs per MUFU via lg2(a) + lg2(b) = lg2(a b)
//          (phi_0 = -ln r = -(ln 2 / 2) lg2 r^2)
//   q > 0: sum 2^(-q/2 lg2 r^2)      (phi_q = r^-q / q)
// Exactly coincident pairs (r = 0) are skipped and counted.  Triangular
// persistent schedule: target block tb (TPB targets) pairs with source tiles
// from its own first tile on; the unit space is split into G equal ranges and
// every CTA writes one FP64 partial (FP32 within a tile, FP64 across tiles).
constexpr float kR2Floor = 1e-18f;  // r^2 clamp: keeps products of two r^2 normal
constexpr uint32_t kP4Lo = 0x0d800000u;  // 2^-100: bit patterns of the accepted product range
constexpr uint32_t kP4Hi = 0x7e800000u;  // 2^126

template <int DIM>
__device__ __forceinline__ f2x entropy_r2(f2x X, f2x Y, f2x Z, const float4& sv) {
    const f2x dx = sub_bc(X, sv.x), dy = sub_bc(Y, sv.y);
    f2x r2 = mul2(dx, dx);
    r2 = fma2(dy, dy, r2);
    if constexpr (DIM == 3) {
        const f2x dz = sub_bc(Z, sv.z);
        r2 = fma2(dz, dz, r2);
    }
    return r2;
}

// phi-sum contribution of two pairs with (clamped) r^2 = a, b:
// q = 0: lg2(a) + lg2(b) = lg2(a b)  (one MUFU);  q > 0: 2^(cq lg2 a) + 2^(cq lg2 b)
// CLAMP = false: q <= kQNoClampE, where r^2 >= kR2Floor bounds cq lg2 r^2 <= 126
template <bool QPOW, bool CLAMP = true>
__device__ __forceinline__ float entropy_phi2(float a, float b, float cq) {
    if constexpr (!QPOW) {
        return lg2_approx(a * b);
    } else if constexpr (CLAMP) {
        return ex2_approx(fminf(cq * lg2_approx(a), kExpClamp)) + ex2_approx(fminf(cq * lg2_approx(b), kExpClamp));
    } else {
        return ex2_approx(cq * lg2_approx(a)) + ex2_approx(cq * lg2_approx(b));
    }
}

#ifndef MM_ENT_POLY
#define MM_ENT_POLY 1  // q > 0 energy: the second target pair of every other source uses ex2_poly2 (Q29)
#endif
// one source against the thread's 2 x 2 targets (no mask); POLY1: 2^y of group 1 on the FMA pipe
template <int DIM, bool QPOW, bool POLY1, bool CLAMP>
__device__ __forceinline__ void entropy_src(const float4& sv, const f2x (&X)[2], const f2x (&Y)[2],
                                            const f2x (&Z)[2], float cq, float& acc, int32_t& zt) {
#pragma unroll
    for (int gg = 0; gg < 2; ++gg) {
        float ra, rb;
        upk(entropy_r2<DIM>(X[gg], Y[gg], Z[gg], sv), ra, rb);
        zt += (ra == 0.f) + (rb == 0.f);
        ra = fmaxf(ra, kR2Floor);
        rb = fmaxf(rb, kR2Floor);
        if (QPOW && POLY1 && gg == 1) {
            float ea, eb;
            upk(ex2_poly2_scaled<CLAMP>(pk(lg2_approx(ra), lg2_approx(rb)), cq, kExpClamp / cq, -125.f / cq), ea, eb);
            acc += ea + eb;
        } else {
            acc += entropy_phi2<QPOW, CLAMP>(ra, rb, cq);
        }
    }
}

template <int DIM, bool QPOW, bool CLAMP = true>
__global__ void __launch_bounds__(kBlock) k_entropy_tri(int32_t n, const float* __restrict__ x, float cq,
                                                        TriSched ts, double* __restrict__ partial,
                                                        int32_t* __restrict__ coinc) {
    constexpr int T = 4, G = 2, TPB = kBlock * T;
    constexpr int stride = DIM == 2 ? 2 : 4;
    __shared__ float4 sm[kBlock];
    __shared__ double red[kBlock / 32];
    __shared__ int32_t redc[kBlock / 32];
    const int tid = threadIdx.x;
    const int32_t g = blockIdx.x;
    const int64_t u0 = (int64_t)g * ts.U / ts.G, u1 = (int64_t)(g + 1) * ts.U / ts.G;
    double dacc = 0.0;
    int32_t zc = 0;
    for (int64_t u = u0; u < u1;) {
        // target block containing unit u: largest tb with prefix(tb) <= u
        int32_t lo = 0, hi = ts.TB - 1;
        while (lo < hi) {
            const int32_t mid = (lo + hi + 1) >> 1;
            if (tri_prefix(mid, ts) <= u) lo = mid; else hi = mid - 1;
        }
        const int32_t tb = lo;
        const int64_t pre = tri_prefix(tb, ts);
        const int32_t first_tile = tb * (TPB / kBlock);
        const int64_t seg_end = min(u1, tri_prefix(tb + 1, ts));
        const int32_t tile0 = first_tile + (int32_t)(u - pre), tile1 = first_tile + (int32_t)(seg_end - pre);
        const int64_t base = (int64_t)tb * TPB;
        f2x X[G], Y[G], Z[G];
        int32_t ti[T];
#pragma unroll
        for (int gg = 0; gg < G; ++gg) {
            const int64_t ia = base + (2 * gg) * kBlock + tid, ib = base + (2 * gg + 1) * kBlock + tid;
            ti[2 * gg] = (int32_t)ia;
            ti[2 * gg + 1] = (int32_t)ib;
            const int64_t ca = ia < n ? ia : n - 1, cb = ib < n ? ib : n - 1;
            const float* pa = x + ca * stride;
            const float* pb = x + cb * stride;
            X[gg] = pk(__ldg(pa), __ldg(pb));
            Y[gg] = pk(__ldg(pa + 1), __ldg(pb + 1));
            Z[gg] = (DIM == 3) ? pk(__ldg(pa + 2), __ldg(pb + 2)) : 0ull;
        }
        for (int32_t tile = tile0; tile < tile1; ++tile) {
            const int64_t t0 = (int64_t)tile * kBlock;
            const int cnt = (int)min((int64_t)kBlock, (int64_t)n - t0);
            __syncthreads();
            if (tid < cnt) sm[tid] = load_x<DIM>(x, t0 + tid);
            __syncthreads();
            // tiles overlapping the target block need the i < j mask (and targets >= n)
            const bool diag = (t0 < base + TPB) || (base + TPB > n);
            float acc = 0.f;
            int32_t zt = 0;
            if (!diag && !QPOW) {
                // q = 0: lg2 of the product of the four r^2 of one source (one MUFU
                // per 4 pairs) when that product is a normal float in
                // [2^-100, 2^126]; a thread that saw any other product (coincident,
                // tiny or huge r^2) redoes its tile pair by pair (branch-free hot loop)
                bool bad = false;
#pragma unroll 4
                for (int jj = 0; jj < cnt; ++jj) {
                    const float4 sv = sm[jj];
                    const f2x r0 = entropy_r2<DIM>(X[0], Y[0], Z[0], sv), r1 = entropy_r2<DIM>(X[1], Y[1], Z[1], sv);
                    float pa, pb;
                    upk(mul2(r0, r1), pa, pb);
                    const float p4 = pa * pb;
                    const bool ok = (__float_as_uint(p4) - kP4Lo) < (kP4Hi - kP4Lo);
                    const float l = lg2_approx(p4);
                    acc += ok ? l : 0.f;
                    bad |= !ok;
                }
                if (bad) {
                    acc = 0.f;
                    for (int jj = 0; jj < cnt; ++jj) {
                        const float4 sv = sm[jj];
#pragma unroll
                        for (int gg = 0; gg < G; ++gg) {
                            float ra, rb;
                            upk(entropy_r2<DIM>(X[gg], Y[gg], Z[gg], sv), ra, rb);
                            zt += (ra == 0.f) + (rb == 0.f);
                            acc += entropy_phi2<false>(fmaxf(ra, kR2Floor), fmaxf(rb, kR2Floor), cq);
                        }
                    }
                }
            } else if (!diag) {
                int jj = 0;
                if constexpr (QPOW && MM_ENT_POLY) {
#pragma unroll 2
                    for (; jj + 2 <= cnt; jj += 2) {
                        entropy_src<DIM, QPOW, MM_ENT_POLY >= 2, CLAMP>(sm[jj], X, Y, Z, cq, acc, zt);
                        entropy_src<DIM, QPOW, true, CLAMP>(sm[jj + 1], X, Y, Z, cq, acc, zt);
                    }
                }
#pragma unroll 4
                for (; jj < cnt; ++jj) entropy_src<DIM, QPOW, false, CLAMP>(sm[jj], X, Y, Z, cq, acc, zt);
            } else {
                for (int jj = 0; jj < cnt; ++jj) {
                    const float4 sv = sm[jj];
                    const int32_t j = (int32_t)(t0 + jj);
#pragma unroll
                    for (int gg = 0; gg < G; ++gg) {
                        float ra, rb;
                        upk(entropy_r2<DIM>(X[gg], Y[gg], Z[gg], sv), ra, rb);
                        const bool va = j > ti[2 * gg] && ti[2 * gg] < n;
                        const bool vb = j > ti[2 * gg + 1] && ti[2 * gg + 1] < n;
                        zt += (va && ra == 0.f) + (vb && rb == 0.f);
                        // masked pairs: r^2 = 1 contributes lg2(1) = 0 (q = 0); q > 0 masks the term
                        const float pa = va ? fmaxf(ra, kR2Floor) : 1.f, pb = vb ? fmaxf(rb, kR2Floor) : 1.f;
                        if constexpr (!QPOW) {
                            acc += entropy_phi2<false>(pa, pb, cq);
                        } else {
                            acc += (va ? entropy_phi2<true>(pa, 1.f, cq) - 1.f : 0.f) +
                                   (vb ? entropy_phi2<true>(pb, 1.f, cq) - 1.f : 0.f);
                        }
                    }
                }
            }
            // coincident pairs entered with r^2 = kR2Floor: remove their contribution
            if (zt) acc -= (float)zt * entropy_phi2<QPOW, CLAMP>(kR2Floor, 1.f, cq) - (QPOW ? (float)zt : 0.f);
            zc += zt;
            dacc += (double)acc;
        }
        u = seg_end;
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
        partial[g] = s;
        if (c) atomicAdd(coinc, c);
    }
}

template <int DIM, bool QPOW, bool COARSE>
#ifndef MM_COARSE_BMASK
#define MM_COARSE_BMASK 0  // measured: plain reciprocals beat batching once nu is folded (+2%, cfg3)
#endif
constexpr int kBatchMask = (DIM == 2 && !QPOW) ? (COARSE ? MM_COARSE_BMASK : 1) : 0;  // measured: tools/ubench_repulse.cu

#ifndef MM_C3_MINB
#define MM_C3_MINB 2  // 3-D q > 0 coarse kernel: at least 2 CTAs of 256 per SM (<= 128 registers)
#endif
#ifndef MM_C2_MINB
#define MM_C2_MINB 1  // 2-D coarse kernel: CTAs of 256 per SM the register budget must allow
#endif
template <int DIM, bool QPOW, bool COARSE>
constexpr int kMinB = (DIM == 3 && QPOW && COARSE) ? MM_C3_MINB : (DIM == 2 && COARSE) ? MM_C2_MINB : 1;

// q > 0 with (q + 2)/2 * |lg2 kEps2| <= 126: 2^(c lg2 r^2) cannot overflow, the
// kernels skip the upper clamp (CLAMP = false)
constexpr float kQNoClamp = 2.2f;

template <int DIM, bool QPOW, bool COARSE, int T, bool CLAMP = true>
int resident_ctas() {
    static const int occ = [] {  // per instantiation; queried once
        int o = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_repulse<DIM, QPOW, COARSE, T, kBatchMask<DIM, QPOW, COARSE>, kMinB<DIM, QPOW, COARSE>, MM_REP_UNR, CLAMP>,
                                                      kBlock, 0);
        return o > 0 ? o : 1;
    }();
    return occ;
}

// lazily queried device properties: function-local statics (thread-safe
// initialisation; one process drives one GPU)
int sm_count() {
    static const int sms = [] {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
        return v;
    }();
    return sms;
}

int targets_per_thread(int dim) { return dim == 2 ? MM_T2 : MM_T3; }

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
        occ = coarse ? (qpow ? resident_ctas<2, true, true, MM_T2>() : resident_ctas<2, false, true, MM_T2>())
                     : (qpow ? resident_ctas<2, true, false, MM_T2>() : resident_ctas<2, false, false, MM_T2>());
    } else {
        occ = coarse ? (qpow ? resident_ctas<3, true, true, MM_T3>() : resident_ctas<3, false, true, MM_T3>())
                     : (qpow ? resident_ctas<3, true, false, MM_T3>() : resident_ctas<3, false, false, MM_T3>());
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
                           int32_t n_src, const float4* rep_hi, const float4* rep_lo, const CoarseOrder& co,
                           const RepulsePlan& p, float* part, cudaStream_t st) {
    const float cexp = -(q + 2.0f) * 0.5f;
    LaunchScope ls(coarse ? "repulse_coarse" : "repulse_exact", st);
// batched reciprocals (BMASK) in half of the target groups for 2-D q = 0
// (exact and coarse: measured faster by tools/ubench_repulse.cu); none for q > 0.
#define MM_LAUNCH_CL(D, Q, C, T, CL) \
    k_repulse<D, Q, C, T, kBatchMask<D, Q, C>, kMinB<D, Q, C>, MM_REP_UNR, CL><<<p.sch.G, kBlock, 0, st>>>(n_tgt, x, n_src, rep_hi, rep_lo, co, cexp,  \
                                                                          p.sch, part)
#define MM_LAUNCH(D, Q, C, T) \
    do { if (Q && q <= kQNoClamp) MM_LAUNCH_CL(D, Q, C, T, false); else MM_LAUNCH_CL(D, Q, C, T, true); } while (0)
    if (dim == 2) {
        if (!qpow && !coarse) MM_LAUNCH(2, false, false, MM_T2);
        else if (!qpow && coarse) MM_LAUNCH(2, false, true, MM_T2);
        else if (qpow && !coarse) MM_LAUNCH(2, true, false, MM_T2);
        else MM_LAUNCH(2, true, true, MM_T2);
    } else {
        if (!qpow && !coarse) MM_LAUNCH(3, false, false, MM_T3);
        else if (!qpow && coarse) MM_LAUNCH(3, false, true, MM_T3);
        else if (qpow && !coarse) MM_LAUNCH(3, true, false, MM_T3);
        else MM_LAUNCH(3, true, true, MM_T3);
    }
#undef MM_LAUNCH
#undef MM_LAUNCH_CL
    return cudaGetLastError();
}

int repulse_targets_per_block(int dim) { return kBlock * targets_per_thread(dim); }


namespace {
template <int DIM, bool QPOW>
cudaError_t sym_launch(int32_t n, const float* x, float cexp, const TriSched& ts, float* ipart, float* jpart,
                       cudaStream_t st) {
    constexpr int smem = sym_smem_bytes<DIM>(kSymWarps);
    auto* fn = k_repulse_sym<DIM, QPOW, kSymSG, kSymWarps, kSymSrc>;
    static const bool attr = (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem), true);
    (void)attr;
    fn<<<ts.G, kSymWarps * 32, smem, st>>>(n, x, cexp, ts, ipart, jpart);
    return cudaGetLastError();
}

}  // namespace

SymPlan plan_repulse_sym(int32_t n, int dim) {
    SymPlan p;
    TriSched& t = p.ts;
    // units: (block pair (I, J >= I), source sub-tile): row I has NS (TB - I)
    t.TB = (int32_t)((n + kSymTPB - 1) / kSymTPB);
    t.Ub = t.TB * (kSymTPB / kSymSrc);
    t.c = kSymTPB / kSymSrc;
    t.U = tri_prefix(t.TB, t);
    static const int occ2 = [] {
        int v = 0;
        cudaFuncSetAttribute(k_repulse_sym<2, false, kSymSG, kSymWarps, kSymSrc>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, sym_smem_bytes<2>(kSymWarps));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k_repulse_sym<2, false, kSymSG, kSymWarps, kSymSrc>,
                                                      kSymWarps * 32, sym_smem_bytes<2>(kSymWarps));
        return std::max(v, 1);
    }();
    static const int occ3 = [] {
        int v = 0;
        cudaFuncSetAttribute(k_repulse_sym<3, false, kSymSG, kSymWarps, kSymSrc>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, sym_smem_bytes<3>(kSymWarps));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k_repulse_sym<3, false, kSymSG, kSymWarps, kSymSrc>,
                                                      kSymWarps * 32, sym_smem_bytes<3>(kSymWarps));
        return std::max(v, 1);
    }();
    const int o = dim == 3 ? occ3 : occ2;
    p.full_grid = (int64_t)sm_count() * o;
    t.G = (int32_t)std::max<int64_t>(1, std::min<int64_t>(p.full_grid, t.U));
    int32_t ms = 1;
    for (int32_t I = 0; I < t.TB; ++I) {
        const int32_t a = sched_first_cta_tri(tri_prefix(I, t), t);
        const int32_t b = sched_first_cta_tri(tri_prefix(I + 1, t) - 1, t);
        ms = std::max(ms, b - a + 1);
    }
    p.slots = ms;
    return p;
}

int64_t sym_jpart_rows(const SymPlan& p) { return std::max<int64_t>(p.ts.TB - 1, 1); }

cudaError_t launch_repulse_sym(int dim, bool qpow, float q, int32_t n, const float* x, const SymPlan& p,
                               float* ipart, float* jpart, cudaStream_t st) {
    const float cexp = -(q + 2.0f) * 0.5f;
    LaunchScope ls("repulse_exact", st);
    if (dim == 2) return qpow ? sym_launch<2, true>(n, x, cexp, p.ts, ipart, jpart, st)
                              : sym_launch<2, false>(n, x, cexp, p.ts, ipart, jpart, st);
    return qpow ? sym_launch<3, true>(n, x, cexp, p.ts, ipart, jpart, st)
                : sym_launch<3, false>(n, x, cexp, p.ts, ipart, jpart, st);
}

EntropyPlan plan_entropy(int32_t n) {
    EntropyPlan p;
    TriSched& t = p.ts;
    const int TPB = kBlock * 4;
    t.TB = (int32_t)((n + TPB - 1) / TPB);
    t.Ub = (int32_t)((n + kBlock - 1) / kBlock);
    t.c = TPB / kBlock;
    t.U = tri_prefix(t.TB, t);
    static const int occ = [] {
        int o = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_entropy_tri<2, false>, kBlock, 0);
        return std::max(o, 1);
    }();
    t.G = (int32_t)std::max<int64_t>(1, std::min<int64_t>((int64_t)sm_count() * occ, t.U));
    p.nblocks = t.G;
    return p;
}

cudaError_t launch_entropy_all(int dim, double q, int32_t n, const float* x, const EntropyPlan& p,
                               double* partial, int32_t* coinc, cudaStream_t st) {
    const float cq = (float)(-q * 0.5);
    LaunchScope ls("entropy_pairs", st);
    const bool qpow = q != 0.0;
    const int G = p.ts.G;
    // (q/2) |lg2 kR2Floor| <= 126: the q > 0 pair terms cannot overflow, no clamp
    const bool noclamp = q <= 4.2;
    if (dim == 2) {
        if (qpow && noclamp) k_entropy_tri<2, true, false><<<G, kBlock, 0, st>>>(n, x, cq, p.ts, partial, coinc);
        else if (qpow) k_entropy_tri<2, true><<<G, kBlock, 0, st>>>(n, x, cq, p.ts, partial, coinc);
        else k_entropy_tri<2, false><<<G, kBlock, 0, st>>>(n, x, cq, p.ts, partial, coinc);
    } else {
        if (qpow && noclamp) k_entropy_tri<3, true, false><<<G, kBlock, 0, st>>>(n, x, cq, p.ts, partial, coinc);
        else if (qpow) k_entropy_tri<3, true><<<G, kBlock, 0, st>>>(n, x, cq, p.ts, partial, coinc);
        else k_entropy_tri<3, false><<<G, kBlock, 0, st>>>(n, x, cq, p.ts, partial, coinc);
    }
    return cudaGetLastError();
}

}  // namespace mm
