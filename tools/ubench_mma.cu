// Builder tool: far-tile repulsion sum through the tensor cores (3xTF32 mma.sync)
// against the plain FP32 pair loop, both checked against an FP64 sum.
//
//   T_i = sum_j nu_j (x_i - x_j) / |x_i - x_j|^(q+2)      (3-D, q > 0)
//
// over the source tiles (256 Morton-ordered sources) that are FAR from the
// warp's 64 Morton-ordered targets.  Tile-local frame: x' = x - c_t (tile-box
// centre), so that |x_j'| <= rho << |x_i'| = D and
//   r^2 = |x_i'|^2 - 2 x_i'.x_j' + |x_j'|^2
// loses at most a few ulp(D^2) ~ ulp(r^2).  Both contractions run as TF32
// mma.sync.m16n8k8 with exact hi/lo splits (products exact, FP32 accumulate):
//   MMA1 (K = 16):  r^2[i][j] = A1[i][.] . B1[.][j]
//   MMA2 (K = 8 sources, N = 8 columns): C[i][.] += inv[i][j] * (nu x_j' hi/lo, nu)
// and per tile T_i += x_i' * C[i][nu] - C[i][x hi] - C[i][x lo].
// Prints ms, pairs/s, cycles per 64 pairs per SMSP and the error of both FP32
// paths relative to sum_j |term| (FP64).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1506_04383_b200/csrc/mm_common.cuh"

using namespace mm;

#ifndef UB_POLYMASK
#define UB_POLYMASK 0xFFFFFFFFu  // blocks (of 8 sources) whose 2^y runs on the FMA pipe
#endif
#ifndef UB_SPLIT
#define UB_SPLIT 2  // 2: inv as hi + lo (two MMA2), 1: hi only (round to nearest), 0: truncate
#endif
#ifndef UB_MINB2
#define UB_MINB2 2
#endif
#ifndef UB_MT
#define UB_MT 4
#endif
#ifndef UB_BUNR
#define UB_BUNR 2
#endif
#ifndef UB_MINB
#define UB_MINB 2
#endif

constexpr int kBUnr = UB_BUNR;
constexpr int kTile = 256, kNB = kTile / 8, kThreads = 256, kWarps = kThreads / 32, kTPW = 64;
__constant__ float kFarEta = 0.5f;  // eligible: r_min >= eta * D_max (argv[5])

struct Box {
    float lo[3], hi[3];
};

__device__ __forceinline__ uint32_t rn_tf32(float v) {  // round to nearest (ties away) to 10 mantissa bits
    return (__float_as_uint(v) + 0x1000u) & 0xFFFFE000u;
}
__device__ __forceinline__ void split_tf32(float v, float& h, float& l) {
    h = __uint_as_float(rn_tf32(v));
    l = __uint_as_float(rn_tf32(v - h));
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// 2^(c L) for a packed pair, polynomial (FMA pipe); L <= lmax keeps c L >= -125
__device__ __forceinline__ f2x ex2_poly_scaled(f2x L, float c) {
    constexpr float kShift = 12582912.0f;
    const f2x cc = pk(c, c);
    const f2x t = fma2(L, cc, pk(kShift, kShift));
    float t0, t1;
    upk(t, t0, t1);
    const f2x nn = fma2(t, pk(-1.f, -1.f), pk(kShift, kShift));
    const f2x f = fma2(L, cc, nn);
    f2x p = pk(0.0013266970636323094f, 0.0013266970636323094f);
    p = fma2(p, f, pk(0.009675459936261177f, 0.009675459936261177f));
    p = fma2(p, f, pk(0.05550742521882057f, 0.05550742521882057f));
    p = fma2(p, f, pk(0.24022121727466583f, 0.24022121727466583f));
    p = fma2(p, f, pk(0.6931469440460205f, 0.6931469440460205f));
    p = fma2(p, f, pk(1.0000001192092896f, 1.0000001192092896f));
    float p0, p1;
    upk(p, p0, p1);
    return pk(__int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23)),
              __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23)));
}

__device__ __forceinline__ bool eligible(const Box& w, const float4 blo, const float4 bhi, float (&ct)[3]) {
    float rho2 = 0.f, dn2 = 0.f, df2 = 0.f;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const float lo = d == 0 ? blo.x : d == 1 ? blo.y : blo.z, hi = d == 0 ? bhi.x : d == 1 ? bhi.y : bhi.z;
        ct[d] = 0.5f * (lo + hi);
        const float h = 0.5f * (hi - lo);
        rho2 += h * h;
        const float dn = fmaxf(0.f, fmaxf(w.lo[d] - ct[d], ct[d] - w.hi[d]));
        const float df = fmaxf(fabsf(w.lo[d] - ct[d]), fabsf(w.hi[d] - ct[d]));
        dn2 += dn * dn;
        df2 += df * df;
    }
    const float rho = sqrtf(rho2), dn = sqrtf(dn2), df = sqrtf(df2);
    return dn - rho >= kFarEta * df;
}

__device__ __forceinline__ Box warp_box(const float4* tg, int lane) {
    Box b;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const float a = d == 0 ? tg[lane].x : d == 1 ? tg[lane].y : tg[lane].z;
        const float c = d == 0 ? tg[lane + 32].x : d == 1 ? tg[lane + 32].y : tg[lane + 32].z;
        float lo = fminf(a, c), hi = fmaxf(a, c);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        b.lo[d] = lo;
        b.hi[d] = hi;
    }
    return b;
}

// ---------------------------------------------------------------- MMA path
__global__ void __launch_bounds__(kThreads, UB_MINB)
k_mma(int n_tgt, const float4* __restrict__ tgt, int n_src, const float4* __restrict__ src,
      const float4* __restrict__ tile_box, float cexp, float4* __restrict__ out, unsigned long long* __restrict__ npairs) {
    __shared__ float4 B1s[kNB][32];
    __shared__ float2 B2s[kNB][32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, c = lane & 3;
    const int ntiles = (n_src + kTile - 1) / kTile;
    const int64_t wbase = ((int64_t)blockIdx.x * kWarps + warp) * kTPW;
    if (wbase + kTPW > n_tgt) return;  // ubench: n_tgt is a multiple of the CTA's targets
    const Box wb = warp_box(tgt + wbase, lane);
    // my targets: m-tile m holds targets wbase + 16 m + g and + 8
    float X[4][2][3];
    float T[4][2];
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const float4 v = __ldg(tgt + wbase + 16 * m + 8 * h + g);
            X[m][h][0] = v.x;
            X[m][h][1] = v.y;
            X[m][h][2] = v.z;
            T[m][h] = 0.f;
        }
    unsigned long long cnt = 0;
    for (int tile = 0; tile < ntiles; ++tile) {
        const float4 blo = __ldg(tile_box + 2 * tile), bhi = __ldg(tile_box + 2 * tile + 1);
        float ct[3];
        const bool ok = eligible(wb, blo, bhi, ct);
        __syncthreads();
        {
            // fill: thread = source s of the tile (frame-relative, hi/lo splits)
            const int s = tid, b = s >> 3, j = s & 7;
            const int64_t js = (int64_t)tile * kTile + s;
            float4 v = js < n_src ? __ldg(src + js) : make_float4(ct[0], ct[1], ct[2], 0.f);
            const float xs[3] = {v.x - ct[0], v.y - ct[1], v.z - ct[2]};
            const float nu = v.w;
            float ss = fmaf(xs[0], xs[0], fmaf(xs[1], xs[1], fmaf(xs[2], xs[2], kEps2)));
            float sh, sl;
            split_tf32(ss, sh, sl);
            float* b2 = reinterpret_cast<float*>(&B2s[b][0]);
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                float h, l;
                split_tf32(xs[d], h, l);
                B1s[b][4 * j + d] = make_float4(-2.f * h, -2.f * l, -2.f * h, -2.f * l);
                float ph, pl;
                split_tf32(nu * xs[d], ph, pl);
                b2[((2 * d) * 4 + (j >> 1)) * 2 + (j & 1)] = ph;
                b2[((2 * d + 1) * 4 + (j >> 1)) * 2 + (j & 1)] = pl;
            }
            B1s[b][4 * j + 3] = make_float4(1.f, 1.f, sh, sl);
            b2[(6 * 4 + (j >> 1)) * 2 + (j & 1)] = nu;
            b2[(7 * 4 + (j >> 1)) * 2 + (j & 1)] = 0.f;
        }
        __syncthreads();
        if (!ok) continue;
        cnt += kTile;
        // A1 fragments of the four m-tiles in the tile's frame
        uint32_t A1[4][8];
        float XC[4][2];
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const float x0 = X[m][h][0] - ct[0], x1 = X[m][h][1] - ct[1], x2 = X[m][h][2] - ct[2];
                const float S = fmaf(x0, x0, fmaf(x1, x1, x2 * x2));
                const float v = c == 0 ? x0 : c == 1 ? x1 : c == 2 ? x2 : S;
                float vh, vl;
                split_tf32(v, vh, vl);
                XC[m][h] = v;
                const float one = 1.f;
                // MMA1a: slots c (a0/a1) and c+4 (a2/a3); MMA1b: slots c+8, c+12
                A1[m][0 + h] = __float_as_uint(vh);
                A1[m][2 + h] = __float_as_uint(c == 3 ? vl : vh);
                A1[m][4 + h] = __float_as_uint(c == 3 ? one : vl);
                A1[m][6 + h] = __float_as_uint(c == 3 ? one : vl);
            }
        float C2[4][4];
#pragma unroll
        for (int m = 0; m < 4; ++m) C2[m][0] = C2[m][1] = C2[m][2] = C2[m][3] = 0.f;
#pragma unroll 2
        for (int b = 0; b < kNB; ++b) {
            const float4 b1 = B1s[b][lane];
            const float2 b2 = B2s[b][lane];
            const bool poly = (UB_POLYMASK >> (b & 31)) & 1u;
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                float r[4] = {0.f, 0.f, 0.f, 0.f};
                mma_tf32(r, A1[m][0], A1[m][1], A1[m][2], A1[m][3], __float_as_uint(b1.x), __float_as_uint(b1.y));
                mma_tf32(r, A1[m][4], A1[m][5], A1[m][6], A1[m][7], __float_as_uint(b1.z), __float_as_uint(b1.w));
                // r0: (g, src 2c) r1: (g, 2c+1) r2: (g+8, 2c) r3: (g+8, 2c+1)
                // packed over the two targets of a source: (r0, r2) -> a0/a1, (r1, r3) -> a2/a3 of MMA2
                f2x ia, ib;
                if (poly) {
                    ia = ex2_poly_scaled(pk(lg2_approx(r[0]), lg2_approx(r[2])), cexp);
                    ib = ex2_poly_scaled(pk(lg2_approx(r[1]), lg2_approx(r[3])), cexp);
                } else {
                    float y0, y1, y2, y3;
                    upk(mul_bc(pk(lg2_approx(r[0]), lg2_approx(r[2])), cexp), y0, y2);
                    upk(mul_bc(pk(lg2_approx(r[1]), lg2_approx(r[3])), cexp), y1, y3);
                    ia = pk(ex2_approx(y0), ex2_approx(y2));
                    ib = pk(ex2_approx(y1), ex2_approx(y3));
                }
                float i0, i1, i2, i3;
                upk(ia, i0, i2);
                upk(ib, i1, i3);
                // A2: a0 = (g, k=c <-> src 2c), a1 = (g+8, src 2c), a2 = (g, src 2c+1), a3 = (g+8, src 2c+1)
                if (UB_SPLIT == 2) {
                    const uint32_t h0 = rn_tf32(i0), h1 = rn_tf32(i1), h2 = rn_tf32(i2), h3 = rn_tf32(i3);
                    mma_tf32(C2[m], h0, h2, h1, h3, __float_as_uint(b2.x), __float_as_uint(b2.y));
                    float l0, l1, l2, l3;
                    upk(add2(ia, pk(-__uint_as_float(h0), -__uint_as_float(h2))), l0, l2);
                    upk(add2(ib, pk(-__uint_as_float(h1), -__uint_as_float(h3))), l1, l3);
                    mma_tf32(C2[m], __float_as_uint(l0), __float_as_uint(l2), __float_as_uint(l1), __float_as_uint(l3),
                             __float_as_uint(b2.x), __float_as_uint(b2.y));
                } else if (UB_SPLIT == 1) {
                    mma_tf32(C2[m], rn_tf32(i0), rn_tf32(i2), rn_tf32(i1), rn_tf32(i3), __float_as_uint(b2.x),
                             __float_as_uint(b2.y));
                } else {
                    mma_tf32(C2[m], __float_as_uint(i0), __float_as_uint(i2), __float_as_uint(i1), __float_as_uint(i3),
                             __float_as_uint(b2.x), __float_as_uint(b2.y));
                }
            }
        }
        // fold the tile: lane c < 3 owns component c of targets (g, g+8); W = column 6 lives in lane c = 3
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const float Wa = __shfl_sync(0xffffffffu, C2[m][0], lane | 3), Wb = __shfl_sync(0xffffffffu, C2[m][2], lane | 3);
            T[m][0] += fmaf(XC[m][0], Wa, -(C2[m][0] + C2[m][1]));
            T[m][1] += fmaf(XC[m][1], Wb, -(C2[m][2] + C2[m][3]));
        }
    }
    if (c < 3) {
#pragma unroll
        for (int m = 0; m < 4; ++m)
#pragma unroll
            for (int h = 0; h < 2; ++h) reinterpret_cast<float*>(out + wbase + 16 * m + 8 * h + g)[c] = T[m][h];
    }
    if (lane == 0 && npairs) atomicAdd(npairs, cnt * kTPW);
}

// ---------------------------------------------------------------- MMA2-only path: r^2 on the FMA pipe in expanded form, accumulation on the tensor cores
template <int MT>
__global__ void __launch_bounds__(kThreads, UB_MINB2)
k_mma2(int n_tgt, const float4* __restrict__ tgt, int n_src, const float4* __restrict__ src,
      const float4* __restrict__ tile_box, float cexp, float4* __restrict__ out, unsigned long long* __restrict__ npairs) {
    __shared__ float4 S4[kTile];  // (x', y', z', |x'|^2 + eps) in the tile frame
    __shared__ float2 B2s[kNB][32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, c = lane & 3;
    const int ntiles = (n_src + kTile - 1) / kTile;
    constexpr int TPW = 16 * MT;
    const int64_t wbase = ((int64_t)blockIdx.x * kWarps + warp) * TPW;
    if (wbase + TPW > n_tgt) return;  // ubench: n_tgt is a multiple of the CTA's targets
    const Box wb = warp_box(tgt + (wbase / 64) * 64, lane);  // box of the enclosing 64 targets (ubench)
    // my targets: m-tile m holds targets wbase + 16 m + g and + 8
    float X[MT][2][3];
    float T[MT][2];
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const float4 v = __ldg(tgt + wbase + 16 * m + 8 * h + g);
            X[m][h][0] = v.x;
            X[m][h][1] = v.y;
            X[m][h][2] = v.z;
            T[m][h] = 0.f;
        }
    unsigned long long cnt = 0;
    for (int tile = 0; tile < ntiles; ++tile) {
        const float4 blo = __ldg(tile_box + 2 * tile), bhi = __ldg(tile_box + 2 * tile + 1);
        float ct[3];
        const bool ok = eligible(wb, blo, bhi, ct);
        __syncthreads();
        {
            // fill: thread = source s of the tile (frame-relative, hi/lo splits)
            const int s = tid, b = s >> 3, j = s & 7;
            const int64_t js = (int64_t)tile * kTile + s;
            float4 v = js < n_src ? __ldg(src + js) : make_float4(ct[0], ct[1], ct[2], 0.f);
            const float xs[3] = {v.x - ct[0], v.y - ct[1], v.z - ct[2]};
            const float nu = v.w;
            float ss = fmaf(xs[0], xs[0], fmaf(xs[1], xs[1], fmaf(xs[2], xs[2], kEps2)));
            float sh, sl;
            split_tf32(ss, sh, sl);
            float* b2 = reinterpret_cast<float*>(&B2s[b][0]);
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                float h, l;
                split_tf32(xs[d], h, l);
                float ph, pl;
                split_tf32(nu * xs[d], ph, pl);
                b2[((2 * d) * 4 + (j >> 1)) * 2 + (j & 1)] = ph;
                b2[((2 * d + 1) * 4 + (j >> 1)) * 2 + (j & 1)] = pl;
            }
            S4[s] = make_float4(xs[0], xs[1], xs[2], ss);
            b2[(6 * 4 + (j >> 1)) * 2 + (j & 1)] = nu;
            b2[(7 * 4 + (j >> 1)) * 2 + (j & 1)] = 0.f;
        }
        __syncthreads();
        if (!ok) continue;
        cnt += kTile;
        // targets (g, g+8) of the four m-tiles in the tile frame: -2 x', |x'|^2 packed over the two targets
        f2x MX[MT], MY[4], MZ[4], SI[4];
        float XC[MT][2];
#pragma unroll
        for (int m = 0; m < MT; ++m) {
            float x0[2], x1[2], x2[2], S[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                x0[h] = X[m][h][0] - ct[0];
                x1[h] = X[m][h][1] - ct[1];
                x2[h] = X[m][h][2] - ct[2];
                S[h] = fmaf(x0[h], x0[h], fmaf(x1[h], x1[h], x2[h] * x2[h]));
                XC[m][h] = c == 0 ? x0[h] : c == 1 ? x1[h] : x2[h];
            }
            MX[m] = pk(-2.f * x0[0], -2.f * x0[1]);
            MY[m] = pk(-2.f * x1[0], -2.f * x1[1]);
            MZ[m] = pk(-2.f * x2[0], -2.f * x2[1]);
            SI[m] = pk(S[0], S[1]);
        }
        float C2[MT][4];
#pragma unroll
        for (int m = 0; m < MT; ++m) C2[m][0] = C2[m][1] = C2[m][2] = C2[m][3] = 0.f;
#pragma unroll kBUnr
        for (int b = 0; b < kNB; ++b) {
            const float4 sa = S4[8 * b + 2 * c], sb = S4[8 * b + 2 * c + 1];
            const float2 b2 = B2s[b][lane];
            const bool poly = (UB_POLYMASK >> (b & 31)) & 1u;
#pragma unroll
            for (int m = 0; m < MT; ++m) {
                // r^2 = (|x_i'|^2 + |x_j'|^2) - 2 x_i'.x_j' for (g, g+8) x source c / source c+4
                f2x ra = fma2(MX[m], pk(sa.x, sa.x), fma2(MY[m], pk(sa.y, sa.y), fma2(MZ[m], pk(sa.z, sa.z), add2(SI[m], pk(sa.w, sa.w)))));
                f2x rb = fma2(MX[m], pk(sb.x, sb.x), fma2(MY[m], pk(sb.y, sb.y), fma2(MZ[m], pk(sb.z, sb.z), add2(SI[m], pk(sb.w, sb.w)))));
                float r[4];
                upk(ra, r[0], r[2]);
                upk(rb, r[1], r[3]);
                f2x ia, ib;
                if (poly) {
                    ia = ex2_poly_scaled(pk(lg2_approx(r[0]), lg2_approx(r[2])), cexp);
                    ib = ex2_poly_scaled(pk(lg2_approx(r[1]), lg2_approx(r[3])), cexp);
                } else {
                    float y0, y1, y2, y3;
                    upk(mul_bc(pk(lg2_approx(r[0]), lg2_approx(r[2])), cexp), y0, y2);
                    upk(mul_bc(pk(lg2_approx(r[1]), lg2_approx(r[3])), cexp), y1, y3);
                    ia = pk(ex2_approx(y0), ex2_approx(y2));
                    ib = pk(ex2_approx(y1), ex2_approx(y3));
                }
                float i0, i1, i2, i3;
                upk(ia, i0, i2);
                upk(ib, i1, i3);
                // A2: a0 = (g, k=c <-> src 2c), a1 = (g+8, src 2c), a2 = (g, src 2c+1), a3 = (g+8, src 2c+1)
                if (UB_SPLIT == 2) {
                    const uint32_t h0 = rn_tf32(i0), h1 = rn_tf32(i1), h2 = rn_tf32(i2), h3 = rn_tf32(i3);
                    mma_tf32(C2[m], h0, h2, h1, h3, __float_as_uint(b2.x), __float_as_uint(b2.y));
                    float l0, l1, l2, l3;
                    upk(add2(ia, pk(-__uint_as_float(h0), -__uint_as_float(h2))), l0, l2);
                    upk(add2(ib, pk(-__uint_as_float(h1), -__uint_as_float(h3))), l1, l3);
                    mma_tf32(C2[m], __float_as_uint(l0), __float_as_uint(l2), __float_as_uint(l1), __float_as_uint(l3),
                             __float_as_uint(b2.x), __float_as_uint(b2.y));
                } else if (UB_SPLIT == 1) {
                    mma_tf32(C2[m], rn_tf32(i0), rn_tf32(i2), rn_tf32(i1), rn_tf32(i3), __float_as_uint(b2.x),
                             __float_as_uint(b2.y));
                } else {
                    mma_tf32(C2[m], __float_as_uint(i0), __float_as_uint(i2), __float_as_uint(i1), __float_as_uint(i3),
                             __float_as_uint(b2.x), __float_as_uint(b2.y));
                }
            }
        }
        // fold the tile: lane c < 3 owns component c of targets (g, g+8); W = column 6 lives in lane c = 3
#pragma unroll
        for (int m = 0; m < MT; ++m) {
            const float Wa = __shfl_sync(0xffffffffu, C2[m][0], lane | 3), Wb = __shfl_sync(0xffffffffu, C2[m][2], lane | 3);
            T[m][0] += fmaf(XC[m][0], Wa, -(C2[m][0] + C2[m][1]));
            T[m][1] += fmaf(XC[m][1], Wb, -(C2[m][2] + C2[m][3]));
        }
    }
    if (c < 3) {
#pragma unroll
        for (int m = 0; m < MT; ++m)
#pragma unroll
            for (int h = 0; h < 2; ++h) reinterpret_cast<float*>(out + wbase + 16 * m + 8 * h + g)[c] = T[m][h];
    }
    if (lane == 0 && npairs) atomicAdd(npairs, cnt * TPW);
}

// ---------------------------------------------------------------- plain FP32 / FP64 pair loops (same eligible tiles)
template <typename R>
__global__ void __launch_bounds__(kThreads)
k_direct(int n_tgt, const float4* __restrict__ tgt, int n_src, const float4* __restrict__ src,
         const float4* __restrict__ tile_box, R cexp, R* __restrict__ out, R* __restrict__ out_abs) {
    __shared__ float4 sm[kTile];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ntiles = (n_src + kTile - 1) / kTile;
    const int64_t wbase = ((int64_t)blockIdx.x * kWarps + warp) * kTPW;
    if (wbase + kTPW > n_tgt) return;
    const Box wb = warp_box(tgt + wbase, lane);
    R acc[2][3] = {{0, 0, 0}, {0, 0, 0}}, aabs[2] = {0, 0};
    float4 me[2] = {__ldg(tgt + wbase + lane), __ldg(tgt + wbase + lane + 32)};
    for (int tile = 0; tile < ntiles; ++tile) {
        const float4 blo = __ldg(tile_box + 2 * tile), bhi = __ldg(tile_box + 2 * tile + 1);
        float ct[3];
        const bool ok = eligible(wb, blo, bhi, ct);
        __syncthreads();
        const int64_t js = (int64_t)tile * kTile + tid;
        sm[tid] = js < n_src ? __ldg(src + js) : make_float4(0.f, 0.f, 0.f, 0.f);
        __syncthreads();
        if (!ok) continue;
        const int cnt = min(kTile, n_src - tile * kTile);
        R t[2][3] = {{0, 0, 0}, {0, 0, 0}};
        for (int jj = 0; jj < cnt; ++jj) {
            const float4 s = sm[jj];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const R dx = (R)me[h].x - (R)s.x, dy = (R)me[h].y - (R)s.y, dz = (R)me[h].z - (R)s.z;
                const R r2 = dx * dx + dy * dy + dz * dz + (R)kEps2;
                R inv;
                if constexpr (sizeof(R) == 4)
                    inv = ex2_approx((float)cexp * lg2_approx((float)r2));
                else
                    inv = exp2(cexp * log2(r2));
                inv *= (R)s.w;
                t[h][0] += dx * inv;
                t[h][1] += dy * inv;
                t[h][2] += dz * inv;
                if (out_abs) aabs[h] += sqrt(r2) * inv;
            }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int d = 0; d < 3; ++d) acc[h][d] += t[h][d];
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int64_t i = wbase + lane + 32 * h;
        out[4 * i + 0] = acc[h][0];
        out[4 * i + 1] = acc[h][1];
        out[4 * i + 2] = acc[h][2];
        if (out_abs) out_abs[i] = aabs[h];
    }
}

static uint32_t part1by2(uint32_t x) {
    x &= 0x3ff;
    x = (x | (x << 16)) & 0x30000ff;
    x = (x | (x << 8)) & 0x300f00f;
    x = (x | (x << 4)) & 0x30c30c3;
    x = (x | (x << 2)) & 0x9249249;
    return x;
}
static uint32_t morton(float x, float y, float z) {
    return part1by2((uint32_t)(x * 1023.f)) | (part1by2((uint32_t)(y * 1023.f)) << 1) |
           (part1by2((uint32_t)(z * 1023.f)) << 2);
}
static void make_points(int n, uint64_t seed, float scale, float offs, bool masses, std::vector<float4>& p) {
    p.resize(n);
    uint64_t s = seed;
    auto rnd = [&]() {
        s = s * 6364136223846793005ULL + 1442695040888963407ULL;
        return (float)((s >> 40) & 0xFFFFFF) / 16777216.f;
    };
    std::vector<std::pair<uint32_t, int>> key(n);
    std::vector<float4> q(n);
    for (int i = 0; i < n; ++i) {
        float x = rnd(), y = rnd(), z = rnd();
        key[i] = {morton(x, y, z), i};
        q[i] = make_float4(offs + scale * x, offs + scale * y, offs + scale * z, masses ? (float)(1 + (int)(rnd() * 4.f)) : 1.f);
    }
    std::sort(key.begin(), key.end());
    for (int i = 0; i < n; ++i) p[i] = q[key[i].second];
}

int main(int argc, char** argv) {
    const int n_tgt = argc > 1 ? atoi(argv[1]) : 148 * 2 * kWarps * kTPW;  // one wave at 2 CTAs/SM
    const int n_src = argc > 2 ? atoi(argv[2]) : 65536;
    const float q = 0.8f, cexp = -(q + 2.f) / 2.f;
    const float scale = argc > 3 ? atof(argv[3]) : 100.f, offs = argc > 4 ? atof(argv[4]) : -50.f;
    const float eta = argc > 5 ? atof(argv[5]) : 0.5f;
    cudaMemcpyToSymbol(kFarEta, &eta, 4);
    std::vector<float4> ht, hs;
    make_points(n_tgt, 1, scale, offs, false, ht);
    const float soff = argc > 6 ? atof(argv[6]) : 0.f;  // sources shifted along x: > 2 * scale makes every tile eligible
    make_points(n_src, 2, scale, offs, true, hs);
    for (auto& v : hs) v.x += soff;
    const int ntiles = (n_src + kTile - 1) / kTile;
    std::vector<float4> hb(2 * ntiles);
    for (int t = 0; t < ntiles; ++t) {
        float lo[3] = {1e30f, 1e30f, 1e30f}, hi[3] = {-1e30f, -1e30f, -1e30f};
        for (int j = t * kTile; j < std::min(n_src, (t + 1) * kTile); ++j) {
            const float v[3] = {hs[j].x, hs[j].y, hs[j].z};
            for (int d = 0; d < 3; ++d) {
                lo[d] = std::min(lo[d], v[d]);
                hi[d] = std::max(hi[d], v[d]);
            }
        }
        hb[2 * t] = make_float4(lo[0], lo[1], lo[2], 0.f);
        hb[2 * t + 1] = make_float4(hi[0], hi[1], hi[2], 0.f);
    }
    float4 *dt, *ds, *db, *dout;
    float* dref32;
    double *dref64, *dabs;
    unsigned long long* dnp;
    cudaMalloc(&dt, n_tgt * 16);
    cudaMalloc(&ds, n_src * 16);
    cudaMalloc(&db, 2 * ntiles * 16);
    cudaMalloc(&dout, n_tgt * 16);
    cudaMalloc(&dref32, n_tgt * 16);
    cudaMalloc(&dref64, n_tgt * 32);
    cudaMalloc(&dabs, n_tgt * 8);
    cudaMalloc(&dnp, 8);
    cudaMemcpy(dt, ht.data(), n_tgt * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(ds, hs.data(), n_src * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(db, hb.data(), 2 * ntiles * 16, cudaMemcpyHostToDevice);
    cudaMemset(dout, 0, n_tgt * 16);
    cudaMemset(dnp, 0, 8);
    const int blocks = n_tgt / (kWarps * kTPW);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_mma<<<blocks, kThreads>>>(n_tgt, dt, n_src, ds, db, cexp, dout, dnp);
    cudaDeviceSynchronize();
    unsigned long long np = 0;
    cudaMemcpy(&np, dnp, 8, cudaMemcpyDeviceToHost);
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        k_mma<<<blocks, kThreads>>>(n_tgt, dt, n_src, ds, db, cexp, dout, nullptr);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms);
    }
    float best2 = 1e30f;
    float4* dout2;
    cudaMalloc(&dout2, n_tgt * 16);
    cudaMemset(dout2, 0, n_tgt * 16);
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        k_mma2<UB_MT><<<n_tgt / (kWarps * 16 * UB_MT), kThreads>>>(n_tgt, dt, n_src, ds, db, cexp, dout2, nullptr);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best2 = std::min(best2, ms);
    }
    float best32 = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        k_direct<float><<<blocks, kThreads>>>(n_tgt, dt, n_src, ds, db, cexp, dref32, nullptr);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best32 = std::min(best32, ms);
    }
    k_direct<double><<<blocks, kThreads>>>(n_tgt, dt, n_src, ds, db, (double)cexp, dref64, dabs);
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) {
        printf("CUDA error: %s\n", cudaGetErrorString(err));
        return 1;
    }
    std::vector<float4> ho(n_tgt);
    std::vector<float> h32(4 * (size_t)n_tgt);
    std::vector<double> h64(4 * (size_t)n_tgt), habs(n_tgt);
    cudaMemcpy(ho.data(), dout, n_tgt * 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(h32.data(), dref32, n_tgt * 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(h64.data(), dref64, n_tgt * 32, cudaMemcpyDeviceToHost);
    cudaMemcpy(habs.data(), dabs, n_tgt * 8, cudaMemcpyDeviceToHost);
    double emax_m = 0, emax_d = 0, erms_m = 0, erms_d = 0, bias_m = 0, bias_d = 0, rmax_m = 0, rmax_d = 0;
    for (int i = 0; i < n_tgt; ++i) {
        const float om[3] = {ho[i].x, ho[i].y, ho[i].z};
        double nrm = 0;
        for (int d = 0; d < 3; ++d) nrm += h64[4 * (size_t)i + d] * h64[4 * (size_t)i + d];
        nrm = std::sqrt(nrm);
        for (int d = 0; d < 3; ++d) {
            const double ref = h64[4 * (size_t)i + d], a = habs[i] > 0 ? habs[i] : 1;
            const double em = (om[d] - ref) / a, ed = (h32[4 * (size_t)i + d] - ref) / a;
            emax_m = std::max(emax_m, std::fabs(em));
            emax_d = std::max(emax_d, std::fabs(ed));
            erms_m += em * em;
            erms_d += ed * ed;
            if (nrm > 0) {
                rmax_m = std::max(rmax_m, std::fabs(om[d] - ref) / nrm);
                rmax_d = std::max(rmax_d, std::fabs(h32[4 * (size_t)i + d] - ref) / nrm);
                // signed error along the reference direction (bias of the magnitude)
                bias_m += (om[d] - ref) * ref / (nrm * nrm);
                bias_d += (h32[4 * (size_t)i + d] - ref) * ref / (nrm * nrm);
            }
        }
    }
    erms_m = std::sqrt(erms_m / (3.0 * n_tgt));
    erms_d = std::sqrt(erms_d / (3.0 * n_tgt));
    int dev = 0, clk = 0, sms = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const double cyc64 = best * 1e-3 * clk * 1e3 * sms * 4.0 / ((double)np / 64.0);
    const double cyc64d = best32 * 1e-3 * clk * 1e3 * sms * 4.0 / ((double)np / 64.0);
    printf("eta=%.2f polymask=%08x split=%d minb=%d n_tgt=%d n_src=%d eligible pairs=%.4g (%.1f%% of all)\n", eta, (unsigned)UB_POLYMASK,
           UB_SPLIT, UB_MINB, n_tgt, n_src, (double)np, 100.0 * np / ((double)n_tgt * n_src));
    printf("mma    : %.3f ms  %.4g pairs/s  %.1f cycles per 64 pairs per SMSP\n", best, np / (best * 1e-3), cyc64);
    {
        std::vector<float4> ho2(n_tgt);
        cudaMemcpy(ho2.data(), dout2, n_tgt * 16, cudaMemcpyDeviceToHost);
        double emax = 0, erms = 0;
        for (int i = 0; i < n_tgt; ++i) {
            const float om[3] = {ho2[i].x, ho2[i].y, ho2[i].z};
            for (int d = 0; d < 3; ++d) {
                const double e = (om[d] - h64[4 * (size_t)i + d]) / (habs[i] > 0 ? habs[i] : 1);
                emax = std::max(emax, std::fabs(e));
                erms += e * e;
            }
        }
        printf("mma2 MT=%d minb=%d bunr=%d: %.3f ms  %.4g pairs/s  %.1f cycles per 64 pairs per SMSP; error / sum|term| max %.3g rms %.3g\n", UB_MT, UB_MINB2, UB_BUNR, best2,
               np / (best2 * 1e-3), best2 * 1e-3 * clk * 1e3 * sms * 4.0 / ((double)np / 64.0), emax, std::sqrt(erms / (3.0 * n_tgt)));
    }
    printf("direct : %.3f ms  %.4g pairs/s  %.1f cycles per 64 pairs per SMSP (plain loop, not the tuned kernel)\n", best32,
           np / (best32 * 1e-3), cyc64d);
    printf("error / sum|term| : mma max %.3g rms %.3g | fp32 direct max %.3g rms %.3g\n", emax_m, erms_m, emax_d, erms_d);
    printf("error / |T_i|     : mma max %.3g | fp32 direct max %.3g ; mean signed error along T: mma %.3g direct %.3g\n",
           rmax_m, rmax_d, bias_m / n_tgt, bias_d / n_tgt);
    return 0;
}
