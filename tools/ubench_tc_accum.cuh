// ubench_tc_accum.cuh (builder tool, not part of the library) — kernel (c), far tiles: the pair weights on the FMA / XU pipes,
// the accumulation over the sources on the 5th-generation tensor cores
// (tcgen05.mma kind::tf32, A operand = the weights in TMEM, accumulator in TMEM).
//
// For a block of 128 targets (TMEM lanes) and a stage of 128 coarse
// representatives ("sources") that lies FAR from the block,
//     T_i = sum_j nu_j (x_i - x_j) / |x_i - x_j|^(q+2)        (Eq.(3))
// is evaluated as
//   SIMT  r2[i][j] = (|x_i'|^2 + (|x_j'|^2 + eps)) - 2 x_i'.x_j'     1 FADD2 + 3 FFMA2 per packed pair
//         w[i][j]  = 2^(c lg2 r2[i][j])        MUFU.LG2 + a degree-5 polynomial on the FMA pipe (or MUFU.EX2)
//   MMA   D[i][.] += w[i][j] * B2[j][.]        columns of B2: nu x_j' (hi, lo per component), nu
// and T_i = x_i' * D[i][nu] - (D[i][x hi] + D[i][x lo]): the three accumulation
// FMAs per pair (and the nu multiply) leave the FMA pipe, and the difference
// vector x_i - x_j is never formed.
// Coordinates are relative to the centre c_b of the target block's box
// (x' = x - c_b), so |x_i'| <= rho_b and, for an eligible stage,
// r >= eta max|x_j'|: the cancellation in r2 costs a few ulp(max |x_j'|^2)
// <= ulp(r2) / eta^2.  B2 holds exact two-term TF32 splits
// (hi + lo, 11 significant bits each, round to nearest); the weights are
// rounded to TF32 (nearest) as they are written to TMEM, so every product is
// exact and only the FP32 accumulation rounds.  D is drained into FP32
// registers after every 256-source tile (round to nearest), which keeps the
// truncating tensor-core accumulation to 32 steps.
// The first design also computed r2 on the tensor cores (tools/ubench_tc_full.cuh):
// it is bound by TMEM reads (about 64 B/cycle per SM) and slower than the SIMT kernel.
//
// CTA (one per SM, persistent over target blocks), 21 warps:
//   warps 0-15  compute: warp w owns TMEM lanes 32 (w % 4) .. +31 (hardware rule)
//               = targets, and the 32 columns (w / 4) = sources of every 128-column stage
//   warps 16-19 fill: warp f stages the sources of stage k == f (mod 4) into
//               shared-memory buffer f: packed (x', y', z', s) pairs for the compute
//               warps and B2 in the canonical K-major no-swizzle UMMA layout
//   warp 20     one thread issues tcgen05.mma / tcgen05.commit
// Pipelines (mbarriers): bfull / bfree + sfree (smem stage), pfull / wfree (TMEM
// weight stage, 3 deep), d2full / d2free (accumulator, 2 deep).
#pragma once
#include "../paper_1506_04383_b200/csrc/k_repulse.cuh"

namespace mm {
namespace tc {

constexpr int kM = 128;        // targets per block = TMEM lanes
constexpr int kN = 128;        // sources per stage = TMEM columns of one r2 / weight stage
constexpr int kSB = 4;         // shared-memory stages (one per fill warp)
constexpr int kST = 3;         // TMEM stages
constexpr int kD2Col = kST * kN;  // first accumulator column (two accumulators of 16 columns)
constexpr int kTmemCols = 512;
constexpr int kComputeWarps = 16, kFillWarps = 4;
constexpr int kThreads = (kComputeWarps + kFillWarps + 1) * 32;  // 672

// shared-memory carve-up (bytes)
constexpr int kSrcBytes = kN * 16;      // 64 source pairs x 2 float4: (x0,x1,y0,y1), (z0,z1,s0,s1)
constexpr int kB2Bytes = 16 * kN * 4;   // 16 columns (7 used) x K128
constexpr int kOffSrc = 0;
constexpr int kOffB2 = kOffSrc + kSB * kSrcBytes;
constexpr int kOffRed = kOffB2 + kSB * kB2Bytes;
constexpr int kOffBar = kOffRed + 4 * kM * 16;
constexpr int kNumBars = 3 * kSB + 2 * kST + 4;
constexpr int kSmemBytes = kOffBar + kNumBars * 8 + 16;

struct Args {
    int32_t n_tgt;
    const float* x;          // [n][4]
    const int32_t* tperm;    // nullable: target slot -> vertex id
    const float4* frame;     // nullable: origin subtracted from the targets (representatives are frame-relative)
    int32_t n_src;
    const float4* rep_hi;    // (x, y, z, nu)
    const float4* rep_lo;    // nullable
    const float4* blk_box;   // [2 nblk] box of every 128-target block (frame-relative)
    const uint32_t* elig;    // [nblk][words] bit t: tile t (256 sources) is handled here
    int32_t words;
    float cexp;              // -(q+2)/2
    float4* out;             // [n] far-tile sums, stored at the vertex id
};

// ---------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W_%=;\n\t}"
        ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
// D[tmem] (+)= A[smem] . B[smem]^T
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc) : "memory");
}
// D[tmem] (+)= A[tmem] . B[smem]^T
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
        ::"r"(d), "r"(a), "l"(bdesc), "r"(idesc), "r"(acc) : "memory");
}
// canonical K-major, no-swizzle operand: 8-row x 16-byte core matrices; lbo = byte
// offset between the two 16-byte K chunks, sbo = between 8-row groups
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void tmem_ld32(uint32_t addr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(addr));
}
__device__ __forceinline__ void tmem_st32(uint32_t addr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
        ::"r"(addr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
          "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),
          "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),
          "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t addr, uint32_t (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(addr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ---------------------------------------------------------------- TF32 splits
__device__ __forceinline__ uint32_t rn_tf32(float v) {  // nearest (ties away) value with 10 explicit mantissa bits
    return (__float_as_uint(v) + 0x1000u) & 0xFFFFE000u;
}
__device__ __forceinline__ void split_tf32(float v, float& h, float& l) {
    h = __uint_as_float(rn_tf32(v));
    l = __uint_as_float(rn_tf32(v - h));
}

// 2^(c L) for a packed pair of L = lg2 r2 on the FMA pipe (same fit as k_repulse.cu's
// ex2_poly2_scaled; no clamps: eligible stages have eps < r2 < 2^80)
__device__ __forceinline__ f2x pow_poly2(f2x L, float c) {
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


// ---------------------------------------------------------------- pre-kernels
// box of every block of 128 targets (slot order, frame-relative): one warp per block
__global__ void __launch_bounds__(256) k_tc_boxes(int32_t n_tgt, const float* __restrict__ x,
                                                  const int32_t* __restrict__ tperm, const float4* __restrict__ frame,
                                                  float4* __restrict__ blk_box) {
    const int lane = threadIdx.x & 31;
    const int32_t blk = (int32_t)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    const int32_t nblk = (n_tgt + kM - 1) / kM;
    if (blk >= nblk) return;
    const float4 fr = frame ? __ldg(frame) : make_float4(0.f, 0.f, 0.f, 0.f);
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
#pragma unroll
    for (int u = 0; u < kM / 32; ++u) {
        int64_t i = (int64_t)blk * kM + u * 32 + lane;
        if (i >= n_tgt) i = n_tgt - 1;
        if (tperm) i = __ldg(tperm + i);
        const float4 v = __ldg(reinterpret_cast<const float4*>(x) + i);
        const float c[3] = {v.x - fr.x, v.y - fr.y, v.z - fr.z};
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            lo[d] = fminf(lo[d], c[d]);
            hi[d] = fmaxf(hi[d], c[d]);
        }
    }
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo[d] = fminf(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
            hi[d] = fmaxf(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
        }
    if (lane == 0) {
        blk_box[2 * blk] = make_float4(lo[0], lo[1], lo[2], 0.f);
        blk_box[2 * blk + 1] = make_float4(hi[0], hi[1], hi[2], 0.f);
    }
}

// eligibility of (block, tile): with c_b the block-box centre, rho_b its half diagonal,
// D the largest |x_j - c_b| over the tile box and r the box-to-box distance:
//   r >= eta D  and  r >= eta rho_b
__global__ void __launch_bounds__(256) k_tc_elig(int32_t nblk, const float4* __restrict__ blk_box, int32_t ntiles,
                                                 const float4* __restrict__ tile_box, float eta2, int32_t words,
                                                 uint32_t* __restrict__ elig) {
    const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (gid >= (int64_t)nblk * words) return;
    const int32_t blk = (int32_t)(gid / words), w = (int32_t)(gid % words);
    const float4 blo = __ldg(blk_box + 2 * blk), bhi = __ldg(blk_box + 2 * blk + 1);
    const float bl[3] = {blo.x, blo.y, blo.z}, bh[3] = {bhi.x, bhi.y, bhi.z};
    float cb[3], rho2 = 0.f;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        cb[d] = 0.5f * (bl[d] + bh[d]);
        const float h = 0.5f * (bh[d] - bl[d]);
        rho2 += h * h;
    }
    uint32_t m = 0;
    for (int b = 0; b < 32; ++b) {
        const int32_t t = w * 32 + b;
        if (t >= ntiles) break;
        const float4 tlo = __ldg(tile_box + 2 * t), thi = __ldg(tile_box + 2 * t + 1);
        const float tl[3] = {tlo.x, tlo.y, tlo.z}, th[3] = {thi.x, thi.y, thi.z};
        float r2 = 0.f, D2 = 0.f;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const float s = fmaxf(0.f, fmaxf(tl[d] - bh[d], bl[d] - th[d]));
            const float f = fmaxf(fabsf(tl[d] - cb[d]), fabsf(th[d] - cb[d]));
            r2 += s * s;
            D2 += f * f;
        }
        if (r2 >= eta2 * D2 && r2 >= eta2 * rho2 && r2 > 0.f && D2 < 1e30f) m |= 1u << b;
    }
    elig[gid] = m;
}

// ---------------------------------------------------------------- main kernel
#ifndef MM_TC_MUFU_MASK
#define MM_TC_MUFU_MASK 0x0000u  // bit p: source pair p of a thread's 16 takes MUFU.EX2 instead of the polynomial
#endif

__global__ void __launch_bounds__(kThreads, 1) k_repulse_tc(Args a) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t sbase = smem_u32(smem);
    const uint32_t bar0 = sbase + kOffBar;
    auto BFULL = [&](int s) { return bar0 + 8u * s; };                        // sources of smem stage s staged
    auto BFREE = [&](int s) { return bar0 + 8u * (kSB + s); };                // MMA done with B2 of stage s
    auto SFREE = [&](int s) { return bar0 + 8u * (2 * kSB + s); };            // compute warps done with the sources
    auto PFULL = [&](int s) { return bar0 + 8u * (3 * kSB + s); };            // weights of TMEM stage s written
    auto WFREE = [&](int s) { return bar0 + 8u * (3 * kSB + kST + s); };      // MMA done with TMEM stage s
    auto D2FULL = [&](int s) { return bar0 + 8u * (3 * kSB + 2 * kST + s); };
    auto D2FREE = [&](int s) { return bar0 + 8u * (3 * kSB + 2 * kST + 2 + s); };
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffBar + kNumBars * 8);

    if (tid == 0) {
        for (int s = 0; s < kSB; ++s) {
            mbar_init(BFULL(s), 32);
            mbar_init(BFREE(s), 1);
            mbar_init(SFREE(s), kComputeWarps * 32);
        }
        for (int s = 0; s < kST; ++s) {
            mbar_init(PFULL(s), kComputeWarps * 32);
            mbar_init(WFREE(s), 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(D2FULL(s), 1);
            mbar_init(D2FREE(s), 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // B2 rows 7..15 stay zero: clear the B2 buffers once
    for (int i = tid; i < kSB * kB2Bytes / 16; i += kThreads)
        reinterpret_cast<float4*>(smem + kOffB2)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (warp == kComputeWarps + kFillWarps) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    const int32_t nblk = (a.n_tgt + kM - 1) / kM;
    const float4 fr = a.frame ? __ldg(a.frame) : make_float4(0.f, 0.f, 0.f, 0.f);

    if (warp < kComputeWarps) {
        // ================================================================ compute
        const int q = warp >> 2, lq = warp & 3, row = lq * 32 + lane;
        const uint32_t tlane = tmem + ((uint32_t)(lq * 32) << 16);
        uint32_t k = 0, Tc = 0;  // running stage / eligible-tile counters of this CTA
        float* red = reinterpret_cast<float*>(smem + kOffRed);
        for (int32_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
            // own target in the block frame
            int64_t it = (int64_t)blk * kM + row;
            const bool valid = it < a.n_tgt;
            if (!valid) it = a.n_tgt - 1;
            const int64_t vid = a.tperm ? (int64_t)__ldg(a.tperm + it) : it;
            const float4 xv = __ldg(reinterpret_cast<const float4*>(a.x) + vid);
            const float4 blo = __ldg(a.blk_box + 2 * blk), bhi = __ldg(a.blk_box + 2 * blk + 1);
            const float xi0 = (xv.x - fr.x) - 0.5f * (blo.x + bhi.x), xi1 = (xv.y - fr.y) - 0.5f * (blo.y + bhi.y),
                        xi2 = (xv.z - fr.z) - 0.5f * (blo.z + bhi.z);
            const f2x mx = pk(-2.f * xi0, -2.f * xi0), my = pk(-2.f * xi1, -2.f * xi1), mz = pk(-2.f * xi2, -2.f * xi2);
            const float si1 = fmaf(xi0, xi0, fmaf(xi1, xi1, xi2 * xi2));
            const f2x si = pk(si1, si1);
            float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f;
            const uint32_t* bits = a.elig + (int64_t)blk * a.words;
            bool pending = false;  // accumulator of tile Tc-1 not yet drained
            auto drain = [&](uint32_t T) {
                // D of eligible tile T -> registers (warpgroup T & 3), FP32 round-to-nearest fold
                if ((int)(T & 3) == q) {
                    const int db = T & 1;
                    mbar_wait(D2FULL(db), (T >> 1) & 1);
                    tc_fence_after();
                    uint32_t d[8];
                    tmem_ld8(tlane + kD2Col + db * 16, d);
                    tmem_wait_ld();
                    tc_fence_before();
                    mbar_arrive(D2FREE(db));
                    const float W = __uint_as_float(d[6]);
                    acc0 += fmaf(xi0, W, -(__uint_as_float(d[0]) + __uint_as_float(d[1])));
                    acc1 += fmaf(xi1, W, -(__uint_as_float(d[2]) + __uint_as_float(d[3])));
                    acc2 += fmaf(xi2, W, -(__uint_as_float(d[4]) + __uint_as_float(d[5])));
                }
            };
            for (int32_t w = 0; w < a.words; ++w) {
                uint32_t m = __ldg(bits + w);
                while (m) {
                    m &= m - 1;  // the tile index itself is not needed here
#pragma unroll 1
                    for (int half = 0; half < 2; ++half) {
                        const int ts = k % kST, sb = k % kSB;
                        mbar_wait(BFULL(sb), (k / kSB) & 1);
                        const float4* sp = reinterpret_cast<const float4*>(smem + kOffSrc + sb * kSrcBytes) + q * 32;
                        uint32_t r[32];
#ifdef MM_TC_DBG_SKIP_POW
#pragma unroll
                        for (int p = 0; p < 32; ++p) r[p] = 0x3f800000u + p + (uint32_t)sp[0].x;
#else
#pragma unroll
                        for (int p = 0; p < 16; ++p) {
#ifdef MM_TC_DBG_NOLDS
                            const float4 P1 = sp[2 * (p & 1)], P2 = sp[2 * (p & 1) + 1];
#else
                            const float4 P1 = sp[2 * p], P2 = sp[2 * p + 1];  // broadcast LDS.128
#endif
                            f2x r2 = add2(pk(P2.z, P2.w), si);
                            r2 = fma2(mz, pk(P2.x, P2.y), r2);
                            r2 = fma2(my, pk(P1.z, P1.w), r2);
                            r2 = fma2(mx, pk(P1.x, P1.y), r2);
                            float ra, rb;
                            upk(r2, ra, rb);
                            const float l0 = lg2_approx(ra), l1 = lg2_approx(rb);
                            float w0, w1;
                            if ((MM_TC_MUFU_MASK >> p) & 1) {
                                float y0, y1;
                                upk(mul_bc(pk(l0, l1), a.cexp), y0, y1);
                                w0 = ex2_approx(y0);
                                w1 = ex2_approx(y1);
                            } else {
                                upk(pow_poly2(pk(l0, l1), a.cexp), w0, w1);
                            }
                            r[2 * p] = __float_as_uint(w0) + 0x1000u;      // TF32 operand: the MMA drops the low 13 bits
                            r[2 * p + 1] = __float_as_uint(w1) + 0x1000u;  // -> round to nearest
                        }
#endif
                        mbar_arrive(SFREE(sb));
                        mbar_wait(WFREE(ts), ((k / kST) & 1) ^ 1);
                        tc_fence_after();
                        tmem_st32(tlane + ts * kN + q * 32, r);
                        tmem_wait_st();
                        tc_fence_before();
                        mbar_arrive(PFULL(ts));
                        ++k;
                        if (half == 0 && pending) {
                            drain(Tc - 1);
                            pending = false;
                        }
                    }
                    pending = true;
                    ++Tc;
                }
            }
            if (pending) drain(Tc - 1);
            // cross-warpgroup reduction in warpgroup order (deterministic), stored at the vertex id
            reinterpret_cast<float4*>(red)[q * kM + row] = make_float4(acc0, acc1, acc2, 0.f);
            asm volatile("bar.sync 1, 512;" ::: "memory");
            if (q == 0 && valid) {
                float4 s = reinterpret_cast<float4*>(red)[row];
#pragma unroll
                for (int g = 1; g < 4; ++g) {
                    const float4 v = reinterpret_cast<float4*>(red)[g * kM + row];
                    s.x += v.x;
                    s.y += v.y;
                    s.z += v.z;
                }
                a.out[vid] = s;
            }
            asm volatile("bar.sync 1, 512;" ::: "memory");
        }
    } else if (warp < kComputeWarps + kFillWarps) {
        // ================================================================ fill
        const int fw = warp - kComputeWarps;
        uint32_t k = 0;
        for (int32_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
            const float4 blo = __ldg(a.blk_box + 2 * blk), bhi = __ldg(a.blk_box + 2 * blk + 1);
            const float cb[3] = {0.5f * (blo.x + bhi.x), 0.5f * (blo.y + bhi.y), 0.5f * (blo.z + bhi.z)};
            const uint32_t* bits = a.elig + (int64_t)blk * a.words;
            for (int32_t w = 0; w < a.words; ++w) {
                uint32_t m = __ldg(bits + w);
                while (m) {
                    const int32_t tile = w * 32 + (__ffs(m) - 1);
                    m &= m - 1;
                    for (int half = 0; half < 2; ++half, ++k) {
                        if ((int)(k % kSB) != fw) continue;
                        // this warp stages 128 sources (4 per lane = one 16-byte K chunk of B2) into buffer fw
                        float4 hi[4], lo[4];
                        const int64_t j0 = (int64_t)tile * kCoarseTile + half * kN + 4 * lane;
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const bool in = j0 + e < a.n_src;
                            hi[e] = in ? __ldg(a.rep_hi + j0 + e) : make_float4(cb[0], cb[1], cb[2], 0.f);
                            lo[e] = (in && a.rep_lo) ? __ldg(a.rep_lo + j0 + e) : make_float4(0.f, 0.f, 0.f, 0.f);
                        }
                        mbar_wait(BFREE(fw), ((k / kSB) & 1) ^ 1);
                        mbar_wait(SFREE(fw), ((k / kSB) & 1) ^ 1);
                        float4* SP = reinterpret_cast<float4*>(smem + kOffSrc + fw * kSrcBytes);
                        float4* B2 = reinterpret_cast<float4*>(smem + kOffB2 + fw * kB2Bytes);
                        float c2[7][4], xs[4][3], ss[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            xs[e][0] = (hi[e].x - cb[0]) - lo[e].x;
                            xs[e][1] = (hi[e].y - cb[1]) - lo[e].y;
                            xs[e][2] = (hi[e].z - cb[2]) - lo[e].z;
                            const float nu = hi[e].w;
                            ss[e] = fmaf(xs[e][0], xs[e][0], fmaf(xs[e][1], xs[e][1], fmaf(xs[e][2], xs[e][2], kEps2)));
#pragma unroll
                            for (int d = 0; d < 3; ++d) split_tf32(nu * xs[e][d], c2[2 * d][e], c2[2 * d + 1][e]);
                            c2[6][e] = nu;
                        }
                        // source pairs (4 lane + 0, 1) and (2, 3): (x0,x1,y0,y1), (z0,z1,s0,s1)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            SP[2 * (2 * lane + h)] = make_float4(xs[2 * h][0], xs[2 * h + 1][0], xs[2 * h][1], xs[2 * h + 1][1]);
                            SP[2 * (2 * lane + h) + 1] = make_float4(xs[2 * h][2], xs[2 * h + 1][2], ss[2 * h], ss[2 * h + 1]);
                        }
                        // B2: row n (column of D), K chunk = lane: 16-byte unit lane * 16 + n
#pragma unroll
                        for (int n = 0; n < 7; ++n) B2[lane * 16 + n] = make_float4(c2[n][0], c2[n][1], c2[n][2], c2[n][3]);
                        fence_async_smem();
                        mbar_arrive(BFULL(fw));
                    }
                }
            }
        }
    } else if (lane == 0) {
        // ================================================================ MMA issue (one thread)
        constexpr uint32_t id2 = idesc_tf32(kM, 16);
        uint32_t k = 0, Tc = 0;
        for (int32_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
            const uint32_t* bits = a.elig + (int64_t)blk * a.words;
            for (int32_t w = 0; w < a.words; ++w) {
                uint32_t m = __ldg(bits + w);
                while (m) {
                    m &= m - 1;
                    for (int half = 0; half < 2; ++half, ++k) {
                        const int ts = k % kST, sb = k % kSB, db = Tc & 1;
                        mbar_wait(BFULL(sb), (k / kSB) & 1);
                        mbar_wait(PFULL(ts), (k / kST) & 1);
                        if (half == 0) mbar_wait(D2FREE(db), ((Tc >> 1) & 1) ^ 1);
                        tc_fence_after();
                        const uint32_t b2 = sbase + kOffB2 + sb * kB2Bytes;
#ifndef MM_TC_DBG_SKIP_MMA2
#pragma unroll 1
                        for (int i = 0; i < kN / 8; ++i)
                            mma_ts(tmem + kD2Col + db * 16, tmem + ts * kN + 8 * i, umma_desc(b2 + i * 512, 256, 128), id2,
                                   (half | i) != 0);
#endif
                        tc_commit(BFREE(sb));
                        tc_commit(WFREE(ts));
                        if (half == 1) tc_commit(D2FULL(db));
                    }
                    ++Tc;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kComputeWarps + kFillWarps) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols));
    }
}

}  // namespace tc
}  // namespace mm
