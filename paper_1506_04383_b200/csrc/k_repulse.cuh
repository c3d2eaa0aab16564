// k_repulse.cuh — host-side launch plans for the tiled all-pairs kernels.
#pragma once
#include <algorithm>

#include "mm_common.cuh"

namespace mm {

// Static persistent schedule of the all-pairs kernels: the (target block,
// source tile) space of U = TB * Ub work units is split into G contiguous
// ranges [g*U/G, (g+1)*U/G).  Requires G <= U (every range non-empty).
struct Sched {
    int64_t U = 1;
    int32_t Ub = 1;   // source tiles per target block
    int32_t TB = 1;   // target blocks
    int32_t G = 1;    // CTAs
};
#ifndef MM_FASTDIV
#define MM_FASTDIV 1
#endif
// floor(a / b) for 0 <= a < 2^53, b > 0.  On the device the quotient comes from
// an FP64 division (a and b exact in double; the rounded quotient is within
// one of the true one) plus one integer correction step: exact, and far cheaper
// than the 64-bit integer division routine (kernel (a) evaluates three per vertex).
__host__ __device__ __forceinline__ int64_t floor_div_nonneg(int64_t a, int64_t b) {
#if defined(__CUDA_ARCH__) && MM_FASTDIV
    int64_t q = (int64_t)((double)a / (double)b);
    if (q * b > a) --q;
    else if ((q + 1) * b <= a) ++q;
    return q;
#else
    return a / b;
#endif
}
// first CTA whose range contains work unit a: max{g : floor(g U / G) <= a}
__host__ __device__ __forceinline__ int32_t sched_first_cta(int64_t a, const Sched& s) {
    return (int32_t)floor_div_nonneg((a + 1) * (int64_t)s.G - 1, s.U);
}

struct RepulsePlan {
    Sched sch;
    int slots = 1;     // max partial slots per target (size of the partial buffer / n)
};
// Triangular schedule of the unordered-pair entropy kernel: target block tb
// owns source tiles [tb*c, Ub) (c = tiles per target block); prefix(tb) =
// sum_{t<tb} (Ub - t c) = tb Ub - c tb (tb-1) / 2.
struct TriSched {
    int64_t U = 1;
    int32_t Ub = 1, TB = 1, c = 1, G = 1;
};
__host__ __device__ __forceinline__ int64_t tri_prefix(int32_t tb, const TriSched& s) {
    return (int64_t)tb * s.Ub - (int64_t)s.c * tb * (tb - 1) / 2;
}
// first CTA whose range of a triangular schedule contains unit a (same rule as sched_first_cta)
__host__ __device__ __forceinline__ int32_t sched_first_cta_tri(int64_t a, const TriSched& s) {
    return (int32_t)floor_div_nonneg((a + 1) * (int64_t)s.G - 1, s.U);
}
struct SymPlan {
    TriSched ts;        // blocks of 1024 vertices; units = (block pair (I, J >= I), source sub-tile)
    int slots = 1;      // max i-side partial slots per vertex
    int64_t full_grid;  // resident CTAs of a full wave (148 x occupancy); ts.G = min(full_grid, U)
};
SymPlan plan_repulse_sym(int32_t n, int dim);
int64_t sym_jpart_rows(const SymPlan& p);  // rows I of jpart[I][n] (blocks 0..TB-2)
cudaError_t launch_repulse_sym(int dim, bool qpow, float q, int32_t n, const float* x, const SymPlan& p,
                               float* ipart, float* jpart, cudaStream_t st);
struct EntropyPlan {
    TriSched ts;
    int nblocks = 1;   // CTAs = FP64 partials
};

// Orders / metadata of kernel (c) (all nullable; Q26, Q27)
struct CoarseOrder {
    const int32_t* tperm = nullptr;    // target slot -> vertex id (spatial order); partials are written at the vertex id
    const int32_t* tile_nu = nullptr;  // [ceil(k/256)] common mass nu of a source tile, or 0 (mixed)
    const float4* tile_box = nullptr;  // [2 ceil(k/256)] box of a tile's hi coordinates (.w of [0]: max |coord|)
    const float4* frame = nullptr;     // origin c: targets are x - c (exact, Q28); representatives are frame-relative
};
RepulsePlan plan_repulse(int32_t n_tgt, int32_t n_src, int dim, bool coarse, bool qpow);
int repulse_targets_per_block(int dim);
cudaError_t launch_repulse(int dim, bool qpow, bool coarse, float q, int32_t n_tgt, const float* x,
                           int32_t n_src, const float4* rep_hi, const float4* rep_lo, const CoarseOrder& co,
                           const RepulsePlan& p, float* part, cudaStream_t st);
// sources per tile of the coarse kernel (granularity of tile_nu)
constexpr int kCoarseTile = 256;
EntropyPlan plan_entropy(int32_t n);
cudaError_t launch_entropy_all(int dim, double q, int32_t n, const float* x, const EntropyPlan& p,
                               double* partial, int32_t* coinc, cudaStream_t st);

// k_gather.cu
struct GatherArgs {
    int32_t n;
    const int64_t* rp;
    const int32_t* col;
    const float* d;
    const float* w;
    const float* x;
    float alpha;
    float q;
    const double* alpha_dev = nullptr;  // non-NULL: alpha read from device memory (device-driven schedule)
    const float* part;   // [slots][n] stride 2 (dim 2) or 4 (dim 3)
    Sched sch;           // schedule that produced `part` (slot count per target block)
    int tpb;             // targets per block of that schedule
    // symmetric exact mode (k_repulse_sym): i-side slots follow the triangular
    // schedule `tri`; jpart[I][i] for I < block(i) holds the j-side sums
    const float* jpart = nullptr;  // nullable: rectangular schedule
    TriSched tri;
    // Eq.(3) own-representative term, subtracted because kernel (c) sums over
    // all k representatives (nullable: exact mode)
    const int32_t* anc = nullptr;
    const int32_t* rpos = nullptr;  // nullable: slot of representative v in rep_hi/rep_lo (mass order)
    const int32_t* tpos = nullptr;  // nullable: slot of vertex i in kernel (c)'s schedule (spatial order)
    const float4* frame = nullptr;  // nullable: origin of the frame-relative representatives (Q28)
    const float4* rep_hi = nullptr;
    const float4* rep_lo = nullptr;
    // Eq.(3) sibling term (nullable: exact mode)
    const int32_t* parent;
    const int32_t* child_ptr;
    const int32_t* child;
    // nullable: per-vertex sibling (>= 0: the only other child of its parent;
    // -1: none; -2: larger family, walk child_ptr/child) from the renumbered level
    const int32_t* sib = nullptr;
    float* x_out;
    double* stat_partial; // [nblocks][3]
    int32_t* flags;       // device int (OR-ed); re-armed to 0 by the last CTA
    int32_t* ticket;      // device int, 0 between launches (last-CTA-done counter)
    mm_sweep_stats* stats; // nullable: final fixed-order reduction target
};
int gather_blocks(int32_t n, double mean_row);
cudaError_t launch_gather(int dim, const GatherArgs& a, double mean_row, cudaStream_t st);
cudaError_t launch_stats_final(const double* partial, int nblocks, const int32_t* flags, mm_sweep_stats* out,
                               cudaStream_t st);
// energy S part: per-row stress and S-pair phi sums -> partial[nblocks][2]; coincident S-pairs counted
cudaError_t launch_energy_s(int dim, double q, int32_t n, const int64_t* rp, const int32_t* col, const float* d,
                            const float* w, const float* x, double mean_row, double* partial, int32_t* coinc,
                            cudaStream_t st);

cudaError_t launch_validate_sset(int32_t n, const int64_t* rp, const int32_t* col, const float* d, const float* w,
                                 int64_t nnz, int32_t* bad, cudaStream_t st);
}  // namespace mm
