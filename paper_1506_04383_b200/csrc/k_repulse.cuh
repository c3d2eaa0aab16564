// k_repulse.cuh — host-side launch plans for the tiled all-pairs kernels.
#pragma once
#include <algorithm>

#include "mm_common.cuh"

namespace mm {

struct RepulsePlan {
    int tblocks = 1;   // CTAs along targets
    int P = 1;         // source chunks (grid.y) = number of partial-sum slices
    int32_t chunk = 0; // sources per chunk
};
struct EntropyPlan {
    int tblocks = 1;
    int P = 1;
    int32_t chunk = 0;
};

RepulsePlan plan_repulse(int32_t n_tgt, int32_t n_src, int dim);
cudaError_t launch_repulse(int dim, bool qpow, bool coarse, float q, int32_t n_tgt, const float* x,
                           int32_t n_src, const float4* reps, const int32_t* anc, const RepulsePlan& p,
                           float* part, cudaStream_t st);
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
    const float* part;   // [P][n] stride 2 (dim 2) or 4 (dim 3)
    int P;
    // Eq.(3) sibling term (nullable: exact mode)
    const int32_t* parent;
    const int32_t* child_ptr;
    const int32_t* child;
    float* x_out;
    double* stat_partial; // [nblocks][3]
    int32_t* flags;       // device int (OR-ed)
};
int gather_blocks(int32_t n, double mean_row);
cudaError_t launch_gather(int dim, const GatherArgs& a, double mean_row, cudaStream_t st);
cudaError_t launch_stats_final(const double* partial, int nblocks, const int32_t* flags, mm_sweep_stats* out,
                               cudaStream_t st);
// energy S part: per-row stress and S-pair phi sums -> partial[nblocks][2]; coincident S-pairs counted
cudaError_t launch_energy_s(int dim, double q, int32_t n, const int64_t* rp, const int32_t* col, const float* d,
                            const float* w, const float* x, double mean_row, double* partial, int32_t* coinc,
                            cudaStream_t st);

}  // namespace mm
