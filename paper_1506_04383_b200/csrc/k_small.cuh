// k_small.cuh — the persistent small-level kernel (all sweeps of one level in one launch).
#pragma once
#include "mm_common.cuh"
#include "../../include/mm.h"

namespace mm {

struct SmallArgs {
    int32_t n = 0, k = 0;  // k > 0: Eq.(3) with k representatives
    const int64_t* rp = nullptr;
    const int32_t* col = nullptr;
    const float* d = nullptr;
    const float* w = nullptr;
    const float* x0 = nullptr;  // input coordinates (sweep 1 reads x0, writes x1, then ping-pong)
    float* x1 = nullptr;
    float q = 0.f;
    // Eq.(3) maps (from prepare_approx): members of each representative, children of each parent
    const int32_t* anc = nullptr;
    const int32_t* parent = nullptr;
    const int32_t* mptr = nullptr;
    const int32_t* mem = nullptr;
    const int32_t* cptr = nullptr;
    const int32_t* child = nullptr;
    float4* rep_hi = nullptr;
    float4* rep_lo = nullptr;
    // sweeps: mode 0 = K sweeps at alpha0; mode 1 = the schedule
    int32_t mode = 0, K = 0;
    double alpha0 = 0, alpha_min = 0, factor = 0, eps = 0;
    int32_t rounds = 0, max_final = 0;
    double* partial = nullptr;       // [2][grid][4] (sweep parity)
    int32_t* result = nullptr;       // device int32[3]: sweeps, error, result buffer (1 = x1)
    mm_sweep_stats* stats = nullptr; // the last sweep's statistics (nullable)
};

// does a level qualify (sizes, shared memory; MM_SMALL_N caps n, 0 disables)
bool small_level_ok(int dim, int32_t n, int32_t k, bool approx);
int small_level_partials(int32_t n);  // doubles needed in `partial` / 4
cudaError_t launch_small_level(int dim, bool approx, const SmallArgs& a, cudaStream_t st);

}  // namespace mm
