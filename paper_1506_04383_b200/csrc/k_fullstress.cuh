// k_fullstress.cuh — host launchers of the full-stress metric kernel.
#pragma once
#include <algorithm>

#include "mm_common.cuh"

namespace mm {
size_t full_stress_smem(int32_t n);
int full_stress_grid(int32_t n);
cudaError_t launch_full_stress(int dim, int32_t n, const int64_t* rp, const int32_t* col, const float* x, int grid,
                               int32_t* qbuf, double* partial, cudaStream_t st);
}  // namespace mm
