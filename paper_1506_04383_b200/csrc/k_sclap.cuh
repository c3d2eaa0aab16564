// k_sclap.cuh — SCLaP clustering (reading R6) on the GPU.
#pragma once
#include <algorithm>

#include "mm_common.cuh"

namespace mm {
// labels of one SCLaP clustering of (n, rp, col, omega, c) with size bound U;
// `alloc`/`dealloc` give stream-ordered scratch.  Syncs a few times per round.
cudaError_t sclap_labels_gpu(int32_t n, int64_t nnz, const int64_t* rp, const int32_t* col, const int32_t* omega,
                             const int32_t* c, long long U, int32_t rounds, uint64_t seed, int32_t level,
                             int32_t* lab, int32_t* rounds_used, cudaStream_t st, void* (*alloc)(size_t, cudaStream_t),
                             void (*dealloc)(void*, cudaStream_t));
}  // namespace mm
