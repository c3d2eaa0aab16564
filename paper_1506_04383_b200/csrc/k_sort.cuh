// k_sort.cuh — hand-written stable LSD radix sort of (key, int32 value) pairs
// for the per-sweep / per-level orders of kernel (c) (Q26/Q27) and
// the grouping of vertices by representative / parent.
#pragma once
#include "mm_common.cuh"

namespace mm {

// scratch bytes for n pairs of key type K (uint32_t or uint64_t)
template <typename K>
size_t radix_sort_tmp_bytes(int64_t n);

// Stable sort of (kin[i], vin[i]) by bits [begin_bit, end_bit) of the key into
// (kout, vout); 8-bit digits, one histogram / scan / scatter per digit.  Equal
// keys keep their input order.  kin/vin are not modified (kout/vout must not
// alias them).  tmp: radix_sort_tmp_bytes<K>(n) bytes, 256-B aligned.
template <typename K>
cudaError_t radix_sort_pairs(const K* kin, K* kout, const int32_t* vin, int32_t* vout, int64_t n, int begin_bit,
                             int end_bit, void* tmp, size_t tmp_bytes, cudaStream_t st, const char* name);

}  // namespace mm
