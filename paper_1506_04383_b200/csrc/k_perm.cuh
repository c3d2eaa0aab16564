// k_perm.cuh — locality renumbering of one hierarchy level for its Eq.(3)
// sweeps (DESIGN.md §4 "Locality renumbering"): the vertices of a level are
// put in the order of kernel (c)'s representative slots, so the members of
// every representative are contiguous (centroid refresh = coalesced reads of a
// contiguous range) and the own-representative index is non-decreasing.  The
// driver permutes S^l, x, parent and ancestor into this order before the
// level's sweeps and scatters x back afterwards; maps and coordinates at the
// C-ABI stay in the canonical numbering.
#pragma once
#include "mm_common.cuh"

namespace mm {

// bytes of scratch for scan_i32_excl over n inputs
size_t perm_scan_tmp_bytes(int64_t n);
// out[i] = sum_{t < i} in[t] for i = 0..n (n + 1 outputs; out[n] = total).
// Hand-written three-phase block scan (block sums, one-block scan of the
// sums, block re-scan); OutT = int32_t or int64_t.
template <typename OutT>
cudaError_t scan_i32_excl(const int32_t* in, OutT* out, int64_t n, void* tmp, cudaStream_t st);

// The level permutation from the representative orders: slot s holds rep
// r = rord[s] with members mem[mptr[r] .. mptr[r+1]) (ascending ids).
// perm[new] = old, inv[old] = new, anc_new[new] = s (the slot, so kernel (c)'s
// rord / rpos become the identity after re-grouping).  cnt: int32[k] scratch,
// sptr: int32[k + 1] scratch.
cudaError_t level_perm(int32_t k, const int32_t* rord, const int32_t* mptr, const int32_t* mem, int32_t* cnt,
                       int32_t* sptr, int32_t* perm, int32_t* inv, int32_t* anc_new, void* tmp, cudaStream_t st);
// S rows in the new order: row new = row perm[new] with columns mapped
// through inv; entries keep their order within the row.  len: int32[n] scratch.
cudaError_t permute_sset(int32_t n, const int64_t* rp, const int32_t* col, const float* d, const float* w,
                         const int32_t* perm, const int32_t* inv, int64_t* rp2, int32_t* col2, float* d2, float* w2,
                         int32_t* len, void* tmp, cudaStream_t st);
// coordinates: gather y[i] = x[perm[i]] (scatter = false) or scatter y[perm[i]] = x[i]
cudaError_t permute_x(int dim, int32_t n, const int32_t* perm, const float* x, float* y, bool scatter,
                      cudaStream_t st);
// out[i] = a[perm[i]]
cudaError_t gather_i32(int32_t n, const int32_t* perm, const int32_t* a, int32_t* out, cudaStream_t st);
// sib[v] for the children lists (cptr, child) of np parents: the other child
// when the parent has exactly two, -1 for an only child, -2 for larger
// families (the gather then walks the child list)
cudaError_t sibling_of(int32_t np, const int32_t* cptr, const int32_t* child, int32_t* sib, cudaStream_t st);

}  // namespace mm
