// k_hier.cuh — host launchers of the hierarchy / centroid / prolongation kernels.
#pragma once
#include "mm_common.cuh"

namespace mm {

cudaError_t run_match_round(int32_t n, int64_t nnz, const int64_t* rp, const int32_t* col, const int32_t* omega,
                            const int32_t* c, int32_t* mate, int32_t* cand, uint64_t seed, int32_t level,
                            int32_t round, int32_t* added, cudaStream_t st);
// all handshake rounds of one level in one cooperative launch; *rounds_out (device) = rounds run;
// added: device int32[2] scratch.  cudaErrorCooperativeLaunchTooLarge: use run_match_round instead
cudaError_t run_match_level(int32_t n, int64_t nnz, const int64_t* rp, const int32_t* col, const int32_t* omega,
                            const int32_t* c, int32_t* mate, int32_t* cand, uint64_t seed, int32_t level,
                            int32_t max_rounds, int32_t* added, int32_t* rounds_out, cudaStream_t st);
cudaError_t launch_fill(int64_t n, int32_t v, int32_t* a, cudaStream_t st);
size_t scan_temp_bytes(int32_t n);
size_t sort_temp_bytes_u64(int64_t m);
size_t sort_temp_bytes_i32(int32_t n);
cudaError_t exclusive_scan_i32(const int32_t* in, int32_t* out, int32_t n, void* tmp, size_t tmp_bytes,
                               cudaStream_t st);
cudaError_t contract_leaders(int32_t n, const int32_t* mate, const int32_t* c, int32_t* flag, int32_t* cid,
                             int32_t* parent, int32_t* c_next, void* tmp, size_t tmp_bytes, cudaStream_t st);
cudaError_t contract_edges(int32_t n, int64_t nnz, const int64_t* rp, const int32_t* col, const int32_t* omega,
                           const int32_t* parent, int32_t nc, uint64_t* keys, uint64_t* keys_alt, int32_t* vals,
                           int32_t* vals_alt, int32_t* head, int32_t* pos, int32_t* ccol_tmp,
                           int32_t* comega_tmp, int32_t* rowcnt, void* tmp, size_t tmp_bytes, cudaStream_t st);
// coarse row_ptr from the row ids of the m2 unique entries (written into `vals` by contract_edges)
cudaError_t rowptr_from_rows(int32_t nc, const int32_t* urow, int64_t m2, int64_t* rp, cudaStream_t st);
// coarse S^l distances / weights (Q7), edge-parallel over the m unique entries with row ids urow
cudaError_t launch_coarse_sset(int64_t m, const int32_t* urow, const int32_t* col, const int32_t* c, int dim,
                               float* d, float* w, cudaStream_t st);
cudaError_t group_by_key(int32_t n, const int32_t* key, int32_t k, int32_t* ptr, int32_t* members,
                         int32_t* key_sorted, int32_t* iota, int32_t* cnt, void* tmp, size_t tmp_bytes,
                         cudaStream_t st);
cudaError_t launch_compose(int32_t n, const int32_t* a, const int32_t* map, int32_t* out, cudaStream_t st);
// Frame origin of kernel (c) (Q28): box = bounding box of x (uint32[6]
// order-preserving scratch); frame->xyz = per-axis origin c with x - c exact in FP32, or 0
cudaError_t launch_frame(int dim, int32_t n, const float* x, uint32_t* box, float4* frame, cudaStream_t st);
// the same in one launch; box must hold the armed state left by launch_frame / a previous fused launch
cudaError_t launch_frame_fused(int dim, int32_t n, const float* x, uint32_t* box, float4* frame, cudaStream_t st);
// Orders for kernel (c) (Q26, Q27) from the positions x (also computes the frame):
//  targets: tperm[slot] = vertex id in Morton order of x (tpos = inverse);
//  representatives: rord[slot] = rep id ordered by (mass nu, Morton key of its centroid),
//  rpos = inverse, tile_nu[t] = common mass of slots [tile t, tile (t+1)) or 0.
// rep_hi/rep_lo are overwritten (centroids by id, used as keys).
// iota[0..max(n,k)) = 0, 1, ...; tkey*: uint32[n]; rkey*: uint64[k]
cudaError_t approx_orders(int dim, int32_t n, int32_t k, const int32_t* mptr, const int32_t* mem, const float* x,
                          int tile, const int32_t* iota, uint32_t* box, float4* frame, float4* rep_hi,
                          float4* rep_lo, uint32_t* tkey, uint32_t* tkey_sorted, int32_t* tperm, int32_t* tpos,
                          uint64_t* rkey, uint64_t* rkey_sorted, int32_t* rord, int32_t* rpos, int32_t* tile_nu,
                          void* tmp, size_t tmp_bytes, cudaStream_t st, int2* sbound = nullptr);
// rord nullable: representative v at slot v; else rep rord[s] is written at slot s.
// mem nullable: the members of a representative are the contiguous range itself
// (renumbered level); sbound nullable: else the member range of each slot.
// frame nullable: coordinates relative to the origin *frame (Q28).
// tile_box nullable: else the box of every `tile` slots is written (kernel (c)'s skip test, Q27)
cudaError_t launch_centroid(int dim, int32_t n, int32_t k, const int32_t* mptr, const int32_t* mem, const float* x,
                            const int32_t* rord, const float4* frame, float4* rep_hi, float4* rep_lo,
                            float4* tile_box, int tile, cudaStream_t st, const int2* sbound = nullptr,
                            const char* name = "centroid");
cudaError_t launch_prolong(int dim, int32_t n, const int32_t* parent, const float* xc, uint64_t seed,
                           int32_t level, float* x, cudaStream_t st);
cudaError_t launch_init_box(int dim, int32_t n, const float* d, int64_t nnz, double* dsum, uint64_t seed,
                            int32_t level, float* x, cudaStream_t st);

// SCLaP (R6): labels -> parent map, coarse weights; *nc_out_dev = number of clusters
cudaError_t contract_labels_gpu(int32_t n, const int32_t* lab, const int32_t* c, int32_t* flag, int32_t* cid,
                                int32_t* parent, int32_t* c_next, int32_t* nc_out_dev, void* tmp, size_t tmp_bytes,
                                cudaStream_t st);
cudaError_t launch_prolong_disc(int dim, int32_t n, const int32_t* parent, const float* xc, const int32_t* c_coarse,
                                uint64_t seed, int32_t level, float* x, cudaStream_t st);
cudaError_t launch_max_i32(int32_t n, const int32_t* a, int32_t* out, cudaStream_t st);
}  // namespace mm
