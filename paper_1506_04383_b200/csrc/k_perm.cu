// k_perm.cu — locality renumbering of a hierarchy level (see k_perm.cuh).
// All integer work: the permutation, the permuted S^l and the sibling map are
// exact; only the order in which kernels visit the vertices changes.
#include "k_perm.cuh"

namespace mm {

namespace {

inline int nblk(int64_t n, int b = 256) { return (int)((n + b - 1) / b); }

constexpr int kScanThreads = 256, kScanPer = 16, kScanChunk = kScanThreads * kScanPer;  // 4096 per block

// block-wide exclusive scan of one int64 per thread; returns the block total
__device__ __forceinline__ int64_t block_scan_excl(int64_t v, int64_t* warp_tot, int64_t& total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int64_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) warp_tot[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        int64_t w = lane < (kScanThreads / 32) ? warp_tot[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t t = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += t;
        }
        if (lane < (kScanThreads / 32)) warp_tot[lane] = w;  // inclusive
    }
    __syncthreads();
    const int64_t before = wid > 0 ? warp_tot[wid - 1] : 0;
    total = warp_tot[kScanThreads / 32 - 1];
    __syncthreads();
    return before + inc - v;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_sums(const int32_t* __restrict__ in, int64_t n,
                                                            int64_t* __restrict__ bsum) {
    __shared__ int64_t wt[kScanThreads / 32];
    const int64_t base = (int64_t)blockIdx.x * kScanChunk;
    int64_t s = 0;
#pragma unroll
    for (int t = 0; t < kScanPer; ++t) {
        const int64_t i = base + (int64_t)t * kScanThreads + threadIdx.x;  // coalesced
        if (i < n) s += in[i];
    }
    int64_t tot;
    block_scan_excl(s, wt, tot);
    if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

// one block: exclusive scan of the nb block sums, in place; bsum[nb] = total
__global__ void __launch_bounds__(kScanThreads) k_scan_top(int64_t* __restrict__ bsum, int64_t nb) {
    __shared__ int64_t wt[kScanThreads / 32];
    int64_t carry = 0;
    for (int64_t b0 = 0; b0 < nb; b0 += kScanThreads) {
        const int64_t i = b0 + threadIdx.x;
        const int64_t v = i < nb ? bsum[i] : 0;
        int64_t tot;
        const int64_t ex = block_scan_excl(v, wt, tot);
        if (i < nb) bsum[i] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) bsum[nb] = carry;
}

template <typename OutT>
__global__ void __launch_bounds__(kScanThreads) k_scan_out(const int32_t* __restrict__ in, int64_t n,
                                                           const int64_t* __restrict__ bsum, OutT* __restrict__ out) {
    // padded staging (one skip word per 32) so that each thread's 16 consecutive
    // inputs are read without bank conflicts
    __shared__ int32_t buf[kScanChunk + kScanChunk / 32];
    __shared__ int64_t wt[kScanThreads / 32];
    const int64_t base = (int64_t)blockIdx.x * kScanChunk;
#pragma unroll
    for (int t = 0; t < kScanPer; ++t) {
        const int j = t * kScanThreads + threadIdx.x;
        const int64_t i = base + j;
        buf[j + (j >> 5)] = i < n ? in[i] : 0;
    }
    __syncthreads();
    int64_t s = 0;
    int32_t v[kScanPer];
#pragma unroll
    for (int t = 0; t < kScanPer; ++t) {
        const int j = threadIdx.x * kScanPer + t;
        v[t] = buf[j + (j >> 5)];
        s += v[t];
    }
    int64_t tot;
    int64_t run = bsum[blockIdx.x] + block_scan_excl(s, wt, tot);
#pragma unroll
    for (int t = 0; t < kScanPer; ++t) {
        const int64_t i = base + (int64_t)threadIdx.x * kScanPer + t;
        if (i < n) out[i] = (OutT)run;
        run += v[t];
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = (OutT)bsum[gridDim.x];
}

__global__ void k_slot_counts(int32_t k, const int32_t* __restrict__ rord, const int32_t* __restrict__ mptr,
                              int32_t* __restrict__ cnt) {
    const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= k) return;
    const int32_t r = rord[s];
    cnt[s] = mptr[r + 1] - mptr[r];
}

// one warp per slot: members copied in their (ascending id) order
__global__ void k_slot_fill(int32_t k, const int32_t* __restrict__ rord, const int32_t* __restrict__ mptr,
                            const int32_t* __restrict__ mem, const int32_t* __restrict__ sptr,
                            int32_t* __restrict__ perm, int32_t* __restrict__ inv, int32_t* __restrict__ anc_new) {
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (gw >= k) return;
    const int32_t s = (int32_t)gw, r = rord[s];
    const int32_t b = mptr[r], e = mptr[r + 1], o = sptr[s];
    for (int32_t t = lane; t < e - b; t += 32) {
        const int32_t v = mem[b + t];
        perm[o + t] = v;
        inv[v] = o + t;
        anc_new[o + t] = s;
    }
}

__global__ void k_row_lengths(int32_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ perm,
                              int32_t* __restrict__ len) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t o = perm[i];
    len[i] = (int32_t)(rp[o + 1] - rp[o]);
}

// one warp per new row
__global__ void k_permute_rows(int32_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                               const float* __restrict__ d, const float* __restrict__ w,
                               const int32_t* __restrict__ perm, const int32_t* __restrict__ inv,
                               const int64_t* __restrict__ rp2, int32_t* __restrict__ col2, float* __restrict__ d2,
                               float* __restrict__ w2) {
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (gw >= n) return;
    const int32_t o = perm[gw];
    const int64_t b = rp[o], e = rp[o + 1], b2 = rp2[gw];
    for (int64_t t = lane; t < e - b; t += 32) {
        col2[b2 + t] = inv[col[b + t]];
        d2[b2 + t] = d[b + t];
        w2[b2 + t] = w[b + t];
    }
}

template <int DIM>
__global__ void k_permute_x(int32_t n, const int32_t* __restrict__ perm, const float* __restrict__ x,
                            float* __restrict__ y, bool scatter) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t o = perm[i];
    if (scatter) store_x<DIM>(y, o, load_x<DIM>(x, i));
    else store_x<DIM>(y, i, load_x<DIM>(x, o));
}

__global__ void k_gather_i32(int32_t n, const int32_t* __restrict__ perm, const int32_t* __restrict__ a,
                             int32_t* __restrict__ out) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = a[perm[i]];
}

__global__ void k_sibling(int32_t np, const int32_t* __restrict__ cptr, const int32_t* __restrict__ child,
                          int32_t* __restrict__ sib) {
    const int32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= np) return;
    const int32_t b = cptr[p], e = cptr[p + 1];
    if (e - b == 2) {
        sib[child[b]] = child[b + 1];
        sib[child[b + 1]] = child[b];
    } else {
        for (int32_t c = b; c < e; ++c) sib[child[c]] = (e - b == 1) ? -1 : -2;
    }
}

}  // namespace

size_t perm_scan_tmp_bytes(int64_t n) {
    const int64_t nb = (n + kScanChunk - 1) / kScanChunk;
    return (size_t)(nb + 1) * sizeof(int64_t);
}

template <typename OutT>
cudaError_t scan_i32_excl(const int32_t* in, OutT* out, int64_t n, void* tmp, cudaStream_t st) {
    LaunchScope ls("perm_scan", st);
    int64_t* bsum = static_cast<int64_t*>(tmp);
    const int64_t nb = std::max<int64_t>(1, (n + kScanChunk - 1) / kScanChunk);
    k_scan_sums<<<(unsigned)nb, kScanThreads, 0, st>>>(in, n, bsum);
    k_scan_top<<<1, kScanThreads, 0, st>>>(bsum, nb);
    k_scan_out<OutT><<<(unsigned)nb, kScanThreads, 0, st>>>(in, n, bsum, out);
    return cudaGetLastError();
}
template cudaError_t scan_i32_excl<int32_t>(const int32_t*, int32_t*, int64_t, void*, cudaStream_t);
template cudaError_t scan_i32_excl<int64_t>(const int32_t*, int64_t*, int64_t, void*, cudaStream_t);

cudaError_t level_perm(int32_t k, const int32_t* rord, const int32_t* mptr, const int32_t* mem, int32_t* cnt,
                       int32_t* sptr, int32_t* perm, int32_t* inv, int32_t* anc_new, void* tmp, cudaStream_t st) {
    {
        LaunchScope ls("perm_level", st);
        k_slot_counts<<<nblk(k), 256, 0, st>>>(k, rord, mptr, cnt);
    }
    cudaError_t e = scan_i32_excl<int32_t>(cnt, sptr, k, tmp, st);
    if (e != cudaSuccess) return e;
    LaunchScope ls("perm_level", st);
    k_slot_fill<<<nblk((int64_t)k * 32), 256, 0, st>>>(k, rord, mptr, mem, sptr, perm, inv, anc_new);
    return cudaGetLastError();
}

cudaError_t permute_sset(int32_t n, const int64_t* rp, const int32_t* col, const float* d, const float* w,
                         const int32_t* perm, const int32_t* inv, int64_t* rp2, int32_t* col2, float* d2, float* w2,
                         int32_t* len, void* tmp, cudaStream_t st) {
    {
        LaunchScope ls("perm_sset", st);
        k_row_lengths<<<nblk(n), 256, 0, st>>>(n, rp, perm, len);
    }
    cudaError_t e = scan_i32_excl<int64_t>(len, rp2, n, tmp, st);
    if (e != cudaSuccess) return e;
    LaunchScope ls("perm_sset", st);
    k_permute_rows<<<nblk((int64_t)n * 32), 256, 0, st>>>(n, rp, col, d, w, perm, inv, rp2, col2, d2, w2);
    return cudaGetLastError();
}

cudaError_t permute_x(int dim, int32_t n, const int32_t* perm, const float* x, float* y, bool scatter,
                      cudaStream_t st) {
    LaunchScope ls("perm_x", st);
    if (dim == 2) k_permute_x<2><<<nblk(n), 256, 0, st>>>(n, perm, x, y, scatter);
    else k_permute_x<3><<<nblk(n), 256, 0, st>>>(n, perm, x, y, scatter);
    return cudaGetLastError();
}

cudaError_t gather_i32(int32_t n, const int32_t* perm, const int32_t* a, int32_t* out, cudaStream_t st) {
    LaunchScope ls("perm_x", st);
    k_gather_i32<<<nblk(n), 256, 0, st>>>(n, perm, a, out);
    return cudaGetLastError();
}

cudaError_t sibling_of(int32_t np, const int32_t* cptr, const int32_t* child, int32_t* sib, cudaStream_t st) {
    LaunchScope ls("sibling", st);
    k_sibling<<<nblk(np), 256, 0, st>>>(np, cptr, child, sib);
    return cudaGetLastError();
}

}  // namespace mm
