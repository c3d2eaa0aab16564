// k_sclap.cu — SCLaP clustering on the GPU
// in the synchronous reading R6 of DESIGN.md §3, integer-exact and therefore
// bit-identical to oracle/sclap.c.  One round:
//   1. score_v(L) = sum of omega(v,u) over neighbours with label L: edge keys
//      (v << 32 | label(u)) -> radix sort -> reduce by key;
//   2. warp per node: own score s0, best admissible label L < label(v) with
//      cw(L) + c(v) <= U by (score desc, hash desc, L asc); request if > s0;
//   3. requests ordered per target label by (gain desc, hash desc, v asc) with
//      three stable radix sorts; segmented prefix sums of c; a request is
//      accepted iff cw(L) + prefix <= U (the longest fitting prefix);
//   4. apply, recompute cluster weights (integer atomics: order-free).
#include <cub/cub.cuh>

#include "k_sclap.cuh"

namespace mm {
namespace {

constexpr uint64_t kTagLP = 0x4c505250ULL;  // "LPRP"

__device__ __forceinline__ uint64_t lp_hash(uint64_t seed, int32_t level, int32_t round, int32_t v, int32_t L) {
    uint64_t k = mix64(seed ^ kTagLP);
    k = mix64(k ^ (uint64_t)level);
    k = mix64(k ^ (uint64_t)round);
    return mix64(k ^ (((uint64_t)(uint32_t)v << 32) | (uint32_t)L));
}

inline int nblk(int64_t n, int b = 256) { return (int)((n + b - 1) / b); }

__global__ void k_lp_init(int32_t n, const int32_t* __restrict__ c, int32_t* __restrict__ lab,
                          long long* __restrict__ cw) {
    const int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n) return;
    lab[v] = v;
    cw[v] = c[v];
}

// edge keys: warp per row
__global__ void k_lp_keys(int32_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                          const int32_t* __restrict__ omega, const int32_t* __restrict__ lab,
                          uint64_t* __restrict__ keys, int32_t* __restrict__ vals) {
    const int32_t v = (int32_t)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (v >= n) return;
    for (int64_t e = rp[v] + lane; e < rp[v + 1]; e += 32) {
        const int32_t u = col[e];
        keys[e] = ((uint64_t)(uint32_t)v << 32) | (uint32_t)lab[u];
        vals[e] = omega ? omega[e] : 1;
    }
}

struct LpCand {
    int32_t L;
    long long s;
    uint64_t h;
};
__device__ __forceinline__ bool lp_better(const LpCand& a, const LpCand& b) {
    if (a.L < 0) return false;
    if (b.L < 0) return true;
    if (a.s != b.s) return a.s > b.s;
    if (a.h != b.h) return a.h > b.h;
    return a.L < b.L;
}

// warp per node: choose the request from the node's (label, score) runs
__global__ void k_lp_choose(int32_t n, const uint64_t* __restrict__ ukeys, const int32_t* __restrict__ uscore,
                            int64_t m, const int32_t* __restrict__ lab, const long long* __restrict__ cw,
                            const int32_t* __restrict__ c, long long U, uint64_t seed, int32_t level, int32_t round,
                            int32_t* __restrict__ req_flag, int32_t* __restrict__ req_L,
                            long long* __restrict__ req_gain, uint64_t* __restrict__ req_h) {
    const int32_t v = (int32_t)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (v >= n) return;
    // run [lo, hi) of node v in the unique keys (sorted by v, then label)
    const uint64_t k0 = (uint64_t)(uint32_t)v << 32, k1 = (uint64_t)(uint32_t)(v + 1) << 32;
    int64_t lo = 0, hi = m;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (ukeys[mid] < k0) lo = mid + 1; else hi = mid;
    }
    int64_t end = lo, top = m;
    while (end < top) {
        const int64_t mid = (end + top) >> 1;
        if (ukeys[mid] < k1) end = mid + 1; else top = mid;
    }
    const int32_t my = lab[v];
    const long long cv = c[v];
    long long s0 = 0;
    LpCand best{-1, 0, 0};
    for (int64_t t = lo + lane; t < end; t += 32) {
        const int32_t L = (int32_t)(uint32_t)(ukeys[t] & 0xffffffffULL);
        const long long s = uscore[t];
        if (L == my) {
            s0 = s;
            continue;
        }
        if (L >= my || cw[L] + cv > U) continue;
        const LpCand cand{L, s, lp_hash(seed, level, round, v, L)};
        if (lp_better(cand, best)) best = cand;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        LpCand other;
        other.L = __shfl_xor_sync(0xffffffffu, best.L, o);
        other.s = __shfl_xor_sync(0xffffffffu, best.s, o);
        other.h = __shfl_xor_sync(0xffffffffu, best.h, o);
        if (lp_better(other, best)) best = other;
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);  // exactly one lane holds the own-label score
    }
    if (lane == 0) {
        const bool rq = best.L >= 0 && best.s > s0;
        req_flag[v] = rq ? 1 : 0;
        req_L[v] = best.L;
        req_gain[v] = rq ? best.s - s0 : 0;
        req_h[v] = best.h;
    }
}

// compact requests (pos = exclusive scan of flags); sort keys for the stable passes
__global__ void k_lp_compact(int32_t n, const int32_t* __restrict__ flag, const int32_t* __restrict__ pos,
                             const int32_t* __restrict__ req_L, const long long* __restrict__ req_gain,
                             const uint64_t* __restrict__ req_h, int32_t* __restrict__ idx,
                             uint64_t* __restrict__ key_h, uint64_t* __restrict__ key_g) {
    const int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n || !flag[v]) return;
    const int32_t p = pos[v];
    idx[p] = v;                                            // ascending v (scan order)
    key_h[p] = ~req_h[v];                                  // hash descending
    key_g[p] = (uint64_t)(0x7fffffffffffffffLL - req_gain[v]);  // gain descending
    (void)req_L;
}

__global__ void k_lp_gather_keys(int32_t r, const int32_t* __restrict__ idx, const uint64_t* __restrict__ req_h,
                                 const long long* __restrict__ req_gain, const int32_t* __restrict__ req_L,
                                 int which, uint64_t* __restrict__ key) {
    const int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= r) return;
    const int32_t v = idx[t];
    if (which == 0) key[t] = (uint64_t)(0x7fffffffffffffffLL - req_gain[v]);
    else key[t] = (uint64_t)(uint32_t)req_L[v];
    (void)req_h;
}

__global__ void k_lp_segvals(int32_t r, const int32_t* __restrict__ idx, const int32_t* __restrict__ req_L,
                             const int32_t* __restrict__ c, long long* __restrict__ cval, int32_t* __restrict__ headpos) {
    const int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= r) return;
    const int32_t v = idx[t];
    cval[t] = c[v];
    headpos[t] = (t == 0 || req_L[idx[t - 1]] != req_L[v]) ? t : 0;
}

__global__ void k_lp_apply(int32_t r, const int32_t* __restrict__ idx, const int32_t* __restrict__ req_L,
                           const long long* __restrict__ incl, const int32_t* __restrict__ segstart,
                           const long long* __restrict__ cw, long long U, int32_t* __restrict__ lab,
                           int32_t* __restrict__ moved) {
    const int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    int hit = 0;
    if (t < r) {
        const int32_t v = idx[t];
        const int32_t L = req_L[v];
        const int32_t s0 = segstart[t];
        const long long prefix = incl[t] - (s0 > 0 ? incl[s0 - 1] : 0);
        if (cw[L] + prefix <= U) {
            lab[v] = L;
            hit = 1;
        }
    }
    hit = __reduce_add_sync(0xffffffffu, hit);
    if ((threadIdx.x & 31) == 0 && hit) atomicAdd(moved, hit);
}

__global__ void k_lp_weights(int32_t n, const int32_t* __restrict__ lab, const int32_t* __restrict__ c,
                             long long* __restrict__ cw) {
    const int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v < n) atomicAdd((unsigned long long*)(cw + lab[v]), (unsigned long long)c[v]);
}

struct MaxOp {
    __device__ __forceinline__ int32_t operator()(int32_t a, int32_t b) const { return a > b ? a : b; }
};

}  // namespace

cudaError_t sclap_labels_gpu(int32_t n, int64_t nnz, const int64_t* rp, const int32_t* col, const int32_t* omega,
                             const int32_t* c, long long U, int32_t rounds, uint64_t seed, int32_t level,
                             int32_t* lab, int32_t* rounds_used, cudaStream_t st, void* (*alloc)(size_t, cudaStream_t),
                             void (*dealloc)(void*, cudaStream_t)) {
    const int64_t m0 = std::max<int64_t>(nnz, 1);
    // scratch
    size_t tmp_b = 0, t2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, t2, (uint64_t*)nullptr, (uint64_t*)nullptr, (int32_t*)nullptr,
                                    (int32_t*)nullptr, m0);
    tmp_b = std::max(tmp_b, t2);
    cub::DeviceReduce::ReduceByKey(nullptr, t2, (uint64_t*)nullptr, (uint64_t*)nullptr, (int32_t*)nullptr,
                                   (int32_t*)nullptr, (int64_t*)nullptr, cub::Sum(), m0);
    tmp_b = std::max(tmp_b, t2);
    cub::DeviceScan::ExclusiveSum(nullptr, t2, (int32_t*)nullptr, (int32_t*)nullptr, n + 1);
    tmp_b = std::max(tmp_b, t2);
    cub::DeviceScan::InclusiveSum(nullptr, t2, (long long*)nullptr, (long long*)nullptr, n);
    tmp_b = std::max(tmp_b, t2);
    cub::DeviceScan::InclusiveScan(nullptr, t2, (int32_t*)nullptr, (int32_t*)nullptr, MaxOp(), n);
    tmp_b = std::max(tmp_b, t2);
    cub::DeviceRadixSort::SortPairs(nullptr, t2, (uint64_t*)nullptr, (uint64_t*)nullptr, (int32_t*)nullptr,
                                    (int32_t*)nullptr, n);
    tmp_b = std::max(tmp_b, t2);
    tmp_b += 256;
    const size_t al8 = 256;
    auto A = [&](size_t b) { return (b + al8 - 1) / al8 * al8; };
    const size_t bytes = A(tmp_b) + 2 * A(m0 * 8) + 2 * A(m0 * 4) + A(m0 * 8) + A(m0 * 8) + A(16) +
                         A((size_t)n * 8) /*cw*/ + A((size_t)(n + 1) * 4) * 2 /*flag,pos*/ + A((size_t)n * 4) /*L*/ +
                         A((size_t)n * 8) * 2 /*gain,h*/ + A((size_t)n * 4) * 2 /*idx,idx2*/ + A((size_t)n * 8) * 2 +
                         A((size_t)n * 8) * 2 /*cval,incl*/ + A((size_t)n * 4) * 2 /*headpos,segstart*/ + A(64);
    char* base = (char*)alloc(bytes, st);
    if (!base) return cudaErrorMemoryAllocation;
    size_t off = 0;
    auto take = [&](size_t b) {
        char* p = base + off;
        off += A(b);
        return (void*)p;
    };
    void* tmp = take(tmp_b);
    uint64_t* keys = (uint64_t*)take(m0 * 8);
    uint64_t* keys2 = (uint64_t*)take(m0 * 8);
    int32_t* vals = (int32_t*)take(m0 * 4);
    int32_t* vals2 = (int32_t*)take(m0 * 4);
    uint64_t* ukeys = (uint64_t*)take(m0 * 8);
    int32_t* uscore = (int32_t*)take(m0 * 4);
    int64_t* nruns = (int64_t*)take(16);
    long long* cw = (long long*)take((size_t)n * 8);
    int32_t* flag = (int32_t*)take((size_t)(n + 1) * 4);
    int32_t* pos = (int32_t*)take((size_t)(n + 1) * 4);
    int32_t* reqL = (int32_t*)take((size_t)n * 4);
    long long* reqG = (long long*)take((size_t)n * 8);
    uint64_t* reqH = (uint64_t*)take((size_t)n * 8);
    int32_t* idx = (int32_t*)take((size_t)n * 4);
    int32_t* idx2 = (int32_t*)take((size_t)n * 4);
    uint64_t* skey = (uint64_t*)take((size_t)n * 8);
    uint64_t* skey2 = (uint64_t*)take((size_t)n * 8);
    long long* cval = (long long*)take((size_t)n * 8);
    long long* incl = (long long*)take((size_t)n * 8);
    int32_t* headpos = (int32_t*)take((size_t)n * 4);
    int32_t* segstart = (int32_t*)take((size_t)n * 4);
    int32_t* moved = (int32_t*)take(64);
    (void)skey2;
    cudaError_t e = cudaSuccess;
#define LP_CK(x)                 \
    do {                         \
        e = (x);                 \
        if (e != cudaSuccess) {  \
            dealloc(base, st);   \
            return e;            \
        }                        \
    } while (0)
    {
        LaunchScope ls("lp_init", st);
        k_lp_init<<<nblk(n), 256, 0, st>>>(n, c, lab, cw);
    }
    int32_t used = 0;
    int key_bits = 1;
    while (key_bits < 31 && ((n - 1) >> key_bits) != 0) ++key_bits;
    for (int32_t r = 0; r < rounds; ++r) {
        ++used;
        if (nnz > 0) {
            {
                LaunchScope ls("lp_keys", st);
                k_lp_keys<<<nblk((int64_t)n * 32), 256, 0, st>>>(n, rp, col, omega, lab, keys, vals);
            }
            {
                LaunchScope ls("cub_sort_lp", st);
                LP_CK(cub::DeviceRadixSort::SortPairs(tmp, tmp_b, keys, keys2, vals, vals2, nnz, 0, 32 + key_bits,
                                                      st));
            }
            {
                LaunchScope ls("cub_reduce_lp", st);
                // scores fit int32: a node's scores sum to at most the total edge weight
                LP_CK(cub::DeviceReduce::ReduceByKey(tmp, tmp_b, keys2, ukeys, vals2, uscore, nruns, cub::Sum(), nnz,
                                                     st));
            }
        }
        int64_t m = 0;
        if (nnz > 0) {
            LP_CK(cudaMemcpyAsync(&m, nruns, 8, cudaMemcpyDeviceToHost, st));
            LP_CK(cudaStreamSynchronize(st));
        }
        {
            LaunchScope ls("lp_choose", st);
            k_lp_choose<<<nblk((int64_t)n * 32), 256, 0, st>>>(n, ukeys, uscore, m, lab, cw, c, U, seed, level, r,
                                                                  flag, reqL, reqG, reqH);
        }
        LP_CK(cudaMemsetAsync(flag + n, 0, 4, st));
        {
            LaunchScope ls("cub_scan_lp", st);
            LP_CK(cub::DeviceScan::ExclusiveSum(tmp, tmp_b, flag, pos, n + 1, st));
        }
        int32_t R = 0;
        LP_CK(cudaMemcpyAsync(&R, pos + n, 4, cudaMemcpyDeviceToHost, st));
        LP_CK(cudaStreamSynchronize(st));
        if (R == 0) break;
        {
            LaunchScope ls("lp_compact", st);
            k_lp_compact<<<nblk(n), 256, 0, st>>>(n, flag, pos, reqL, reqG, reqH, idx, skey, skey2);
        }
        // stable passes: hash desc, gain desc, label asc (idx starts in ascending v)
        {
            LaunchScope ls("cub_sort_req", st);
            LP_CK(cub::DeviceRadixSort::SortPairs(tmp, tmp_b, skey, skey2, idx, idx2, R, 0, 64, st));
        }
        {
            LaunchScope ls("lp_keys_gain", st);
            k_lp_gather_keys<<<nblk(R), 256, 0, st>>>(R, idx2, reqH, reqG, reqL, 0, skey);
        }
        {
            LaunchScope ls("cub_sort_req", st);
            LP_CK(cub::DeviceRadixSort::SortPairs(tmp, tmp_b, skey, skey2, idx2, idx, R, 0, 64, st));
        }
        {
            LaunchScope ls("lp_keys_label", st);
            k_lp_gather_keys<<<nblk(R), 256, 0, st>>>(R, idx, reqH, reqG, reqL, 1, skey);
        }
        {
            LaunchScope ls("cub_sort_req", st);
            LP_CK(cub::DeviceRadixSort::SortPairs(tmp, tmp_b, skey, skey2, idx, idx2, R, 0, key_bits, st));
        }
        {
            LaunchScope ls("lp_segvals", st);
            k_lp_segvals<<<nblk(R), 256, 0, st>>>(R, idx2, reqL, c, cval, headpos);
        }
        {
            LaunchScope ls("cub_scan_lp", st);
            LP_CK(cub::DeviceScan::InclusiveSum(tmp, tmp_b, cval, incl, R, st));
            LP_CK(cub::DeviceScan::InclusiveScan(tmp, tmp_b, headpos, segstart, MaxOp(), R, st));
        }
        LP_CK(cudaMemsetAsync(moved, 0, 4, st));
        {
            LaunchScope ls("lp_apply", st);
            k_lp_apply<<<nblk(R), 256, 0, st>>>(R, idx2, reqL, incl, segstart, cw, U, lab, moved);
        }
        LP_CK(cudaMemsetAsync(cw, 0, (size_t)n * 8, st));
        {
            LaunchScope ls("lp_weights", st);
            k_lp_weights<<<nblk(n), 256, 0, st>>>(n, lab, c, cw);
        }
        int32_t hm = 0;
        LP_CK(cudaMemcpyAsync(&hm, moved, 4, cudaMemcpyDeviceToHost, st));
        LP_CK(cudaStreamSynchronize(st));
        if (hm == 0) break;
    }
#undef LP_CK
    if (rounds_used) *rounds_used = used;
    dealloc(base, st);
    return cudaGetLastError();
}

}  // namespace mm
