// k_sort.cu — stable LSD radix sort of (key, int32 value) pairs (k_sort.cuh).
//
// One pass per 8-bit digit, three launches per pass:
//  1. k_rs_hist:    per 2,048-key tile, a shared-memory digit histogram,
//                   written digit-major (ghist[d][tile]);
//  2. k_rs_offsets: one block per digit scans its tiles' counts (start of
//                   every tile's run within the digit) and totals the digit;
//  3. k_rs_scatter: each tile re-reads its keys in 8 rounds of 256 (index
//                   order) and ranks them stably: __match_any_sync groups the
//                   lanes of a warp with equal digits (rank = peers below the
//                   lane), per-warp digit counts in shared memory order the
//                   warps, a running per-digit offset orders the rounds; the
//                   tile is staged in shared memory sorted by digit and each
//                   digit's run is written to consecutive output positions.
// Equal keys therefore keep their input order, as the sort keys of kernel
// (c)'s orders and of the member / child lists require (ties by vertex id).
#include "k_sort.cuh"

namespace mm {

namespace {

constexpr int kRsThreads = 256, kRsItems = 8, kRsTile = kRsThreads * kRsItems, kRsRadix = 256;
inline size_t al256(size_t b) { return (b + 255) & ~(size_t)255; }
inline int64_t rs_tiles(int64_t n) { return std::max<int64_t>(1, (n + kRsTile - 1) / kRsTile); }

template <typename K>
__global__ void __launch_bounds__(kRsThreads) k_rs_hist(const K* __restrict__ keys, int64_t n, int bit, int64_t nb,
                                                        int32_t* __restrict__ ghist) {
    __shared__ int32_t h[kRsRadix];
    h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kRsTile;
#pragma unroll
    for (int r = 0; r < kRsItems; ++r) {
        const int64_t i = base + r * kRsThreads + threadIdx.x;
        if (i < n) atomicAdd(&h[(int)((keys[i] >> bit) & 255u)], 1);
    }
    __syncthreads();
    ghist[(int64_t)threadIdx.x * nb + blockIdx.x] = h[threadIdx.x];
}

// block-wide exclusive scan of one int per thread (256 threads); total out
__device__ __forceinline__ int32_t rs_block_scan(int32_t v, int32_t* wtot, int32_t& total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) wtot[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        int32_t w = lane < kRsThreads / 32 ? wtot[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t t = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += t;
        }
        if (lane < kRsThreads / 32) wtot[lane] = w;
    }
    __syncthreads();
    const int32_t r = (wid > 0 ? wtot[wid - 1] : 0) + inc - v;
    total = wtot[kRsThreads / 32 - 1];
    __syncthreads();
    return r;
}

// one block per digit d: exclusive scan of ghist[d][0..nb) into gofs[d][.]
// (positions relative to the digit's start) and the digit total dtot[d]
__global__ void __launch_bounds__(kRsThreads) k_rs_offsets(const int32_t* __restrict__ ghist, int64_t nb,
                                                           int32_t* __restrict__ gofs, int32_t* __restrict__ dtot) {
    __shared__ int32_t wt[kRsThreads / 32];
    const int64_t base = (int64_t)blockIdx.x * nb;
    int32_t carry = 0;
    for (int64_t b0 = 0; b0 < nb; b0 += kRsThreads) {
        const int64_t b = b0 + threadIdx.x;
        const int32_t v = b < nb ? ghist[base + b] : 0;
        int32_t tot;
        const int32_t ex = rs_block_scan(v, wt, tot);
        if (b < nb) gofs[base + b] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) dtot[blockIdx.x] = carry;
}

// Ranks the tile's keys stably (see the file comment), stages them in shared
// memory sorted by digit, then writes each digit's run to consecutive global
// positions (coalesced).
template <typename K>
__global__ void __launch_bounds__(kRsThreads) k_rs_scatter(const K* __restrict__ kin, const int32_t* __restrict__ vin,
                                                           int64_t n, int bit, int64_t nb,
                                                           const int32_t* __restrict__ ghist,
                                                           const int32_t* __restrict__ gofs,
                                                           const int32_t* __restrict__ dtot, K* __restrict__ kout,
                                                           int32_t* __restrict__ vout) {
    __shared__ int32_t run[kRsRadix], tstart[kRsRadix], gbase[kRsRadix];
    __shared__ int32_t wc[kRsThreads / 32][kRsRadix];
    __shared__ int32_t wt[kRsThreads / 32];
    __shared__ K skey[kRsTile];
    __shared__ int32_t sval[kRsTile];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t below = (1u << lane) - 1u;
    {
        int32_t tot;
        const int32_t d = threadIdx.x;
        const int32_t dbase = rs_block_scan(dtot[d], wt, tot);      // digit starts in the output
        const int32_t th = ghist[(int64_t)d * nb + blockIdx.x];
        tstart[d] = rs_block_scan(th, wt, tot);                      // digit starts in the tile
        gbase[d] = dbase + gofs[(int64_t)d * nb + blockIdx.x];       // this tile's run of digit d
        run[d] = tstart[d];
    }
    const int64_t base = (int64_t)blockIdx.x * kRsTile;
    const int cnt = (int)min((int64_t)kRsTile, n - base);
    for (int r = 0; r < kRsItems; ++r) {
#pragma unroll
        for (int t = 0; t < kRsRadix / 32; ++t) wc[wid][t * 32 + lane] = 0;
        const int li = r * kRsThreads + threadIdx.x;
        const bool valid = li < cnt;
        K key = 0;
        int32_t val = 0;
        int d = kRsRadix + lane;  // past the end: a digit no other lane has
        if (valid) {
            key = kin[base + li];
            val = vin[base + li];
            d = (int)((key >> bit) & 255u);
        }
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const int rank = __popc(peers & below);
        __syncwarp();
        if (valid && rank == 0) wc[wid][d] = __popc(peers);
        __syncthreads();
        if (valid) {
            int off = run[d] + rank;
            for (int w = 0; w < wid; ++w) off += wc[w][d];
            skey[off] = key;
            sval[off] = val;
        }
        __syncthreads();
        int tot = 0;
#pragma unroll
        for (int w = 0; w < kRsThreads / 32; ++w) tot += wc[w][threadIdx.x];
        run[threadIdx.x] += tot;
        __syncthreads();
    }
    for (int j = threadIdx.x; j < cnt; j += kRsThreads) {
        const K key = skey[j];
        const int d = (int)((key >> bit) & 255u);
        const int32_t pos = gbase[d] + (j - tstart[d]);
        kout[pos] = key;
        vout[pos] = sval[j];
    }
}

}  // namespace

template <typename K>
size_t radix_sort_tmp_bytes(int64_t n) {
    const int64_t nb = rs_tiles(n);
    return al256((size_t)n * sizeof(K)) + al256((size_t)n * 4) + 2 * al256((size_t)(kRsRadix * nb + 1) * 4) +
           al256(kRsRadix * 4) + 256;
}

template <typename K>
cudaError_t radix_sort_pairs(const K* kin, K* kout, const int32_t* vin, int32_t* vout, int64_t n, int begin_bit,
                             int end_bit, void* tmp, size_t tmp_bytes, cudaStream_t st, const char* name) {
    if (n <= 0) return cudaSuccess;
    if (tmp_bytes < radix_sort_tmp_bytes<K>(n)) return cudaErrorInvalidValue;
    const int64_t nb = rs_tiles(n);
    char* p = static_cast<char*>(tmp);
    K* kalt = reinterpret_cast<K*>(p);
    p += al256((size_t)n * sizeof(K));
    int32_t* valt = reinterpret_cast<int32_t*>(p);
    p += al256((size_t)n * 4);
    int32_t* ghist = reinterpret_cast<int32_t*>(p);
    p += al256((size_t)(kRsRadix * nb + 1) * 4);
    int32_t* gofs = reinterpret_cast<int32_t*>(p);
    p += al256((size_t)(kRsRadix * nb + 1) * 4);
    int32_t* dtot = reinterpret_cast<int32_t*>(p);
    const int passes = std::max(0, (end_bit - begin_bit + 7) / 8);
    if (passes == 0) {
        cudaError_t e = cudaMemcpyAsync(kout, kin, (size_t)n * sizeof(K), cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) return e;
        return cudaMemcpyAsync(vout, vin, (size_t)n * 4, cudaMemcpyDeviceToDevice, st);
    }
    const K* ks = kin;
    const int32_t* vs = vin;
    for (int ps = 0; ps < passes; ++ps) {
        const int bit = begin_bit + 8 * ps;
        const bool to_out = ((passes - 1 - ps) % 2) == 0;  // the last pass lands in (kout, vout)
        K* kd = to_out ? kout : kalt;
        int32_t* vd = to_out ? vout : valt;
        LaunchScope ls(name, st);
        k_rs_hist<K><<<(unsigned)nb, kRsThreads, 0, st>>>(ks, n, bit, nb, ghist);
        k_rs_offsets<<<kRsRadix, kRsThreads, 0, st>>>(ghist, nb, gofs, dtot);
        k_rs_scatter<K><<<(unsigned)nb, kRsThreads, 0, st>>>(ks, vs, n, bit, nb, ghist, gofs, dtot, kd, vd);
        ks = kd;
        vs = vd;
    }
    return cudaGetLastError();
}

template size_t radix_sort_tmp_bytes<uint32_t>(int64_t);
template size_t radix_sort_tmp_bytes<uint64_t>(int64_t);
template cudaError_t radix_sort_pairs<uint32_t>(const uint32_t*, uint32_t*, const int32_t*, int32_t*, int64_t, int, int,
                                                void*, size_t, cudaStream_t, const char*);
template cudaError_t radix_sort_pairs<uint64_t>(const uint64_t*, uint64_t*, const int32_t*, int32_t*, int64_t, int, int,
                                                void*, size_t, cudaStream_t, const char*);

}  // namespace mm
