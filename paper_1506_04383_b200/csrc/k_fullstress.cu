// k_fullstress.cu — the full-stress quality metric F(x) and its optimal scale
// (PAPER.md P:323-328):
//   F(x) = sum_{u<v} w_uv (|x_u - x_v| - d_uv)^2,  d_uv = BFS distance, w = d^-2
//   F(s x) = s^2 B - 2 s A + C,  A = sum w d l,  B = sum w l^2,  C = sum w d^2,
//   s* = A / B  ("We find a scalar s such that ... is minimized").
// One CTA runs one BFS at a time: the visited set of the current source is a
// bitset in shared memory (n/8 bytes), the level queues live in a per-CTA
// global scratch (L2-resident); every vertex v > s reached at level d adds its
// pair terms to per-thread FP64 accumulators (unordered pairs, each once).
// The accumulation order follows the BFS claim order (atomics), so the FP64
// sums may differ in the last bits between runs; the metric is not part of a
// layout trajectory (R5).
#include "k_fullstress.cuh"

namespace mm {
namespace {

constexpr int kFsBlock = 256;

template <int DIM>
__global__ void __launch_bounds__(kFsBlock) k_full_stress(int32_t n, const int64_t* __restrict__ rp,
                                                          const int32_t* __restrict__ col, const float* __restrict__ x,
                                                          int32_t* __restrict__ qbuf, double* __restrict__ partial) {
    extern __shared__ uint32_t vis[];  // ceil(n / 32) words
    __shared__ int32_t s_qlen, s_next;
    const int tid = threadIdx.x;
    const int32_t words = (n + 31) >> 5;
    int32_t* qa = qbuf + (int64_t)blockIdx.x * 2 * n;
    int32_t* qb = qa + n;
    double A = 0.0, B = 0.0, C = 0.0, F = 0.0, P = 0.0;
    for (int32_t s = blockIdx.x; s < n; s += gridDim.x) {
        for (int32_t t = tid; t < words; t += kFsBlock) vis[t] = 0u;
        __syncthreads();
        if (tid == 0) {
            vis[s >> 5] = 1u << (s & 31);
            qa[0] = s;
            s_qlen = 1;
            s_next = 0;
        }
        __syncthreads();
        const float4 xs = load_x<DIM>(x, s);
        int32_t* cur = qa;
        int32_t* nxt = qb;
        for (int32_t d = 1;; ++d) {
            const int32_t qlen = s_qlen;
            if (qlen == 0) break;
            const double dd = (double)d, w = 1.0 / (dd * dd);
            for (int32_t t = tid; t < qlen; t += kFsBlock) {
                const int32_t a = cur[t];
                for (int64_t e = rp[a]; e < rp[a + 1]; ++e) {
                    const int32_t b = col[e];
                    const uint32_t bit = 1u << (b & 31);
                    if (vis[b >> 5] & bit) continue;
                    const uint32_t old = atomicOr(&vis[b >> 5], bit);
                    if (old & bit) continue;  // another thread claimed b
                    nxt[atomicAdd(&s_next, 1)] = b;
                    if (b > s) {
                        const float4 xb = load_x<DIM>(x, b);
                        const double ex = (double)xs.x - xb.x, ey = (double)xs.y - xb.y, ez = (double)xs.z - xb.z;
                        const double l = sqrt(ex * ex + ey * ey + ez * ez);
                        A += w * dd * l;
                        B += w * l * l;
                        C += w * dd * dd;
                        F += w * (l - dd) * (l - dd);
                        P += 1.0;
                    }
                }
            }
            __syncthreads();
            if (tid == 0) {
                s_qlen = s_next;
                s_next = 0;
            }
            __syncthreads();
            int32_t* t = cur;
            cur = nxt;
            nxt = t;
        }
        __syncthreads();
    }
    // block reduction -> partial[blockIdx.x][5]
    __shared__ double red[5][kFsBlock / 32];
    double v[5] = {A, B, C, F, P};
#pragma unroll
    for (int k = 0; k < 5; ++k) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
        if ((tid & 31) == 0) red[k][tid >> 5] = v[k];
    }
    __syncthreads();
    if (tid < 5) {
        double sum = 0.0;
        for (int w = 0; w < kFsBlock / 32; ++w) sum += red[tid][w];
        partial[(int64_t)blockIdx.x * 5 + tid] = sum;
    }
}

}  // namespace

size_t full_stress_smem(int32_t n) { return (size_t)((n + 31) / 32) * 4; }

int full_stress_grid(int32_t n) {
    int dev = 0, sms = 148, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = full_stress_smem(n);
    cudaFuncSetAttribute(k_full_stress<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_full_stress<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_full_stress<2>, kFsBlock, smem);
    if (occ < 1) occ = 1;
    return (int)std::min<int64_t>((int64_t)sms * occ, n);
}

cudaError_t launch_full_stress(int dim, int32_t n, const int64_t* rp, const int32_t* col, const float* x, int grid,
                               int32_t* qbuf, double* partial, cudaStream_t st) {
    const size_t smem = full_stress_smem(n);
    LaunchScope ls("full_stress", st);
    if (dim == 2) k_full_stress<2><<<grid, kFsBlock, smem, st>>>(n, rp, col, x, qbuf, partial);
    else k_full_stress<3><<<grid, kFsBlock, smem, st>>>(n, rp, col, x, qbuf, partial);
    return cudaGetLastError();
}

}  // namespace mm
