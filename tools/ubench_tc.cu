// Builder tool: kernel (c)'s tensor-core far-tile path (k_repulse_tc.cuh: tcgen05.mma kind::tf32,
// weights in TMEM) on synthetic Morton-ordered points, against plain FP32 and FP64 pair loops over
// the same eligible (128-target block, 256-source tile) pairs.  Prints time, pairs/s, cycles per 64
// pairs per SMSP and the error of both FP32 paths relative to sum_j |term|.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ubench_tc_accum.cuh"

using namespace mm;

template <typename R>
__global__ void __launch_bounds__(128) k_direct(int n_tgt, const float4* __restrict__ tgt, int n_src,
                                                const float4* __restrict__ src, const uint32_t* __restrict__ elig,
                                                int words, R cexp, R* __restrict__ out, R* __restrict__ out_abs,
                                                unsigned long long* __restrict__ npairs) {
    __shared__ float4 sm[256];
    const int tid = threadIdx.x, blk = blockIdx.x;
    const int ntiles = (n_src + 255) / 256;
    int64_t i = (int64_t)blk * 128 + tid;
    const bool valid = i < n_tgt;
    if (!valid) i = n_tgt - 1;
    const float4 me = __ldg(tgt + i);
    R acc[3] = {0, 0, 0}, aabs = 0;
    unsigned long long cnt = 0;
    for (int tile = 0; tile < ntiles; ++tile) {
        if (!((elig[(int64_t)blk * words + (tile >> 5)] >> (tile & 31)) & 1)) continue;
        __syncthreads();
        for (int s = tid; s < 256; s += 128) {
            const int64_t js = (int64_t)tile * 256 + s;
            sm[s] = js < n_src ? __ldg(src + js) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        __syncthreads();
        const int cntj = min(256, n_src - tile * 256);
        cnt += cntj;
        R t[3] = {0, 0, 0};
        for (int jj = 0; jj < cntj; ++jj) {
            const float4 s = sm[jj];
            const R dx = (R)me.x - (R)s.x, dy = (R)me.y - (R)s.y, dz = (R)me.z - (R)s.z;
            const R r2 = dx * dx + dy * dy + dz * dz + (R)kEps2;
            R inv;
            if constexpr (sizeof(R) == 4)
                inv = ex2_approx((float)cexp * lg2_approx((float)r2));
            else
                inv = exp2(cexp * log2(r2));
            inv *= (R)s.w;
            t[0] += dx * inv;
            t[1] += dy * inv;
            t[2] += dz * inv;
            if (out_abs) aabs += sqrt(r2) * inv;
        }
        for (int d = 0; d < 3; ++d) acc[d] += t[d];
    }
    if (valid) {
        out[4 * i + 0] = acc[0];
        out[4 * i + 1] = acc[1];
        out[4 * i + 2] = acc[2];
        if (out_abs) out_abs[i] = aabs;
    }
    if (npairs && tid == 0) atomicAdd(npairs, cnt * (unsigned long long)min(128, n_tgt - blk * 128));
}

static uint32_t part1by2(uint32_t x) {
    x &= 0x3ff;
    x = (x | (x << 16)) & 0x30000ff;
    x = (x | (x << 8)) & 0x300f00f;
    x = (x | (x << 4)) & 0x30c30c3;
    x = (x | (x << 2)) & 0x9249249;
    return x;
}
static uint32_t morton(float x, float y, float z) {
    return part1by2((uint32_t)(x * 1023.f)) | (part1by2((uint32_t)(y * 1023.f)) << 1) |
           (part1by2((uint32_t)(z * 1023.f)) << 2);
}
static void make_points(int n, uint64_t seed, float scale, float offs, bool masses, std::vector<float4>& p) {
    p.resize(n);
    uint64_t s = seed;
    auto rnd = [&]() {
        s = s * 6364136223846793005ULL + 1442695040888963407ULL;
        return (float)((s >> 40) & 0xFFFFFF) / 16777216.f;
    };
    std::vector<std::pair<uint32_t, int>> key(n);
    std::vector<float4> q(n);
    for (int i = 0; i < n; ++i) {
        float x = rnd(), y = rnd(), z = rnd();
        key[i] = {morton(x, y, z), i};
        q[i] = make_float4(offs + scale * x, offs + scale * y, offs + scale * z, masses ? (float)(1 + (int)(rnd() * 4.f)) : 1.f);
    }
    std::sort(key.begin(), key.end());
    for (int i = 0; i < n; ++i) p[i] = q[key[i].second];
}


#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); return 1; } } while (0)

int main(int argc, char** argv) {
    const int n_tgt = argc > 1 ? atoi(argv[1]) : 148 * 8 * 128;
    const int n_src = argc > 2 ? atoi(argv[2]) : 262144;
    const float q = 0.8f, cexp = -(q + 2.f) / 2.f;
    const float scale = argc > 3 ? atof(argv[3]) : 100.f, offs = argc > 4 ? atof(argv[4]) : -50.f;
    const float eta = argc > 5 ? atof(argv[5]) : 0.5f;
    const int check = argc > 6 ? atoi(argv[6]) : 1;
    std::vector<float4> ht, hs;
    make_points(n_tgt, 1, scale, offs, false, ht);
    make_points(n_src, 2, scale, offs, true, hs);
    const int ntiles = (n_src + 255) / 256, nblk = (n_tgt + 127) / 128, words = (ntiles + 31) / 32;
    std::vector<float4> hb(2 * ntiles);
    for (int t = 0; t < ntiles; ++t) {
        float lo[3] = {1e30f, 1e30f, 1e30f}, hi[3] = {-1e30f, -1e30f, -1e30f};
        for (int j = t * 256; j < std::min(n_src, (t + 1) * 256); ++j) {
            const float v[3] = {hs[j].x, hs[j].y, hs[j].z};
            for (int d = 0; d < 3; ++d) {
                lo[d] = std::min(lo[d], v[d]);
                hi[d] = std::max(hi[d], v[d]);
            }
        }
        hb[2 * t] = make_float4(lo[0], lo[1], lo[2], 0.f);
        hb[2 * t + 1] = make_float4(hi[0], hi[1], hi[2], 0.f);
    }
    float4 *dt, *ds, *db, *dout, *dbb;
    uint32_t* delig;
    float* dref32;
    double *dref64, *dabs;
    unsigned long long* dnp;
    CK(cudaMalloc(&dt, (size_t)n_tgt * 16));
    CK(cudaMalloc(&ds, (size_t)n_src * 16));
    CK(cudaMalloc(&db, (size_t)2 * ntiles * 16));
    CK(cudaMalloc(&dbb, (size_t)2 * nblk * 16));
    CK(cudaMalloc(&delig, (size_t)nblk * words * 4));
    CK(cudaMalloc(&dout, (size_t)n_tgt * 16));
    CK(cudaMalloc(&dref32, (size_t)n_tgt * 16));
    CK(cudaMalloc(&dref64, (size_t)n_tgt * 32));
    CK(cudaMalloc(&dabs, (size_t)n_tgt * 8));
    CK(cudaMalloc(&dnp, 8));
    CK(cudaMemcpy(dt, ht.data(), (size_t)n_tgt * 16, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ds, hs.data(), (size_t)n_src * 16, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(db, hb.data(), (size_t)2 * ntiles * 16, cudaMemcpyHostToDevice));
    CK(cudaMemset(dout, 0, (size_t)n_tgt * 16));
    CK(cudaMemset(dref32, 0, (size_t)n_tgt * 16));
    CK(cudaMemset(dref64, 0, (size_t)n_tgt * 32));
    CK(cudaMemset(dabs, 0, (size_t)n_tgt * 8));
    CK(cudaMemset(dnp, 0, 8));
    tc::k_tc_boxes<<<(nblk * 32 + 255) / 256, 256>>>(n_tgt, reinterpret_cast<const float*>(dt), nullptr, nullptr, dbb);
    tc::k_tc_elig<<<(int)(((int64_t)nblk * words + 255) / 256), 256>>>(nblk, dbb, ntiles, db, eta * eta, words, delig);
    CK(cudaDeviceSynchronize());
    tc::Args a{};
    a.n_tgt = n_tgt; a.x = reinterpret_cast<const float*>(dt); a.tperm = nullptr; a.frame = nullptr;
    a.n_src = n_src; a.rep_hi = ds; a.rep_lo = nullptr; a.blk_box = dbb; a.elig = delig; a.words = words;
    a.cexp = cexp; a.out = dout;
    int dev = 0, clk = 0, sms = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    CK(cudaFuncSetAttribute(tc::k_repulse_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::kSmemBytes));
    const int grid = std::min(nblk, sms);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0);
        tc::k_repulse_tc<<<grid, tc::kThreads, tc::kSmemBytes>>>(a);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms);
    }
    k_direct<float><<<nblk, 128>>>(n_tgt, dt, n_src, ds, delig, words, cexp, dref32, nullptr, dnp);
    CK(cudaDeviceSynchronize());
    unsigned long long np = 0;
    CK(cudaMemcpy(&np, dnp, 8, cudaMemcpyDeviceToHost));
    printf("eta=%.2f mufu_mask=%04x n_tgt=%d n_src=%d eligible pairs=%.4g (%.1f%% of all)\n", eta, (unsigned)MM_TC_MUFU_MASK,
           n_tgt, n_src, (double)np, 100.0 * np / ((double)n_tgt * n_src));
    const double cyc64 = best * 1e-3 * clk * 1e3 * sms * 4.0 / ((double)np / 64.0);
    printf("tc     : %.3f ms  %.4g pairs/s  %.1f cycles per 64 pairs per SMSP\n", best, np / (best * 1e-3), cyc64);
    if (!check) return 0;
    k_direct<double><<<nblk, 128>>>(n_tgt, dt, n_src, ds, delig, words, (double)cexp, dref64, dabs, nullptr);
    CK(cudaDeviceSynchronize());
    std::vector<float4> ho(n_tgt);
    std::vector<float> h32(4 * (size_t)n_tgt);
    std::vector<double> h64(4 * (size_t)n_tgt), habs(n_tgt);
    CK(cudaMemcpy(ho.data(), dout, (size_t)n_tgt * 16, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h32.data(), dref32, (size_t)n_tgt * 16, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h64.data(), dref64, (size_t)n_tgt * 32, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(habs.data(), dabs, (size_t)n_tgt * 8, cudaMemcpyDeviceToHost));
    double emax_m = 0, emax_d = 0, erms_m = 0, erms_d = 0, bias_m = 0, bias_d = 0;
    int worst = -1;
    for (int i = 0; i < n_tgt; ++i) {
        const float om[3] = {ho[i].x, ho[i].y, ho[i].z};
        double nrm = 0;
        for (int d = 0; d < 3; ++d) nrm += h64[4 * (size_t)i + d] * h64[4 * (size_t)i + d];
        for (int d = 0; d < 3; ++d) {
            const double ref = h64[4 * (size_t)i + d], ab = habs[i] > 0 ? habs[i] : 1;
            const double em = (om[d] - ref) / ab, ed = (h32[4 * (size_t)i + d] - ref) / ab;
            if (!(std::fabs(em) <= emax_m)) { emax_m = std::fabs(em); worst = i; }
            emax_d = std::max(emax_d, std::fabs(ed));
            erms_m += em * em;
            erms_d += ed * ed;
            if (nrm > 0) {
                bias_m += (om[d] - ref) * ref / nrm;
                bias_d += (h32[4 * (size_t)i + d] - ref) * ref / nrm;
            }
        }
    }
    erms_m = std::sqrt(erms_m / (3.0 * n_tgt));
    erms_d = std::sqrt(erms_d / (3.0 * n_tgt));
    printf("error / sum|term| : tc max %.3g rms %.3g | fp32 direct max %.3g rms %.3g\n", emax_m, erms_m, emax_d, erms_d);
    printf("mean signed error along T (relative to |T|): tc %.3g direct %.3g\n", bias_m / n_tgt, bias_d / n_tgt);
    if (worst >= 0)
        printf("worst target %d: tc (%g %g %g) ref (%g %g %g) sum|term| %g\n", worst, ho[worst].x, ho[worst].y, ho[worst].z,
               h64[4 * (size_t)worst], h64[4 * (size_t)worst + 1], h64[4 * (size_t)worst + 2], habs[worst]);
    return 0;
}
