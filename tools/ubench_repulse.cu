// Variant sweep of the exact 2-D q=0 repulsion kernel (b): targets per thread
// T, batched-reciprocal group mask, min blocks per SM.  Standalone timing tool
// (includes the library's kernel source; LaunchScope is stubbed).
#include "../paper_1506_04383_b200/csrc/k_repulse.cu"
#include <cstdio>
#include <vector>
#include <random>
namespace mm {
LaunchScope::LaunchScope(const char* n, cudaStream_t s) : name(n), stream(s), slot(-1) {}
LaunchScope::~LaunchScope() {}
}
using namespace mm;

template <int T, int BM, int MINB, int UNR = 4>
void run(int n, const float* x, float* part, int sms) {
    auto kern = k_repulse<2, false, false, T, BM, MINB, UNR>;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, 0);
    Sched s;
    const int64_t TPB = 256 * T;
    s.TB = (int32_t)((n + TPB - 1) / TPB);
    s.Ub = (n + 255) / 256;
    s.U = (int64_t)s.TB * s.Ub;
    s.G = (int32_t)std::min<int64_t>((int64_t)sms * occ, s.U);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, kern);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 2; ++i) kern<<<s.G, 256>>>(n, x, n, nullptr, nullptr, nullptr, -1.f, s, part);
    const int reps = 10;
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) kern<<<s.G, 256>>>(n, x, n, nullptr, nullptr, nullptr, -1.f, s, part);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    ms /= reps;
    const double pairs = (double)n * n;
    printf("T=%d BMASK=%d MINB=%d UNR=%d regs=%d occ=%d G=%d  %.4f ms  %.4e pairs/s  (%.1f%% of 16 MUFU/clk/SM @1965)\n", T, BM,
           MINB, UNR, fa.numRegs, occ, s.G, ms, pairs / (ms * 1e-3), 100.0 * pairs / (ms * 1e-3) / (148 * 16 * 1.965e9));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("  error %s\n", cudaGetErrorString(e));
}

template <int DIM, bool QPOW, int T, int BM, int MINB>
void run_coarse(int n, int k, const float* x, const float4* hi, const float4* lo, const int32_t* anc, float* part,
                int sms, float cexp) {
    auto kern = k_repulse<DIM, QPOW, true, T, BM, MINB>;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, 0);
    Sched s;
    const int64_t TPB = 256 * T;
    s.TB = (int32_t)((n + TPB - 1) / TPB);
    s.Ub = (k + 255) / 256;
    s.U = (int64_t)s.TB * s.Ub;
    s.G = (int32_t)std::min<int64_t>((int64_t)sms * occ, s.U);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, kern);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 2; ++i) kern<<<s.G, 256>>>(n, x, k, hi, lo, anc, cexp, s, part);
    const int reps = 5;
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) kern<<<s.G, 256>>>(n, x, k, hi, lo, anc, cexp, s, part);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    ms /= reps;
    const double pairs = (double)n * k;
    printf("COARSE dim=%d q=%d T=%d BMASK=%d MINB=%d regs=%d occ=%d G=%d  %.4f ms  %.4e pairs/s\n", DIM, (int)QPOW, T, BM,
           MINB, fa.numRegs, occ, s.G, ms, pairs / (ms * 1e-3));
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 65428;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    std::vector<float> hx(2 * (size_t)n);
    std::mt19937 rng(1);
    std::uniform_real_distribution<float> U(0.f, 1.f);
    for (auto& v : hx) v = U(rng);
    float *x, *part;
    cudaMalloc(&x, hx.size() * 4);
    cudaMalloc(&part, (size_t)n * 2 * 4 * 64);
    cudaMemcpy(x, hx.data(), hx.size() * 4, cudaMemcpyHostToDevice);
    run<4, 1, 1, 1>(n, x, part, sms);
    run<4, 1, 1, 2>(n, x, part, sms);
    run<4, 1, 1, 4>(n, x, part, sms);
    run<4, 1, 1, 8>(n, x, part, sms);
    run<4, 1, 3, 2>(n, x, part, sms);
    run<4, 1, 3, 1>(n, x, part, sms);
    run<4, 1, 4, 1>(n, x, part, sms);
    run<2, 1, 1, 8>(n, x, part, sms);
    run<2, 1, 4, 4>(n, x, part, sms);
    run<6, 1, 1, 2>(n, x, part, sms);
    run<6, 5, 1, 2>(n, x, part, sms);
    run<8, 1, 1, 2>(n, x, part, sms);
    run<8, 5, 2, 1>(n, x, part, sms);
    // coarse: n = 262,144 targets in [0,512)^2, k = 77,649 reps (cfg3 finest level shape)
    {
        const int nt = 262144, k = 77649;
        std::vector<float> tx(4 * (size_t)nt);
        std::vector<float4> rh(k), rl(k);
        std::vector<int32_t> an(nt);
        std::uniform_real_distribution<float> P(0.f, 512.f);
        for (auto& v : tx) v = P(rng);
        for (int v = 0; v < k; ++v) { rh[v] = make_float4(P(rng), P(rng), P(rng), 1.f + (v % 8)); rl[v] = make_float4(1e-6f, -1e-6f, 1e-6f, 0.f); }
        for (int i = 0; i < nt; ++i) an[i] = i % k;
        float *dx, *dpart; float4 *dh, *dl; int32_t* da;
        cudaMalloc(&dx, tx.size() * 4); cudaMalloc(&dh, k * 16); cudaMalloc(&dl, k * 16); cudaMalloc(&da, nt * 4);
        cudaMalloc(&dpart, (size_t)nt * 4 * 4 * 8);
        cudaMemcpy(dx, tx.data(), tx.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dh, rh.data(), k * 16, cudaMemcpyHostToDevice);
        cudaMemcpy(dl, rl.data(), k * 16, cudaMemcpyHostToDevice);
        cudaMemcpy(da, an.data(), nt * 4, cudaMemcpyHostToDevice);
        run_coarse<2, false, 4, 0, 1>(nt, k, dx, dh, dl, da, dpart, sms, -1.f);
        run_coarse<2, false, 4, 1, 1>(nt, k, dx, dh, dl, da, dpart, sms, -1.f);
        run_coarse<2, false, 2, 0, 1>(nt, k, dx, dh, dl, da, dpart, sms, -1.f);
        run_coarse<2, false, 2, 1, 1>(nt, k, dx, dh, dl, da, dpart, sms, -1.f);
        run_coarse<2, false, 4, 0, 3>(nt, k, dx, dh, dl, da, dpart, sms, -1.f);
        run_coarse<2, false, 4, 1, 3>(nt, k, dx, dh, dl, da, dpart, sms, -1.f);
        run_coarse<2, false, 8, 0, 1>(nt, k, dx, dh, dl, da, dpart, sms, -1.f);
        run_coarse<2, false, 8, 1, 1>(nt, k, dx, dh, dl, da, dpart, sms, -1.f);
        run_coarse<2, false, 8, 5, 1>(nt, k, dx, dh, dl, da, dpart, sms, -1.f);
        // 3-D q = 0.8 (cfg5 shape, smaller)
        run_coarse<3, true, 2, 0, 1>(nt, k, dx, dh, dl, da, dpart, sms, -1.4f);
        run_coarse<3, true, 2, 0, 3>(nt, k, dx, dh, dl, da, dpart, sms, -1.4f);
        run_coarse<3, true, 4, 0, 1>(nt, k, dx, dh, dl, da, dpart, sms, -1.4f);
        run_coarse<3, true, 4, 0, 2>(nt, k, dx, dh, dl, da, dpart, sms, -1.4f);
        run_coarse<3, true, 8, 0, 1>(nt, k, dx, dh, dl, da, dpart, sms, -1.4f);
    }
    return 0;
}
