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

template <int T, int BM, int MINB>
void run(int n, const float* x, float* part, int sms) {
    auto kern = k_repulse<2, false, false, T, BM, MINB>;
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
    printf("T=%d BMASK=%d MINB=%d regs=%d occ=%d G=%d  %.4f ms  %.4e pairs/s  (%.1f%% of 16 MUFU/clk/SM @1965)\n", T, BM,
           MINB, fa.numRegs, occ, s.G, ms, pairs / (ms * 1e-3), 100.0 * pairs / (ms * 1e-3) / (148 * 16 * 1.965e9));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("  error %s\n", cudaGetErrorString(e));
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
    run<4, 0, 1>(n, x, part, sms);
    run<4, 1, 1>(n, x, part, sms);
    run<4, 3, 1>(n, x, part, sms);
    run<4, 0, 6>(n, x, part, sms);
    run<4, 1, 6>(n, x, part, sms);
    run<2, 0, 1>(n, x, part, sms);
    run<2, 1, 1>(n, x, part, sms);
    run<6, 0, 1>(n, x, part, sms);
    run<6, 1, 1>(n, x, part, sms);
    run<6, 3, 1>(n, x, part, sms);
    run<8, 0, 1>(n, x, part, sms);
    run<8, 1, 1>(n, x, part, sms);
    run<8, 5, 1>(n, x, part, sms);
    run<8, 3, 1>(n, x, part, sms);
    run<8, 7, 1>(n, x, part, sms);
    run<8, 1, 3>(n, x, part, sms);
    run<12, 1, 1>(n, x, part, sms);
    run<12, 9, 1>(n, x, part, sms);
    return 0;
}
