// Pipe-overlap microbenchmark (builder tool): cycles per warp-iteration per
// SMSP of loops that mix NF FFMA2, NM MUFU.EX2, NS scalar FFMA and NA FMNMX
// independent operations (inline PTX, no folding), at 32 warps per SM.
// Tells whether the FMA pipe (FFMA2 = 2 pipe cycles) and the XU pipe (MUFU =
// 8 cycles per warp) overlap, and what the ALU ops cost on top.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int NF, int NM, int NS, int NA>
__global__ void __launch_bounds__(256) k(float* out, int iters) {
    uint64_t f[NF > 0 ? NF : 1];
    float m[NM > 0 ? NM : 1], s[NS > 0 ? NS : 1], a[NA > 0 ? NA : 1];
    const float t = threadIdx.x * 1e-6f;
    for (int i = 0; i < (NF > 0 ? NF : 1); ++i) {
        float lo = 1.f + t + i, hi = 2.f + t + i;
        asm volatile("mov.b64 %0, {%1,%2};" : "=l"(f[i]) : "f"(lo), "f"(hi));
    }
    for (int i = 0; i < (NM > 0 ? NM : 1); ++i) m[i] = 0.5f + t + 0.01f * i;
    for (int i = 0; i < (NS > 0 ? NS : 1); ++i) s[i] = 0.25f + t + i;
    for (int i = 0; i < (NA > 0 ? NA : 1); ++i) a[i] = 0.75f + t + i;
    uint64_t c1, c2;
    {
        float x = 0.9999f, y = 1e-7f;
        asm volatile("mov.b64 %0, {%1,%1};" : "=l"(c1) : "f"(x));
        asm volatile("mov.b64 %0, {%1,%1};" : "=l"(c2) : "f"(y));
    }
    const float cm = 0.3f + t;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NF; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(f[i]) : "l"(c1), "l"(c2));
#pragma unroll
        for (int i = 0; i < NM; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(m[i]));
#pragma unroll
        for (int i = 0; i < NS; ++i) asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(s[i]) : "f"(cm));
#pragma unroll
        for (int i = 0; i < NA; ++i) asm volatile("min.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(cm));
    }
    float acc = 0.f;
    for (int i = 0; i < NF; ++i) {
        float lo, hi;
        asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(f[i]));
        acc += lo + hi;
    }
    for (int i = 0; i < NM; ++i) acc += m[i];
    for (int i = 0; i < NS; ++i) acc += s[i];
    for (int i = 0; i < NA; ++i) acc += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int NF, int NM, int NS, int NA>
void run(float* o, int sms, int clk_khz) {
    const int iters = 20000, blocks = sms * 4, threads = 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        k<NF, NM, NS, NA><<<blocks, threads>>>(o, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
    }
    // warp-iterations per SMSP: (blocks * threads / 32) warps * iters / (sms * 4 SMSPs)
    const double wi = (double)blocks * threads / 32 * iters / (sms * 4.0);
    const double cyc = ms * 1e-3 * clk_khz * 1e3 / wi;
    printf("FFMA2=%d MUFU=%d FFMA=%d FMNMX=%d : %.2f cycles/warp-iter/SMSP (pipe model: FMA %d, XU %d, issue %d)\n",
           NF, NM, NS, NA, cyc, 2 * NF + NS, 8 * NM, NF + NM + NS + NA);
}

int main() {
    float* o;
    cudaMalloc(&o, 148 * 4 * 256 * 4);
    int sms, clk;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    run<8, 0, 0, 0>(o, sms, clk);
    run<0, 2, 0, 0>(o, sms, clk);
    run<0, 0, 16, 0>(o, sms, clk);
    run<0, 0, 0, 16>(o, sms, clk);
    run<8, 2, 0, 0>(o, sms, clk);
    run<4, 2, 0, 0>(o, sms, clk);
    run<12, 2, 0, 0>(o, sms, clk);
    run<8, 2, 0, 4>(o, sms, clk);
    run<8, 2, 0, 8>(o, sms, clk);
    run<8, 0, 0, 8>(o, sms, clk);
    run<8, 0, 8, 0>(o, sms, clk);
    run<6, 2, 4, 4>(o, sms, clk);
    run<10, 3, 2, 3>(o, sms, clk);
    run<11, 4, 2, 2>(o, sms, clk);
    return 0;
}
