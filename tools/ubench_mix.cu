// Practical ceiling of the exact-repulsion instruction mix (no memory traffic):
// per source: 2 packed target groups, group 0 batched reciprocal, group 1 two MUFU.RCP.
#include <cstdio>
#include "../paper_1506_04383_b200/csrc/mm_common.cuh"
using namespace mm;
namespace mm {
LaunchScope::LaunchScope(const char* n, cudaStream_t s) : name(n), stream(s), slot(-1) {}
LaunchScope::~LaunchScope() {}
}
template <int BM, int G>
__global__ void __launch_bounds__(256) k(float* out, int iters) {
    f2x X[G], Y[G], AX[G], AY[G];
    for (int g = 0; g < G; ++g) {
        X[g] = pk(threadIdx.x * 1e-3f + g, 0.5f + g);
        Y[g] = pk(0.25f * g, threadIdx.x * 2e-3f);
        asm volatile("" : "+l"(X[g]), "+l"(Y[g]));
        AX[g] = AY[g] = 0ull;
    }
    const f2x eps = pk(1e-18f, 1e-18f);
    float sx = 0.1f, sy = 0.2f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll 4
        for (int j = 0; j < 16; ++j) {
            sx += 0.001f;  // cheap source change (1 FADD per source)
#pragma unroll
            for (int g = 0; g < G; ++g) {
                f2x dx = sub_bc(X[g], sx), dy = sub_bc(Y[g], sy);
                f2x r2 = fma2(dx, dx, eps);
                r2 = fma2(dy, dy, r2);
                float r0, r1;
                upk(r2, r0, r1);
                f2x inv;
                if ((BM >> g) & 1) {
                    const float ip = rcp_approx(r0 * r1);
                    inv = mul2(pk(r1, r0), pk(ip, ip));
                } else {
                    inv = pk(rcp_approx(r0), rcp_approx(r1));
                }
                AX[g] = fma2(dx, inv, AX[g]);
                AY[g] = fma2(dy, inv, AY[g]);
            }
        }
    }
    float s = 0.f;
    for (int g = 0; g < G; ++g) {
        float a, b;
        upk(AX[g], a, b);
        s += a + b;
        upk(AY[g], a, b);
        s += a + b;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int BM, int G>
void run(float* o, int blocks_per_sm) {
    const int iters = 2000, sms = 148, blocks = sms * blocks_per_sm;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k<BM, G><<<blocks, 256>>>(o, 10);
    cudaEventRecord(a);
    k<BM, G><<<blocks, 256>>>(o, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k<BM, G>);
    const double pairs = (double)blocks * 256 * iters * 16 * 2 * G;
    printf("BM=%d G=%d blocks/SM=%d regs=%d: %.4e pairs/s = %.2f pairs/clk/SM @1965\n", BM, G, blocks_per_sm,
           fa.numRegs, pairs / (ms * 1e-3), pairs / (ms * 1e-3) / 148 / 1.965e9);
}
int main() {
    float* o;
    cudaMalloc(&o, 148 * 8 * 256 * 4);
    for (int bps : {2, 4, 8}) {
        run<0, 2>(o, bps);
        run<1, 2>(o, bps);
        run<3, 2>(o, bps);
        run<1, 4>(o, bps);
        run<5, 4>(o, bps);
    }
    return 0;
}
