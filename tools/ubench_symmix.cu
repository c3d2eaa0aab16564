// Instruction-mix ceiling of the symmetric (rotation) repulsion loop, no memory:
// MODE 0: as k_repulse_sym (SHFL of sx, sy, bx, by per step, j-side FFMAs)
// MODE 1: j-side FFMAs, sources shuffled, accumulators kept in place (2 SHFL/step)
// MODE 2: j-side FFMAs, no shuffles at all (source changed by one FADD)
// MODE 3: no j side, sources shuffled (the one-sided mix + 2 SHFL/step)
// MODE 4: as 0, but the j side accumulates packed (FFMA2) and folds lo+hi per step
// MODE 5: as 0, but sources come from shared memory at a rotated index (LDS), only bx/by shuffled
// MODE 6: as 0 with scalar (unpacked) target arithmetic throughout
#include <cstdio>
#include "../paper_1506_04383_b200/csrc/mm_common.cuh"
using namespace mm;
namespace mm {
LaunchScope::LaunchScope(const char* n, cudaStream_t s) : name(n), stream(s), slot(-1) {}
LaunchScope::~LaunchScope() {}
}
template <int MODE, int G, int UNR>
__global__ void __launch_bounds__(256) k(float* out, int iters) {
    f2x X[G], Y[G], AX[G], AY[G];
    const int lane = threadIdx.x & 31, nxt = (lane + 1) & 31;
    for (int g = 0; g < G; ++g) {
        X[g] = pk(threadIdx.x * 1e-3f + g, 0.5f + g);
        Y[g] = pk(0.25f * g, threadIdx.x * 2e-3f);
        asm volatile("" : "+l"(X[g]), "+l"(Y[g]));
        AX[g] = AY[g] = 0ull;
    }
    const f2x eps = pk(1e-18f, 1e-18f);
    float sx = 0.1f + lane, sy = 0.2f, bx = 0.f, by = 0.f;
    __shared__ float2 ssrc[8][32];
    ssrc[threadIdx.x >> 5][lane] = make_float2(sx, sy);
    __syncwarp();
    for (int it = 0; it < iters; ++it) {
#pragma unroll UNR
        for (int j = 0; j < 32; ++j) {
            if (MODE == 2) sx += 0.001f;
            if (MODE == 5) {
                const float2 v = ssrc[threadIdx.x >> 5][(lane + j) & 31];
                sx = v.x;
                sy = v.y;
            }
            if (MODE == 6) {
                float fx[2 * G], fy[2 * G];
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    upk(X[g], fx[2 * g], fx[2 * g + 1]);
                    upk(Y[g], fy[2 * g], fy[2 * g + 1]);
                }
                float ax[2 * G], ay[2 * G];
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    upk(AX[g], ax[2 * g], ax[2 * g + 1]);
                    upk(AY[g], ay[2 * g], ay[2 * g + 1]);
                }
#pragma unroll
                for (int t = 0; t < 2 * G; t += 2) {
                    const float dx0 = fx[t] - sx, dy0 = fy[t] - sy, dx1 = fx[t + 1] - sx, dy1 = fy[t + 1] - sy;
                    const float r0 = fmaf(dy0, dy0, fmaf(dx0, dx0, 1e-18f));
                    const float r1 = fmaf(dy1, dy1, fmaf(dx1, dx1, 1e-18f));
                    float i0, i1;
                    if ((t & 2) == 0) {
                        const float ip = rcp_approx(r0 * r1);
                        i0 = r1 * ip;
                        i1 = r0 * ip;
                    } else {
                        i0 = rcp_approx(r0);
                        i1 = rcp_approx(r1);
                    }
                    ax[t] = fmaf(dx0, i0, ax[t]);
                    ay[t] = fmaf(dy0, i0, ay[t]);
                    ax[t + 1] = fmaf(dx1, i1, ax[t + 1]);
                    ay[t + 1] = fmaf(dy1, i1, ay[t + 1]);
                    bx = fmaf(-dx0, i0, bx);
                    by = fmaf(-dy0, i0, by);
                    bx = fmaf(-dx1, i1, bx);
                    by = fmaf(-dy1, i1, by);
                }
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    AX[g] = pk(ax[2 * g], ax[2 * g + 1]);
                    AY[g] = pk(ay[2 * g], ay[2 * g + 1]);
                }
                sx = __shfl_sync(0xffffffffu, sx, nxt);
                sy = __shfl_sync(0xffffffffu, sy, nxt);
                bx = __shfl_sync(0xffffffffu, bx, nxt);
                by = __shfl_sync(0xffffffffu, by, nxt);
                continue;
            }
            f2x BX = pk(bx, 0.f), BY = pk(by, 0.f);
#pragma unroll
            for (int g = 0; g < G; ++g) {
                f2x dx = sub_bc(X[g], sx), dy = sub_bc(Y[g], sy);
                f2x r2 = fma2(dx, dx, eps);
                r2 = fma2(dy, dy, r2);
                float r0, r1;
                upk(r2, r0, r1);
                f2x inv;
                if ((g & 1) == 0) {
                    const float ip = rcp_approx(r0 * r1);
                    inv = mul2(pk(r1, r0), pk(ip, ip));
                } else {
                    inv = pk(rcp_approx(r0), rcp_approx(r1));
                }
                AX[g] = fma2(dx, inv, AX[g]);
                AY[g] = fma2(dy, inv, AY[g]);
                if (MODE == 4) {
                    BX = fma2(dx, inv, BX);
                    BY = fma2(dy, inv, BY);
                } else if (MODE != 3) {
                    float i0, i1, a0, a1;
                    upk(inv, i0, i1);
                    upk(dx, a0, a1);
                    bx = fmaf(-a0, i0, bx);
                    bx = fmaf(-a1, i1, bx);
                    upk(dy, a0, a1);
                    by = fmaf(-a0, i0, by);
                    by = fmaf(-a1, i1, by);
                }
            }
            if (MODE == 4) {
                float a, b;
                upk(BX, a, b);
                bx = a + b;
                upk(BY, a, b);
                by = a + b;
            }
            if (MODE != 2 && MODE != 5) {
                sx = __shfl_sync(0xffffffffu, sx, nxt);
                sy = __shfl_sync(0xffffffffu, sy, nxt);
            }
            if (MODE == 0 || MODE == 4 || MODE == 5) {
                bx = __shfl_sync(0xffffffffu, bx, nxt);
                by = __shfl_sync(0xffffffffu, by, nxt);
            }
        }
    }
    float s = bx + by;
    for (int g = 0; g < G; ++g) {
        float a, b;
        upk(AX[g], a, b);
        s += a + b;
        upk(AY[g], a, b);
        s += a + b;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int MODE, int G, int UNR>
void run(float* o, int blocks_per_sm) {
    const int iters = 1000, sms = 148, blocks = sms * blocks_per_sm;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k<MODE, G, UNR><<<blocks, 256>>>(o, 10);
    cudaEventRecord(a);
    k<MODE, G, UNR><<<blocks, 256>>>(o, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k<MODE, G, UNR>);
    const double pairs = (double)blocks * 256 * iters * 32 * 2 * G;
    printf("MODE=%d G=%d UNR=%d blocks/SM=%d regs=%d: %.2f pair-evals/clk/SM @1965\n", MODE, G, UNR, blocks_per_sm,
           fa.numRegs, pairs / (ms * 1e-3) / 148 / 1.965e9);
}
int main() {
    float* o;
    cudaMalloc(&o, 148 * 8 * 256 * 4);
    for (int bps : {3, 4}) {
        run<0, 2, 8>(o, bps);
        run<4, 2, 8>(o, bps);
        run<5, 2, 8>(o, bps);
        run<6, 2, 8>(o, bps);
        run<0, 4, 4>(o, bps);
        run<4, 4, 4>(o, bps);
        run<5, 4, 4>(o, bps);
        run<6, 4, 4>(o, bps);
    }
    return 0;
}
