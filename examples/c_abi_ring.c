/* c_abi_ring.c — the C-ABI used from plain C (no Python, no torch).
 *
 * One exact Jacobi sweep (Eq.(2)) of the ring C_n drawn
 * as a regular n-gon of radius R, through mm_sweep, checked on the host
 * against the closed form of SURVEY §8(c) pin P3:
 *   R' = R cos(2 pi/n) + d sin(pi/n) + (alpha/2) sum_{k=2}^{n-2} R c_k / (2 R^2 c_k)^(1+q/2),
 *   c_k = 1 - cos(2 pi k/n)   (q = 0: the sum is (n-3)/(2R)),
 * then mm_energy on the 3-path worked example (tests/golden/path3_energy.txt).
 * The coordinates are computed here in double from the FP32 inputs, so the
 * check does not depend on any other part of the repository.
 *
 * Build (done by __graft_entry__.build()):
 *   gcc -O2 -std=c99 -I include examples/c_abi_ring.c -o examples/c_abi_ring \
 *       -L paper_1506_04383_b200 -lmm_b200 -L /usr/local/cuda/lib64 -lcudart -lm \
 *       -Wl,-rpath,$ORIGIN/../paper_1506_04383_b200 -Wl,-rpath,/usr/local/cuda/lib64
 * Run: examples/c_abi_ring [n] [q]   (exit 0 = pass) */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "mm.h"

/* the few CUDA runtime calls used, declared here so that no CUDA header is needed */
typedef int cudaError_t;
enum { cudaMemcpyHostToDevice = 1, cudaMemcpyDeviceToHost = 2 };
extern cudaError_t cudaMalloc(void** p, size_t bytes);
extern cudaError_t cudaFree(void* p);
extern cudaError_t cudaMemcpy(void* dst, const void* src, size_t bytes, int kind);
extern cudaError_t cudaDeviceSynchronize(void);

#define CK(call)                                                                  \
    do {                                                                          \
        int rc_ = (int)(call);                                                    \
        if (rc_ != 0) {                                                           \
            fprintf(stderr, "%s failed: %d (%s)\n", #call, rc_, mm_last_error()); \
            return 2;                                                             \
        }                                                                         \
    } while (0)

static void* dev_copy(const void* h, size_t bytes) {
    void* d = NULL;
    if (cudaMalloc(&d, bytes) != 0) return NULL;
    if (cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice) != 0) return NULL;
    return d;
}

static int ring_sweep(int32_t n, float q) {
    const double pi = 3.14159265358979323846;
    const double R = 0.5 * n / pi, alpha = 0.05, dd = 1.0;
    int64_t* rp = malloc(sizeof(int64_t) * (n + 1));
    int32_t* col = malloc(sizeof(int32_t) * 2 * (size_t)n);
    float* d = malloc(sizeof(float) * 2 * (size_t)n);
    float* w = malloc(sizeof(float) * 2 * (size_t)n);
    float* x = malloc(sizeof(float) * 2 * (size_t)n);
    float* y = malloc(sizeof(float) * 2 * (size_t)n);
    for (int32_t i = 0; i < n; ++i) {
        rp[i] = 2 * (int64_t)i;
        col[2 * i] = (i + n - 1) % n;
        col[2 * i + 1] = (i + 1) % n;
        d[2 * i] = d[2 * i + 1] = (float)dd;
        w[2 * i] = w[2 * i + 1] = (float)(1.0 / (dd * dd));
        x[2 * i] = (float)(R * cos(2 * pi * i / n));
        x[2 * i + 1] = (float)(R * sin(2 * pi * i / n));
    }
    rp[n] = 2 * (int64_t)n;
    mm_sset S = {n, 2 * (int64_t)n, dev_copy(rp, sizeof(int64_t) * (n + 1)), dev_copy(col, 8 * (size_t)n),
                 dev_copy(d, 8 * (size_t)n), dev_copy(w, 8 * (size_t)n)};
    float* xd = dev_copy(x, 8 * (size_t)n);
    float* yd = NULL;
    if (!S.row_ptr || !S.col || !S.d || !S.w || !xd || cudaMalloc((void**)&yd, 8 * (size_t)n) != 0) {
        fprintf(stderr, "device allocation failed\n");
        return 2;
    }
    CK(mm_validate_sset(&S, NULL));
    CK(mm_sweep(&S, 2, (float)alpha, q, NULL, xd, yd, NULL, NULL, 0, NULL));
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(y, yd, 8 * (size_t)n, cudaMemcpyDeviceToHost));
    /* closed form per vertex, from the exact radius of its FP32 input point */
    double ent = 0.0;
    if (q == 0.0f) {
        ent = alpha * (n - 3) / (4.0 * R);
    } else {
        for (int32_t k = 2; k <= n - 2; ++k) {
            const double ck = 1.0 - cos(2 * pi * k / n);
            ent += R * ck / pow(2.0 * R * R * ck, 1.0 + q / 2.0);
        }
        ent *= 0.5 * alpha;
    }
    double err = 0.0, lo[2] = {1e300, 1e300}, hi[2] = {-1e300, -1e300};
    for (int32_t i = 0; i < n; ++i) {
        const double xi = x[2 * i], yi = x[2 * i + 1], rin = sqrt(xi * xi + yi * yi);
        const double rp_ = rin * cos(2 * pi / n) + dd * sin(pi / n) + ent;
        const double wx = xi * rp_ / rin, wy = yi * rp_ / rin;
        const double e = fmax(fabs(y[2 * i] - wx), fabs(y[2 * i + 1] - wy));
        if (e > err) err = e;
        lo[0] = fmin(lo[0], wx); hi[0] = fmax(hi[0], wx);
        lo[1] = fmin(lo[1], wy); hi[1] = fmax(hi[1], wy);
    }
    const double diam = sqrt((hi[0] - lo[0]) * (hi[0] - lo[0]) + (hi[1] - lo[1]) * (hi[1] - lo[1]));
    const int ok = err <= 1e-4 * diam;
    printf("ring n=%d q=%.2f: max |gpu - closed form| = %.3e = %.2e x diameter (tolerance 1e-4) %s\n", n, q, err,
           err / diam, ok ? "PASS" : "FAIL");
    cudaFree((void*)S.row_ptr); cudaFree((void*)S.col); cudaFree((void*)S.d); cudaFree((void*)S.w);
    cudaFree(xd); cudaFree(yd);
    free(rp); free(col); free(d); free(w); free(x); free(y);
    return ok ? 0 : 1;
}

static int path3_energy(void) {
    /* path a-b-c at 0, 1, 2 on a line, S = E, d = w = 1, alpha = 0.008, q = 0:
     * stress 0, entropy = -ln 2 (the only non-S pair, counted once), total = -0.008 ln 2 */
    const int64_t rp[4] = {0, 1, 3, 4};
    const int32_t col[4] = {1, 0, 2, 1};
    const float d[4] = {1, 1, 1, 1}, w[4] = {1, 1, 1, 1};
    const float x[6] = {0, 0, 1, 0, 2, 0};
    mm_sset S = {3, 4, dev_copy(rp, sizeof rp), dev_copy(col, sizeof col), dev_copy(d, sizeof d),
                 dev_copy(w, sizeof w)};
    float* xd = dev_copy(x, sizeof x);
    double out[3];
    CK(mm_energy(&S, 2, 0.008, 0.0, xd, out, NULL));
    const double want = -0.008 * log(2.0);
    const int ok = fabs(out[0]) < 1e-7 && fabs(out[1] + log(2.0)) < 1e-6 && fabs(out[2] - want) < 1e-8;
    printf("path3 energy: stress %.3e entropy %.9f total %.9f (want 0, %.9f, %.9f) %s\n", out[0], out[1], out[2],
           -log(2.0), want, ok ? "PASS" : "FAIL");
    cudaFree((void*)S.row_ptr); cudaFree((void*)S.col); cudaFree((void*)S.d); cudaFree((void*)S.w); cudaFree(xd);
    return ok ? 0 : 1;
}

int main(int argc, char** argv) {
    const int32_t n = argc > 1 ? atoi(argv[1]) : 65536;
    const float q = argc > 2 ? (float)atof(argv[2]) : 0.0f;
    printf("%s\n", mm_version());
    int rc = ring_sweep(n, q);
    if (rc == 0) rc = path3_energy();
    return rc;
}
