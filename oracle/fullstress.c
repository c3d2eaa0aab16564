/* ORACLE (test infrastructure only) — full stress F(x) and the optimal scale,
 * FP64.
 *
 * "The first metric is the full stress measure,
 *   F(x) = sum_{u,v in V} w_uv (||x_u - x_v|| - d_uv)^2"
 * with d_uv the shortest-path distance (unit edge lengths P:350)
 * and w_uv = d_uv^-2 ("Throughout the paper, we use this as a
 * weight factor").  P:327-328: "We find a scalar s such that
 *   sum_{u,v} w_uv (s ||x_u - x_v|| - d_uv)^2 is minimized."
 * Reading R5: unordered pairs u < v; the quadratic in s,
 *   F(s) = s^2 B - 2 s A + C,  A = sum w d l,  B = sum w l^2,  C = sum w d^2,
 * has its minimum at s* = A / B.  Distances by a plain BFS from every vertex;
 * unreachable pairs are skipped (the inputs are connected).
 * out[0] = F(1), out[1] = s*, out[2] = F(s*), out[3] = pairs counted. */
#include <math.h>
#include <stdlib.h>

#include "mm_oracle.h"

int or_full_stress(int32_t n, const int64_t* rp, const int32_t* col, int dim, const double* x, double out[4],
                   int nthreads) {
    if (n <= 0 || !rp || !x || !out || (dim != 2 && dim != 3)) return OR_EINVAL;
    double* rowA = (double*)calloc((size_t)n, sizeof(double));
    double* rowB = (double*)calloc((size_t)n, sizeof(double));
    double* rowC = (double*)calloc((size_t)n, sizeof(double));
    double* rowF = (double*)calloc((size_t)n, sizeof(double));
    int64_t* rowP = (int64_t*)calloc((size_t)n, sizeof(int64_t));
    if (!rowA || !rowB || !rowC || !rowF || !rowP) {
        free(rowA); free(rowB); free(rowC); free(rowF); free(rowP);
        return OR_ENOMEM;
    }
    int err = 0;
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel num_threads(nthreads)
    {
        int32_t* dist = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
        int32_t* queue = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
        if (!dist || !queue) {
#pragma omp atomic write
            err = OR_ENOMEM;
        }
#pragma omp for schedule(dynamic, 8)
        for (int32_t u = 0; u < n; ++u) {
            if (!dist || !queue) continue;
            for (int32_t v = 0; v < n; ++v) dist[v] = -1;
            int32_t head = 0, tail = 0;
            dist[u] = 0;
            queue[tail++] = u;
            while (head < tail) {
                const int32_t a = queue[head++];
                for (int64_t e = rp[a]; e < rp[a + 1]; ++e) {
                    const int32_t b = col[e];
                    if (dist[b] < 0) { dist[b] = dist[a] + 1; queue[tail++] = b; }
                }
            }
            double A = 0.0, B = 0.0, C = 0.0, F = 0.0;
            int64_t P = 0;
            for (int32_t v = u + 1; v < n; ++v) {
                if (dist[v] <= 0) continue;
                double l2 = 0.0;
                for (int k = 0; k < dim; ++k) {
                    const double t = x[(int64_t)u * dim + k] - x[(int64_t)v * dim + k];
                    l2 += t * t;
                }
                const double l = sqrt(l2), dd = (double)dist[v], w = 1.0 / (dd * dd);
                A += w * dd * l;
                B += w * l * l;
                C += w * dd * dd;
                F += w * (l - dd) * (l - dd);
                ++P;
            }
            rowA[u] = A; rowB[u] = B; rowC[u] = C; rowF[u] = F; rowP[u] = P;
        }
        free(dist);
        free(queue);
    }
    double A = 0.0, B = 0.0, C = 0.0, F = 0.0;
    int64_t P = 0;
    for (int32_t u = 0; u < n; ++u) { A += rowA[u]; B += rowB[u]; C += rowC[u]; F += rowF[u]; P += rowP[u]; }
    free(rowA); free(rowB); free(rowC); free(rowF); free(rowP);
    if (err) return err;
    const double s = (B > 0.0) ? A / B : 1.0;
    out[0] = F;
    out[1] = s;
    out[2] = s * s * B - 2.0 * s * A + C;
    out[3] = (double)P;
    return 0;
}
