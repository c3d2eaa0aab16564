/* ORACLE (test infrastructure only) — maxent-stress energy, Eq.(1), FP64.
 *
 * PAPER.md P:163-171:  M(x) = sum_{{u,v} in E} w_uv (|x_u - x_v| - d_uv)^2
 *                            - alpha sum_{{u,v} notin E} ln |x_u - x_v|
 * in the general S form (P:163 footnote) with readings Q3 (phi_q) and Q4
 * (per-row S_i; one half of the ordered-pair sums, equal to the unordered
 * sums when S is symmetric):
 *   stress  = 1/2 sum_i sum_{j in S_i} w_ij (|x_i - x_j| - d_ij)^2
 *   entropy = 1/2 sum_i sum_{j notin S_i, j != i} phi_q(|x_i - x_j|),
 *             phi_0(r) = -ln r,  phi_q(r) = r^-q / q  (q > 0)
 *   M = stress + alpha * entropy.
 * A coincident non-S pair makes ln 0 undefined: OR_ECOINC (S:333 reading).
 * Row sums are formed independently and added in row order. */
#include <math.h>
#include <stdlib.h>

#include "mm_oracle.h"

int or_energy(int32_t n, int dim, const int64_t* srp, const int32_t* scol,
              const double* d, const double* w, const double* x,
              double alpha, double q, double out[3], int nthreads) {
    if (n < 0 || (dim != 2 && dim != 3) || !srp || !x || !out || q < 0.0) return OR_EINVAL;
    double* rs = (double*)calloc((size_t)n + 1, sizeof(double));
    double* re = (double*)calloc((size_t)n + 1, sizeof(double));
    if (!rs || !re) { free(rs); free(re); return OR_ENOMEM; }
    int err = 0;
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel num_threads(nthreads)
    {
        unsigned char* mark = (unsigned char*)calloc((size_t)n + 1, 1);
        if (!mark) {
#pragma omp atomic write
            err = OR_ENOMEM;
        }
#pragma omp for schedule(dynamic, 16)
        for (int32_t i = 0; i < n; ++i) {
            if (!mark) continue;
            const double* xi = x + (int64_t)i * dim;
            double s = 0.0, ent = 0.0;
            for (int64_t e = srp[i]; e < srp[i + 1]; ++e) {
                const double* xj = x + (int64_t)scol[e] * dim;
                double r2 = 0.0;
                for (int k = 0; k < dim; ++k) r2 += (xi[k] - xj[k]) * (xi[k] - xj[k]);
                const double dev = sqrt(r2) - d[e];
                s += w[e] * dev * dev;
                mark[scol[e]] = 1;
            }
            for (int32_t j = 0; j < n; ++j) {
                if (j == i || mark[j]) continue;
                const double* xj = x + (int64_t)j * dim;
                double r2 = 0.0;
                for (int k = 0; k < dim; ++k) r2 += (xi[k] - xj[k]) * (xi[k] - xj[k]);
                if (r2 == 0.0) {
#pragma omp atomic write
                    err = OR_ECOINC;
                    continue;
                }
                const double r = sqrt(r2);
                ent += (q == 0.0) ? -log(r) : pow(r, -q) / q;
            }
            for (int64_t e = srp[i]; e < srp[i + 1]; ++e) mark[scol[e]] = 0;
            rs[i] = s;
            re[i] = ent;
        }
        free(mark);
    }
    double S = 0.0, E = 0.0;
    for (int32_t i = 0; i < n; ++i) { S += rs[i]; E += re[i]; }
    free(rs); free(re);
    out[0] = 0.5 * S;
    out[1] = 0.5 * E;
    out[2] = out[0] + alpha * out[1];
    return err;
}
