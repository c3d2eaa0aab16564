/* ORACLE (test infrastructure only) — Eq.(2) and Eq.(3) sweeps, FP64.
 *
 * Eq.(2), PAPER.md P:176-181 (in S-set form, P:163 footnote; BASELINE.json
 * north_star's exponent q):
 *   x_i <- (1/rho_i) sum_{j in S_i} w_ij (x_j + d_ij (x_i-x_j)/|x_i-x_j|)
 *        + (alpha/rho_i) sum_{j notin S_i, j != i} (x_i-x_j)/|x_i-x_j|^(q+2),
 *   rho_i = sum_{j in S_i} w_ij.
 * Synchronous (Jacobi) iteration: "The current iteration uses the
 * coordinates that have been computed in the previous iteration", so
 * every row reads only the input x.  The sum over j notin S_i is evaluated
 * directly (a membership mark per row), never as all-pairs minus S.
 * Coincident pairs contribute 0 to both the unit vector and r (Q6).
 *
 * Eq.(3): the entropy term becomes
 *   sum_{j != i, P(j) = P(i)} r(i,j)
 * + sum_{v' != H(i)} nu(v') (x_i - x'_v')/|x_i - x'_v'|^(q+2)
 * - sum_{j in S_i} r(i,j)
 * with P the one-level clustering and H the map to the level h' above
 * (reading Q8), nu(v') the number of current-level vertices that
 * v' represents (Q10) and x'_v' their unweighted midpoint (P:283-284,
 * Q11), computed from the sweep's input x (Q12). */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "mm_oracle.h"

/* acc += s * (xi - xj) / |xi - xj|^(q+2); contributes 0 when coincident */
static void add_r(int dim, const double* xi, const double* xj, double q, double s, double* acc) {
    double diff[3], r2 = 0.0;
    for (int k = 0; k < dim; ++k) { diff[k] = xi[k] - xj[k]; r2 += diff[k] * diff[k]; }
    if (r2 == 0.0) return;
    const double den = (q == 0.0) ? r2 : pow(r2, 0.5 * (q + 2.0));
    for (int k = 0; k < dim; ++k) acc[k] += s * diff[k] / den;
}

/* first term of Eq.(2): rho_i and A_i = sum w (x_j + d u_ij) */
static double stress_part(int32_t i, int dim, const int64_t* srp, const int32_t* scol,
                          const double* d, const double* w, const double* x, double* A) {
    double rho = 0.0;
    const double* xi = x + (int64_t)i * dim;
    for (int k = 0; k < dim; ++k) A[k] = 0.0;
    for (int64_t e = srp[i]; e < srp[i + 1]; ++e) {
        const double* xj = x + (int64_t)scol[e] * dim;
        double diff[3], r2 = 0.0;
        for (int k = 0; k < dim; ++k) { diff[k] = xi[k] - xj[k]; r2 += diff[k] * diff[k]; }
        const double dist = sqrt(r2);
        rho += w[e];
        for (int k = 0; k < dim; ++k) {
            const double u = (dist > 0.0) ? diff[k] / dist : 0.0;
            A[k] += w[e] * (xj[k] + d[e] * u);
        }
    }
    return rho;
}

int or_sweep_exact(int32_t n, int dim, const int64_t* srp, const int32_t* scol,
                   const double* d, const double* w, const double* x,
                   double alpha, double q, const int32_t* rows, int32_t nrows,
                   double* out, int nthreads) {
    if (n < 0 || (dim != 2 && dim != 3) || !srp || !x || !out || q < 0.0) return OR_EINVAL;
    if (!rows) nrows = n;
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
        for (int32_t t = 0; t < nrows; ++t) {
            if (!mark) continue;
            const int32_t i = rows ? rows[t] : t;
            double A[3], R[3] = {0.0, 0.0, 0.0};
            const double rho = stress_part(i, dim, srp, scol, d, w, x, A);
            if (!(rho > 0.0)) {
#pragma omp atomic write
                err = OR_ERHO;
                continue;
            }
            for (int64_t e = srp[i]; e < srp[i + 1]; ++e) mark[scol[e]] = 1;
            const double* xi = x + (int64_t)i * dim;
            for (int32_t j = 0; j < n; ++j) {
                if (j == i || mark[j]) continue;
                add_r(dim, xi, x + (int64_t)j * dim, q, 1.0, R);
            }
            for (int64_t e = srp[i]; e < srp[i + 1]; ++e) mark[scol[e]] = 0;
            for (int k = 0; k < dim; ++k) out[(int64_t)t * dim + k] = (A[k] + alpha * R[k]) / rho;
        }
        free(mark);
    }
    return err;
}

int or_centroids(int32_t n, int dim, const double* x, const int32_t* anc, int32_t k,
                 double* xc, int64_t* nu) {
    if (n < 0 || k <= 0 || !x || !anc || !xc || !nu) return OR_EINVAL;
    for (int32_t v = 0; v < k; ++v) {
        nu[v] = 0;
        for (int c = 0; c < dim; ++c) xc[(int64_t)v * dim + c] = 0.0;
    }
    for (int32_t u = 0; u < n; ++u) {
        const int32_t v = anc[u];
        if (v < 0 || v >= k) return OR_EINVAL;
        nu[v] += 1;
        for (int c = 0; c < dim; ++c) xc[(int64_t)v * dim + c] += x[(int64_t)u * dim + c];
    }
    for (int32_t v = 0; v < k; ++v) {
        if (nu[v] == 0) return OR_EINVAL; /* the map must be surjective */
        for (int c = 0; c < dim; ++c) xc[(int64_t)v * dim + c] /= (double)nu[v];
    }
    return 0;
}

int or_sweep_approx(int32_t n, int dim, const int64_t* srp, const int32_t* scol,
                    const double* d, const double* w, const double* x,
                    double alpha, double q, const int32_t* parent, const int32_t* anc, int32_t k,
                    const int32_t* rows, int32_t nrows, double* out, int nthreads) {
    if (n < 0 || (dim != 2 && dim != 3) || !srp || !x || !out || !parent || !anc || k <= 0 ||
        q < 0.0)
        return OR_EINVAL;
    if (!rows) nrows = n;
    /* coarse representatives x' and counts nu */
    double* xc = (double*)malloc(sizeof(double) * (size_t)k * dim);
    int64_t* nu = (int64_t*)malloc(sizeof(int64_t) * (size_t)k);
    /* children lists of the one-level map P (for the same-cluster sum) */
    int32_t np = 0;
    for (int32_t u = 0; u < n; ++u) if (parent[u] + 1 > np) np = parent[u] + 1;
    int64_t* cstart = (int64_t*)calloc((size_t)np + 1, sizeof(int64_t));
    int32_t* child = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    if (!xc || !nu || !cstart || !child) {
        free(xc); free(nu); free(cstart); free(child);
        return OR_ENOMEM;
    }
    int err = or_centroids(n, dim, x, anc, k, xc, nu);
    if (err) { free(xc); free(nu); free(cstart); free(child); return err; }
    for (int32_t u = 0; u < n; ++u) {
        if (parent[u] < 0) { free(xc); free(nu); free(cstart); free(child); return OR_EINVAL; }
        cstart[parent[u] + 1] += 1;
    }
    for (int32_t p = 0; p < np; ++p) cstart[p + 1] += cstart[p];
    {
        int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(np > 0 ? np : 1));
        if (!fill) { free(xc); free(nu); free(cstart); free(child); return OR_ENOMEM; }
        for (int32_t p = 0; p < np; ++p) fill[p] = cstart[p];
        for (int32_t u = 0; u < n; ++u) child[fill[parent[u]]++] = u; /* ascending ids */
        free(fill);
    }
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(dynamic, 16) num_threads(nthreads)
    for (int32_t t = 0; t < nrows; ++t) {
        const int32_t i = rows ? rows[t] : t;
        const double* xi = x + (int64_t)i * dim;
        double A[3], R[3] = {0.0, 0.0, 0.0};
        const double rho = stress_part(i, dim, srp, scol, d, w, x, A);
        if (!(rho > 0.0)) {
#pragma omp atomic write
            err = OR_ERHO;
            continue;
        }
        /* (1) same-cluster vertices, exact r-values */
        const int32_t p = parent[i];
        for (int64_t c = cstart[p]; c < cstart[p + 1]; ++c) {
            const int32_t j = child[c];
            if (j != i) add_r(dim, xi, x + (int64_t)j * dim, q, 1.0, R);
        }
        /* (2) coarse representatives v' != H(i), weighted by nu(v') */
        const int32_t hi = anc[i];
        for (int32_t v = 0; v < k; ++v) {
            if (v == hi) continue;
            add_r(dim, xi, xc + (int64_t)v * dim, q, (double)nu[v], R);
        }
        /* (3) subtract the S-pairs' r-values added "in good faith" (Q9) */
        for (int64_t e = srp[i]; e < srp[i + 1]; ++e)
            add_r(dim, xi, x + (int64_t)scol[e] * dim, q, -1.0, R);
        for (int kk = 0; kk < dim; ++kk) out[(int64_t)t * dim + kk] = (A[kk] + alpha * R[kk]) / rho;
    }
    free(xc); free(nu); free(cstart); free(child);
    return err;
}

double or_relative_change(int64_t len, const double* x_old, const double* x_new) {
    double num = 0.0, den = 0.0;
    for (int64_t t = 0; t < len; ++t) {
        const double dlt = x_new[t] - x_old[t];
        num += dlt * dlt;
        den += x_old[t] * x_old[t];
    }
    if (den == 0.0) return INFINITY;
    return sqrt(num) / sqrt(den);
}
