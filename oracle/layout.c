/* ORACLE (test infrastructure only) — coarse S sets, initial layout,
 * prolongation and the multilevel driver, FP64.
 *
 * "After computing an initial layout on the coarsest hierarchy
 * level, we improve the drawing on each finer level by iterating Eq.(2)."
 * P:240-242 prolongation; P:247-248 coarse distances sqrt(c(u)) + sqrt(c(v));
 * P:254-257 iterations.  BASELINE.json fixes alpha and the sweep counts per
 * level (the paper's alpha schedule is a later row).
 * Readings: Q7 (coarse S = E^l, d = c_u^(1/dim) + c_v^(1/dim), w = d^-2;
 * finest level keeps the user's d, w), Q13 (h' = min(h, L-l); level L exact),
 * Q14 (box init), Q15 (prolongation = copy parent + U[-1e-3, 1e-3] jitter). */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "mm_oracle.h"

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

static double root_dim(double c, int dim) { return dim == 2 ? sqrt(c) : cbrt(c); }

int or_coarse_sset(int32_t n, int64_t nnz, const int64_t* rp, const int32_t* col,
                   const int64_t* c, int dim, double* d, double* w) {
    if (n < 0 || !rp || !c || (dim != 2 && dim != 3)) return OR_EINVAL;
    for (int32_t u = 0; u < n; ++u)
        for (int64_t e = rp[u]; e < rp[u + 1]; ++e) {
            const double dd = root_dim((double)c[u], dim) + root_dim((double)c[col[e]], dim);
            d[e] = dd;
            w[e] = 1.0 / (dd * dd);
        }
    (void)nnz;
    return 0;
}

int or_init_box(int32_t n, int dim, double box, uint64_t seed, int32_t level, double* x) {
    if (n < 0 || !x) return OR_EINVAL;
    for (int32_t u = 0; u < n; ++u)
        for (int k = 0; k < dim; ++k)
            x[(int64_t)u * dim + k] =
                box * or_uniform24(or_key_vertex(seed, OR_TAG_INIT, (uint64_t)level, (uint64_t)u, dim, k));
    return 0;
}

int or_prolong(int32_t n_fine, int dim, const int32_t* parent, const double* xc,
               uint64_t seed, int32_t level, double* x) {
    if (n_fine < 0 || !parent || !xc || !x) return OR_EINVAL;
    for (int32_t u = 0; u < n_fine; ++u)
        for (int k = 0; k < dim; ++k) {
            const double U = or_uniform24(or_key_vertex(seed, OR_TAG_JITTER, (uint64_t)level, (uint64_t)u, dim, k));
            x[(int64_t)u * dim + k] = xc[(int64_t)parent[u] * dim + k] + 1e-3 * (2.0 * U - 1.0);
        }
    return 0;
}

/* the paper's disc prolongation: "picking an angle uniformly at
 * random in [0, 2pi] and a distance to P uniformly at random in [0, r]",
 * r = sqrt(c(v')); dim 3 (extension): radius c^(1/3), direction from a
 * uniform z in [-1, 1] and angle (reading R7). */
int or_prolong_disc(int32_t n_fine, int dim, const int32_t* parent, const double* xc, const int64_t* c_coarse,
                    uint64_t seed, int32_t level, double* x) {
    if (n_fine < 0 || !parent || !xc || !x || !c_coarse) return OR_EINVAL;
    for (int32_t u = 0; u < n_fine; ++u) {
        const int32_t p = parent[u];
        const double U0 = or_uniform24(or_key_vertex(seed, OR_TAG_DISC, (uint64_t)level, (uint64_t)u, 3, 0));
        const double U1 = or_uniform24(or_key_vertex(seed, OR_TAG_DISC, (uint64_t)level, (uint64_t)u, 3, 1));
        const double U2 = or_uniform24(or_key_vertex(seed, OR_TAG_DISC, (uint64_t)level, (uint64_t)u, 3, 2));
        const double theta = 2.0 * M_PI * U0;
        const double r = root_dim((double)c_coarse[p], dim) * U1;
        if (dim == 2) {
            x[(int64_t)u * 2 + 0] = xc[(int64_t)p * 2 + 0] + r * cos(theta);
            x[(int64_t)u * 2 + 1] = xc[(int64_t)p * 2 + 1] + r * sin(theta);
        } else {
            const double z = 2.0 * U2 - 1.0, s = sqrt(1.0 - z * z);
            x[(int64_t)u * 3 + 0] = xc[(int64_t)p * 3 + 0] + r * s * cos(theta);
            x[(int64_t)u * 3 + 1] = xc[(int64_t)p * 3 + 1] + r * s * sin(theta);
            x[(int64_t)u * 3 + 2] = xc[(int64_t)p * 3 + 2] + r * z;
        }
    }
    return 0;
}

int or_layout(int32_t n, int dim, const int64_t* rp, const int32_t* col,
              const int64_t* srp, const int32_t* scol, const double* d, const double* w,
              double alpha, double q, int h, const int32_t* sweeps, int32_t nsweeps,
              uint64_t seed, int32_t n_stop, const double* x_init, double* out,
              double energy_out[3], int32_t* levels_out, int nthreads) {
    if (n <= 0 || (dim != 2 && dim != 3) || !srp || !scol || !d || !w || !sweeps || nsweeps < 1 ||
        !out || h < 0)
        return OR_EINVAL;
    const size_t xs = sizeof(double) * (size_t)n * dim;
    double* xa = (double*)malloc(xs);
    double* xb = (double*)malloc(xs);
    if (!xa || !xb) { free(xa); free(xb); return OR_ENOMEM; }
    int rc = 0;
    if (h == 0) {
        if (!x_init) { free(xa); free(xb); return OR_EINVAL; }
        memcpy(xa, x_init, xs);
        for (int32_t s = 0; s < sweeps[0] && !rc; ++s) {
            rc = or_sweep_exact(n, dim, srp, scol, d, w, xa, alpha, q, NULL, 0, xb, nthreads);
            double* t = xa; xa = xb; xb = t;
        }
        if (levels_out) *levels_out = 1;
    } else {
        or_hierarchy* H = NULL;
        rc = or_build_hierarchy(n, rp, col, NULL, NULL, seed, n_stop, 64, 64, &H);
        if (rc) { free(xa); free(xb); return rc; }
        const int32_t nl = or_hier_num_levels(H), L = nl - 1;
        if (levels_out) *levels_out = nl;
        /* level views */
        int32_t* ln = (int32_t*)calloc((size_t)nl, sizeof(int32_t));
        const int64_t** lrp = (const int64_t**)calloc((size_t)nl, sizeof(void*));
        const int32_t** lcol = (const int32_t**)calloc((size_t)nl, sizeof(void*));
        const int64_t** lc = (const int64_t**)calloc((size_t)nl, sizeof(void*));
        const int32_t** lpar = (const int32_t**)calloc((size_t)nl, sizeof(void*));
        for (int32_t l = 0; l < nl; ++l) {
            int64_t nnz; const int64_t* om; int32_t rounds;
            or_hier_level(H, l, &ln[l], &nnz, &lrp[l], &lcol[l], &om, &lc[l], &lpar[l], &rounds);
        }
        /* coarsest: box init + exact sweeps on S^L */
        double* cur = (double*)malloc(sizeof(double) * (size_t)ln[L] * dim);
        double* tmp = (double*)malloc(sizeof(double) * (size_t)ln[L] * dim);
        const int64_t* Srp = srp; const int32_t* Scol = scol; const double* Sd = d; const double* Sw = w;
        double *cd = NULL, *cw = NULL;
        if (L > 0) {
            const int64_t nnzL = lrp[L][ln[L]];
            cd = (double*)malloc(sizeof(double) * (size_t)(nnzL > 0 ? nnzL : 1));
            cw = (double*)malloc(sizeof(double) * (size_t)(nnzL > 0 ? nnzL : 1));
            or_coarse_sset(ln[L], nnzL, lrp[L], lcol[L], lc[L], dim, cd, cw);
            Srp = lrp[L]; Scol = lcol[L]; Sd = cd; Sw = cw;
        }
        {
            double dsum = 0.0;
            const int64_t nnzS = Srp[ln[L]];
            for (int64_t e = 0; e < nnzS; ++e) dsum += Sd[e];
            const double dbar = nnzS > 0 ? dsum / (double)nnzS : 1.0;
            const double box = dbar * (dim == 2 ? sqrt((double)ln[L]) : cbrt((double)ln[L]));
            or_init_box(ln[L], dim, box, seed, L, cur);
        }
        const int32_t KL = sweeps[L < nsweeps ? L : nsweeps - 1];
        for (int32_t s = 0; s < KL && !rc; ++s) {
            rc = or_sweep_exact(ln[L], dim, Srp, Scol, Sd, Sw, cur, alpha, q, NULL, 0, tmp, nthreads);
            double* t = cur; cur = tmp; tmp = t;
        }
        free(cd); free(cw); cd = cw = NULL;
        for (int32_t l = L - 1; l >= 0 && !rc; --l) {
            const int32_t nf = ln[l];
            double* xf = (double*)malloc(sizeof(double) * (size_t)nf * dim);
            double* xt = (double*)malloc(sizeof(double) * (size_t)nf * dim);
            or_prolong(nf, dim, lpar[l], cur, seed, l, xf);
            free(cur); free(tmp);
            cur = xf; tmp = xt;
            /* approximation map H = parent_{l+h'-1} o ... o parent_l */
            const int32_t hp = (h < L - l) ? h : (L - l);
            int32_t* anc = (int32_t*)malloc(sizeof(int32_t) * (size_t)nf);
            for (int32_t u = 0; u < nf; ++u) {
                int32_t a = u;
                for (int32_t t = 0; t < hp; ++t) a = lpar[l + t][a];
                anc[u] = a;
            }
            if (l == 0) {
                Srp = srp; Scol = scol; Sd = d; Sw = w;
            } else {
                const int64_t nnzl = lrp[l][nf];
                cd = (double*)malloc(sizeof(double) * (size_t)(nnzl > 0 ? nnzl : 1));
                cw = (double*)malloc(sizeof(double) * (size_t)(nnzl > 0 ? nnzl : 1));
                or_coarse_sset(nf, nnzl, lrp[l], lcol[l], lc[l], dim, cd, cw);
                Srp = lrp[l]; Scol = lcol[l]; Sd = cd; Sw = cw;
            }
            const int32_t K = sweeps[l < nsweeps ? l : nsweeps - 1];
            for (int32_t s = 0; s < K && !rc; ++s) {
                rc = or_sweep_approx(nf, dim, Srp, Scol, Sd, Sw, cur, alpha, q, lpar[l], anc,
                                     ln[l + hp], NULL, 0, tmp, nthreads);
                double* t = cur; cur = tmp; tmp = t;
            }
            free(anc); free(cd); free(cw); cd = cw = NULL;
        }
        memcpy(xa, cur, xs);
        free(cur); free(tmp);
        free(ln); free(lrp); free(lcol); free(lc); free(lpar);
        or_hier_free(H);
    }
    memcpy(out, xa, xs);
    if (!rc && energy_out) rc = or_energy(n, dim, srp, scol, d, w, xa, alpha, q, energy_out, nthreads);
    free(xa); free(xb);
    return rc;
}
