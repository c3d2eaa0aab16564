/* ORACLE (test infrastructure only) — the paper's optimizer schedule and the
 * dynamic update mode, FP64, on top of the sweeps of sweep.c.
 *
 * "we set alpha to one initially and gradually reduce it by
 * alpha := 0.3 alpha until alpha_min = 0.008 is reached."
 * "We call a single update step of the coordinates of all vertices
 * ... an iteration.  Multiple iterations with the same value of alpha are
 * called round ... We perform at most a iterations with the same value of
 * alpha in one round.  Then we reduce alpha ... If the relative change
 * ||x^{l+1} - x^l|| / ||x^l|| in the layout is smaller than some threshold
 * epsilon, we directly reduce the value of alpha and continue with the next
 * round."  P:335-336: a = 2, alpha_min = 0.008, and at alpha_min "we iterate
 * until the relative error ... is smaller than 0.0001".
 * P:424-427 (dynamic update): "we start directly at the penalty level
 * alpha = 0.008 and only update coordinates on the finest level of the
 * hierarchy.  We compute the graph hierarchy as before but stop the coarsening
 * process after the computation of h levels.  Coordinates of the vertices on
 * the approximation level are set to the middle point of the vertices in the
 * corresponding cluster initially."
 * Readings: R1 the schedule restarts at alpha0 on every level;
 * R2 alpha is clamped to alpha_min (1, 0.3, 0.09, 0.027, 0.0081, 0.008);
 * R3 max_final_iters caps the alpha_min phase (not in the paper);
 * R4 the coarsest level starts from the box init (Q14). */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "mm_oracle.h"

/* one level under the schedule; x is updated in place (tmp = scratch) */
static int run_level(int32_t n, int dim, const int64_t* srp, const int32_t* scol, const double* d, const double* w,
                     double q, const int32_t* parent, const int32_t* anc, int32_t k, const or_schedule* sch,
                     int start_at_min, double** x, double** tmp, int32_t* sweeps, int nthreads) {
    double alpha = start_at_min ? sch->alpha_min : sch->alpha0;
    int rc = 0;
    *sweeps = 0;
    for (;;) {
        const int final = alpha <= sch->alpha_min;
        const int32_t max_it = final ? sch->max_final_iters : sch->a;
        for (int32_t it = 0; it < max_it; ++it) {
            if (anc)
                rc = or_sweep_approx(n, dim, srp, scol, d, w, *x, alpha, q, parent, anc, k, NULL, 0, *tmp, nthreads);
            else
                rc = or_sweep_exact(n, dim, srp, scol, d, w, *x, alpha, q, NULL, 0, *tmp, nthreads);
            if (rc) return rc;
            const double rel = or_relative_change((int64_t)n * dim, *x, *tmp);
            double* t = *x; *x = *tmp; *tmp = t;
            *sweeps += 1;
            if (rel < sch->eps) break;
        }
        if (final) break;
        alpha = alpha * sch->factor;
        if (alpha < sch->alpha_min) alpha = sch->alpha_min;
    }
    return 0;
}

static double root_dim(double c, int dim) { return dim == 2 ? sqrt(c) : cbrt(c); }

int or_layout_schedule(int32_t n, int dim, const int64_t* rp, const int32_t* col,
                       const int64_t* srp, const int32_t* scol, const double* d, const double* w,
                       double q, int h, const or_schedule* sch, uint64_t seed, int32_t n_stop, int flags,
                       const double* x_init, double* out, double energy_out[3], int32_t* levels_out,
                       int32_t* sweeps_out, int nthreads) {
    if (n <= 0 || (dim != 2 && dim != 3) || !srp || !scol || !d || !w || !sch || !out || h < 0 ||
        sch->a < 1 || sch->max_final_iters < 1 || !(sch->alpha_min > 0.0) || !(sch->factor > 0.0 && sch->factor < 1.0))
        return OR_EINVAL;
    const int multilevel = flags & 1, dynamic = flags & 2;
    if ((!multilevel || dynamic) && !x_init) return OR_EINVAL;
    const size_t xs = sizeof(double) * (size_t)n * dim;
    double* xa = (double*)malloc(xs);
    double* xb = (double*)malloc(xs);
    if (!xa || !xb) { free(xa); free(xb); return OR_ENOMEM; }
    int rc = 0;
    if (sweeps_out) memset(sweeps_out, 0, sizeof(int32_t) * 64);
    if (!multilevel && !dynamic) {
        memcpy(xa, x_init, xs);
        rc = run_level(n, dim, srp, scol, d, w, q, NULL, NULL, 0, sch, 0, &xa, &xb, sweeps_out ? &sweeps_out[0] : &(int32_t){0}, nthreads);
        if (levels_out) *levels_out = 1;
    } else {
        or_hierarchy* H = NULL;
        /* dynamic: stop the coarsening after h levels (the approximation level) */
        const int32_t max_levels = dynamic ? (h + 1) : 64;
        if (flags & 4)
            rc = or_build_hierarchy_sclap_mode(n, rp, col, NULL, NULL, seed, dynamic ? 1 : n_stop, max_levels, 3, 20.0,
                                               2.0, (flags & 16) ? 1 : 0, &H);
        else
            rc = or_build_hierarchy(n, rp, col, NULL, NULL, seed, dynamic ? 1 : n_stop, max_levels, 64, &H);
        if (rc) { free(xa); free(xb); return rc; }
        const int32_t nl = or_hier_num_levels(H), L = nl - 1;
        if (levels_out) *levels_out = nl;
        int32_t* ln = (int32_t*)calloc((size_t)nl, sizeof(int32_t));
        const int64_t** lrp = (const int64_t**)calloc((size_t)nl, sizeof(void*));
        const int32_t** lcol = (const int32_t**)calloc((size_t)nl, sizeof(void*));
        const int64_t** lc = (const int64_t**)calloc((size_t)nl, sizeof(void*));
        const int32_t** lpar = (const int32_t**)calloc((size_t)nl, sizeof(void*));
        for (int32_t l = 0; l < nl; ++l) {
            int64_t nnz; const int64_t* om; int32_t rounds;
            or_hier_level(H, l, &ln[l], &nnz, &lrp[l], &lcol[l], &om, &lc[l], &lpar[l], &rounds);
        }
        int32_t* anc = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
        if (dynamic) {
            /* finest level only, warm start at alpha_min */
            memcpy(xa, x_init, xs);
            const int32_t hp = (h < L) ? h : L;
            if (hp > 0) {
                for (int32_t u = 0; u < n; ++u) {
                    int32_t a = u;
                    for (int32_t t = 0; t < hp; ++t) a = lpar[t][a];
                    anc[u] = a;
                }
            }
            rc = run_level(n, dim, srp, scol, d, w, q, hp > 0 ? lpar[0] : NULL, hp > 0 ? anc : NULL,
                           hp > 0 ? ln[hp] : 0, sch, 1, &xa, &xb, sweeps_out ? &sweeps_out[0] : &(int32_t){0}, nthreads);
        } else {
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
                or_init_box(ln[L], dim, dbar * root_dim((double)ln[L], dim), seed, L, cur);
            }
            int32_t sw = 0;
            rc = run_level(ln[L], dim, Srp, Scol, Sd, Sw, q, NULL, NULL, 0, sch, 0, &cur, &tmp, &sw, nthreads);
            if (sweeps_out) sweeps_out[L] = sw;
            free(cd); free(cw); cd = cw = NULL;
            for (int32_t l = L - 1; l >= 0 && !rc; --l) {
                const int32_t nf = ln[l];
                double* xf = (double*)malloc(sizeof(double) * (size_t)nf * dim);
                double* xt = (double*)malloc(sizeof(double) * (size_t)nf * dim);
                if (flags & 8) or_prolong_disc(nf, dim, lpar[l], cur, lc[l + 1], seed, l, xf);
                else or_prolong(nf, dim, lpar[l], cur, seed, l, xf);
                free(cur); free(tmp);
                cur = xf; tmp = xt;
                const int32_t hp = (h < L - l) ? h : (L - l);
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
                sw = 0;
                rc = run_level(nf, dim, Srp, Scol, Sd, Sw, q, hp > 0 ? lpar[l] : NULL, hp > 0 ? anc : NULL,
                               hp > 0 ? ln[l + hp] : 0, sch, 0, &cur, &tmp, &sw, nthreads);
                if (sweeps_out) sweeps_out[l] = sw;
                free(cd); free(cw); cd = cw = NULL;
            }
            memcpy(xa, cur, xs);
            free(cur); free(tmp);
        }
        free(anc);
        free(ln); free(lrp); free(lcol); free(lc); free(lpar);
        or_hier_free(H);
    }
    memcpy(out, xa, xs);
    /* energy at alpha_min, the paper's final penalty level */
    if (!rc && energy_out) rc = or_energy(n, dim, srp, scol, d, w, xa, sch->alpha_min, q, energy_out, nthreads);
    free(xa); free(xb);
    return rc;
}
