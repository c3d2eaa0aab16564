/* MulMent ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-precision-free (IEEE FP64, no fast-math) CPU
 * implementation of the maxent-stress hot path of Meyerhenke, Nöllenburg,
 * Schulz, "Drawing large graphs by multilevel maxent-stress optimization"
 * (arXiv 1506.04383).  Citations "P:n" are lines of /root/reference/PAPER.md;
 * "Qn" are the readings listed in DESIGN.md §3.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header,
 * table or constant generator with the CUDA path in paper_1506_04383_b200/.
 *
 * Conventions: graphs and S sets are CSR (row_ptr int64[n+1], col int32);
 * coordinates are double[n*dim] row-major; dim is 2 or 3.  Every function
 * returns 0 on success and a negative code on error:
 *   OR_EINVAL  = -1  bad argument
 *   OR_ERHO    = -2  rho_i <= 0 (vertex with an empty / zero-weight S row)
 *   OR_ECOINC  = -3  coincident non-S pair in the energy (S:333 reading)
 *   OR_ENOMEM  = -4
 * The optional `nthreads` runs independent rows under OpenMP; each row's
 * summation order is fixed, so results are bitwise identical for any
 * thread count. */
#ifndef MM_ORACLE_H
#define MM_ORACLE_H
#include <stdint.h>

#define OR_EINVAL (-1)
#define OR_ERHO (-2)
#define OR_ECOINC (-3)
#define OR_ENOMEM (-4)

/* ---- counter-based RNG (Q18): SplitMix64 output function, oracle's own copy */
uint64_t or_mix64(uint64_t z);
/* U in [0,1): top 24 bits of key / 2^24 (exactly representable in float) */
double or_uniform24(uint64_t key);
uint64_t or_key_vertex(uint64_t seed, uint64_t tag, uint64_t level, uint64_t vertex, int dim, int comp);

/* ---- Eq.(2): one synchronous (Jacobi) sweep, exact entropy term.
 * rows: subset of target vertices (NULL = all n, in order); out: nrows*dim. */
int or_sweep_exact(int32_t n, int dim, const int64_t* srp, const int32_t* scol,
                   const double* d, const double* w, const double* x,
                   double alpha, double q, const int32_t* rows, int32_t nrows,
                   double* out, int nthreads);

/* ---- coarse representatives for Eq.(3), P:274, P:283-284 (Q10-Q12):
 * nu[v'] = #{u : H(u) = v'}, xc[v'] = unweighted mean of x_u over H(u)=v'. */
int or_centroids(int32_t n, int dim, const double* x, const int32_t* anc, int32_t k,
                 double* xc, int64_t* nu);

/* ---- Eq.(3): one sweep with the approximated entropy term.
 * parent: level-(l+1) ids (sibling term, one level up); anc: level-(l+h')
 * ids (representative term); k = number of approximation-level vertices. */
int or_sweep_approx(int32_t n, int dim, const int64_t* srp, const int32_t* scol,
                    const double* d, const double* w, const double* x,
                    double alpha, double q, const int32_t* parent, const int32_t* anc, int32_t k,
                    const int32_t* rows, int32_t nrows, double* out, int nthreads);

/* ---- Eq.(1), P:163-171 with Q3/Q4: out[0] = stress = 1/2 sum_i sum_{j in S_i}
 * w(|x_i-x_j| - d)^2, out[1] = entropy = 1/2 sum_i sum_{j notin S_i, j != i} phi_q,
 * phi_0(r) = -ln r, phi_q(r) = r^-q / q; out[2] = stress + alpha * entropy. */
int or_energy(int32_t n, int dim, const int64_t* srp, const int32_t* scol,
              const double* d, const double* w, const double* x,
              double alpha, double q, double out[3], int nthreads);

/* ---- relative change ||x' - x|| / ||x|| */
double or_relative_change(int64_t len, const double* x_old, const double* x_new);

/* ---- hierarchy (P:193-235 contraction; matching per Q16/Q17) */
typedef struct or_hierarchy or_hierarchy;
int or_build_hierarchy(int32_t n, const int64_t* rp, const int32_t* col,
                       const int64_t* omega /*NULL = unit*/, const int64_t* c /*NULL = unit*/,
                       uint64_t seed, int32_t n_stop, int32_t max_levels, int32_t max_rounds,
                       or_hierarchy** out);
/* SCLaP hierarchy (reading R6 in sclap.c): rounds = l, f0 = 20, b = 2 */
int or_build_hierarchy_sclap(int32_t n, const int64_t* rp, const int32_t* col, const int64_t* omega,
                             const int64_t* c, uint64_t seed, int32_t n_stop, int32_t max_levels, int32_t rounds,
                             double f0, double b, or_hierarchy** out);
int or_build_hierarchy_sclap_mode(int32_t n, const int64_t* rp, const int32_t* col, const int64_t* omega,
                                  const int64_t* c, uint64_t seed, int32_t n_stop, int32_t max_levels,
                                  int32_t rounds, double f0, double b, int seq, or_hierarchy** out);
/* the paper's sequential label propagation (reading R6s in sclap.c) */
int or_sclap_labels_seq(int32_t n, const int64_t* rp, const int32_t* col, const int64_t* omega, const int64_t* c,
                        int64_t U, int32_t rounds, uint64_t seed, int32_t level, int32_t* lab);
int or_sclap_labels(int32_t n, const int64_t* rp, const int32_t* col, const int64_t* omega, const int64_t* c,
                    int64_t U, int32_t rounds, uint64_t seed, int32_t level, int32_t* lab);
int32_t or_hier_num_levels(const or_hierarchy* h);
/* level l graph sizes; arrays are owned by the hierarchy */
int or_hier_level(const or_hierarchy* h, int32_t l, int32_t* n, int64_t* nnz,
                  const int64_t** rp, const int32_t** col, const int64_t** omega,
                  const int64_t** c, const int32_t** parent /*NULL at the coarsest*/,
                  int32_t* rounds);
void or_hier_free(or_hierarchy* h);

/* ---- coarse S^l (Q7): S = E^l, d_uv = c_u^(1/dim) + c_v^(1/dim), w = d^-2 */
int or_coarse_sset(int32_t n, int64_t nnz, const int64_t* rp, const int32_t* col,
                   const int64_t* c, int dim, double* d, double* w);

/* ---- initial layout of the coarsest level (Q14) */
int or_init_box(int32_t n, int dim, double box, uint64_t seed, int32_t level, double* x);
/* ---- prolongation (Q15; variant of P:240-242): x_u = x_{P(u)} + 1e-3 (2U - 1) */
int or_prolong(int32_t n_fine, int dim, const int32_t* parent, const double* xc,
               uint64_t seed, int32_t level, double* x);

/* ---- multilevel driver (P:195-197, P:240-257 with fixed alpha, Q13-Q15).
 * h = 0: single level, x_init required, `sweeps[0]` exact sweeps.
 * h > 0: hierarchy, box init at the coarsest level L, sweeps[l] per level
 * (sweeps has max_levels entries; level l uses sweeps[min(l, len-1)]).
 * out: x^0 (n*dim); energy_out: or_energy at the finest level; levels_out. */
int or_layout(int32_t n, int dim, const int64_t* rp, const int32_t* col,
              const int64_t* srp, const int32_t* scol, const double* d, const double* w,
              double alpha, double q, int h, const int32_t* sweeps, int32_t nsweeps,
              uint64_t seed, int32_t n_stop, const double* x_init, double* out,
              double energy_out[3], int32_t* levels_out, int nthreads);

/* ---- the paper's optimizer schedule, reading R1-R4
 * of DESIGN.md §3: per level, alpha starts at alpha0; a round runs at most
 * `a` Jacobi sweeps at one alpha and ends early when the relative change
 * |x' - x| / |x| < eps; then alpha <- max(factor * alpha, alpha_min).  At
 * alpha_min, sweeps continue until the relative change < eps or
 * max_final_iters sweeps.  flags bit 0: multilevel (hierarchy + prolongation;
 * exact Eq.(2) everywhere when h = 0, Eq.(3) with h' = min(h, L - l) otherwise),
 * else one level from x_init.  flags bit 1: dynamic update: start
 * at alpha_min on the finest level only, from x_init, with the hierarchy built
 * to at most h levels above the finest (the approximation level).
 * flags bit 2: SCLaP hierarchy (R6; lp_rounds = 3, f = 20, b = 2) instead of the
 * matching; bit 3: the paper's disc prolongation (R7) instead of Q15;
 * bit 4 (with bit 2): SCLaP by the paper's sequential label propagation (R6s). 
 * sweeps_out[l] = sweeps performed at level l (nullable, 64 entries). */
typedef struct {
    double alpha0, alpha_min, factor, eps;
    int32_t a, max_final_iters;
} or_schedule;
int or_layout_schedule(int32_t n, int dim, const int64_t* rp, const int32_t* col,
                       const int64_t* srp, const int32_t* scol, const double* d, const double* w,
                       double q, int h, const or_schedule* sch, uint64_t seed, int32_t n_stop, int flags,
                       const double* x_init, double* out, double energy_out[3], int32_t* levels_out,
                       int32_t* sweeps_out, int nthreads);

/* ---- full stress F(x) with graph distances and w = d^-2, and the optimal
 * scale s* = argmin_s F(s x) (reading R5): out = {F(1), s*, F(s*), pairs} */
int or_full_stress(int32_t n, const int64_t* rp, const int32_t* col, int dim, const double* x, double out[4],
                   int nthreads);

#define OR_TAG_INIT 0x494e4954ULL   /* "INIT" */
#define OR_TAG_JITTER 0x4a495454ULL /* "JITT" */
#define OR_TAG_MATCH 0x4d415443ULL  /* "MATC" */
#define OR_TAG_DISC 0x44495343ULL   /* "DISC" */
int or_prolong_disc(int32_t n_fine, int dim, const int32_t* parent, const double* xc, const int64_t* c_coarse,
                    uint64_t seed, int32_t level, double* x);

#endif
