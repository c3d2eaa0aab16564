/* mm.h — C-ABI of the B200-native MulMent hot path (libmm_b200.so).
 *
 * Meyerhenke, Nöllenburg, Schulz, "Drawing large graphs by multilevel
 * maxent-stress optimization", arXiv 1506.04383.  Citations "P:n" are lines of
 * the paper's LaTeX source; "Qn" are the readings of DESIGN.md §3.
 *
 * What the library computes (one GPU, hand-written sm_100a CUDA kernels):
 *   - mm_sweep: one synchronous (Jacobi) sweep of the local update Eq.(2)
 *     (P:176-181), or of Eq.(3) when a coarse-level map is given;
 *   - mm_energy: the maxent-stress energy Eq.(1);
 *   - mm_build_hierarchy: the matching-based multilevel hierarchy with the
 *     contraction of P:225-232 (matching per Q16, stop rule Q17);
 *   - mm_layout: the multilevel driver (P:195-257 with fixed alpha).
 *
 * Conventions (all entry points):
 *   - POINTERS are DEVICE pointers unless the comment says "host".  The caller
 *     owns every input and output buffer; the library owns only what it
 *     returns through an opaque handle (mm_hierarchy) and its internal scratch.
 *   - COORDINATES: dim 2 -> float[2n] interleaved (x0,y0,x1,y1,...), 8-byte
 *     aligned; dim 3 -> float[4n] (x,y,z,pad per vertex), 16-byte aligned; the
 *     pad lane is ignored on input and written 0 on output.
 *   - CSR: row_ptr int64[n+1] (row_ptr[0] = 0), col int32[nnz]; rows need not
 *     be sorted; S rows must not contain i itself or duplicates.
 *   - STREAMS: every call enqueues on `stream` (a cudaStream_t; NULL = legacy
 *     default stream).  Calls marked "async" do not synchronise the host;
 *     calls marked "syncs" synchronise `stream` before returning.
 *   - THREADS: every entry point may be called from several host threads at
 *     once.  mm_layout, mm_layout_schedule and mm_build_hierarchy(_sclap) use
 *     device-resident grid-barrier / schedule state, so the library runs them
 *     one at a time per process (a lock held from their first launch to their
 *     final stream synchronisation); the other calls are not serialised.
 *   - ERRORS: argument checks are synchronous and happen before any launch;
 *     on error nothing is enqueued and mm_last_error() holds a thread-local
 *     message.  Device-detected problems (non-finite coordinates) are written
 *     to mm_sweep_stats.flags and reported as MM_ERR_NONFINITE by the next
 *     syncing call that reads them.  No C++ exception crosses this ABI.
 *   - There is no CPU fallback: a missing or unusable GPU is MM_ERR_CUDA.
 */
#ifndef MM_H
#define MM_H
#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define MM_API __attribute__((visibility("default")))
#else
#define MM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef void* mm_stream_t; /* a cudaStream_t */

typedef enum {
    MM_OK = 0,
    MM_ERR_INVALID_ARGUMENT = -1, /* null pointer, bad size, aliasing, bad dim */
    MM_ERR_INVALID_INPUT = -2,    /* bad CSR / rho_i <= 0 detected by validation */
    MM_ERR_NONFINITE = -3,        /* non-finite coordinate produced or given; coincident non-S pair in mm_energy */
    MM_ERR_OUT_OF_MEMORY = -4,
    MM_ERR_CUDA = -5,             /* a CUDA runtime error (no device, launch failure, ...) */
    MM_ERR_UNSUPPORTED = -6       /* dim not 2|3, q < 0 */
} mm_status;

/* Graph G = (V, E, c, omega), symmetric CSR of E. */
typedef struct {
    int32_t n;
    int64_t nnz;              /* = 2|E| */
    const int64_t* row_ptr;   /* device int64[n+1] */
    const int32_t* col;       /* device int32[nnz] */
    const int32_t* omega;     /* device int32[nnz] edge weights, or NULL = unit */
} mm_graph;

/* Stress pair set S ⊇ E (P:163 footnote): per-vertex rows S_i with target
 * distance d_ij > 0 and weight w_ij >= 0 (w = d^-2 by default).
 * Row i must have rho_i = sum_j w_ij > 0. */
typedef struct {
    int32_t n;
    int64_t nnz;
    const int64_t* row_ptr;   /* device int64[n+1] */
    const int32_t* col;       /* device int32[nnz] */
    const float* d;           /* device float[nnz] */
    const float* w;           /* device float[nnz] */
} mm_sset;

/* Coarse-level map for Eq.(3): parent P (one level up, defines
 * the same-cluster sum) and ancestor H (level l+h', defines the coarse
 * representatives, k of them; H must be surjective onto 0..k-1). */
typedef struct {
    int32_t k;
    const int32_t* parent;    /* device int32[n] */
    const int32_t* ancestor;  /* device int32[n], values in [0,k) */
} mm_approx;

/* Device-side per-sweep statistics (written by mm_sweep when non-NULL). */
typedef struct {
    double dx2;       /* sum_i |x'_i - x_i|^2 */
    double x2;        /* sum_i |x_i|^2 ; relative change = sqrt(dx2 / x2) */
    double stress;    /* 1/2 sum_i sum_{j in S_i} w (|x_i - x_j| - d)^2 at the INPUT x */
    int32_t flags;    /* bit 0: non-finite output coordinate */
    int32_t pad;
} mm_sweep_stats;

typedef struct mm_hierarchy mm_hierarchy;

/* Host view of one hierarchy level; array members are device pointers owned
 * by the hierarchy and valid until mm_hierarchy_free. */
typedef struct {
    int32_t n;
    int64_t nnz;
    const int64_t* row_ptr;
    const int32_t* col;
    const int32_t* omega;   /* coarse edge weights (sum of crossing weights) */
    const int32_t* c;       /* node weights (sum of member weights) */
    const int32_t* parent;  /* int32[n] -> level l+1 ids; NULL at the coarsest level */
    const float* d;         /* coarse S^l = E^l distances (Q7); NULL at level 0 */
    const float* w;         /* coarse weights d^-2; NULL at level 0 */
    int32_t rounds;         /* matching rounds used to build level l+1 */
} mm_level_view;

/* Layout report (host). */
#define MM_MAX_LEVELS 64
typedef struct {
    int32_t levels;
    int32_t n_level[MM_MAX_LEVELS];
    int32_t k_level[MM_MAX_LEVELS];     /* approximation-level size used at level l (0 = exact) */
    double stress, entropy, energy;     /* mm_energy of the final finest layout (Eq.(1)) */
    double rel_change;                  /* relative change of the last finest-level sweep */
    int64_t vertex_updates;             /* sum_l n_l * K_l */
    int64_t pair_interactions;          /* repulsion pairs evaluated (DESIGN.md §5 convention) */
    int64_t coincident_pairs;           /* non-S ordered pairs at distance exactly 0 in the final
                                           layout; they are left out of `entropy` (ln 0 undefined) */
    int32_t sweeps_level[MM_MAX_LEVELS]; /* Jacobi sweeps performed at level l */
} mm_layout_report;

/* The paper's optimizer schedule: alpha0 = 1,
 * factor = 0.3, alpha_min = 0.008, a = 2 iterations per round, eps = 1e-4;
 * max_final_iters caps the alpha_min phase (not in the paper). */
typedef struct {
    double alpha0, alpha_min, factor, eps;
    int32_t a, max_final_iters;
} mm_schedule;
#define MM_LAYOUT_MULTILEVEL 1 /* hierarchy + prolongation; h = 0: exact Eq.(2) on every level */
#define MM_LAYOUT_DYNAMIC 2    /* dynamic update: finest level only, from x_init, at alpha_min */
#define MM_LAYOUT_SCLAP 4      /* SCLaP hierarchy (reading R6; l = 3, f = 20, b = 2) instead of matching */
#define MM_LAYOUT_DISC_PROLONG 8 /* the paper's disc prolongation (R7) instead of Q15's jitter */

/* ------------------------------------------------------------------ API */

/* Human-readable status / thread-local detail of the last error. */
MM_API const char* mm_status_string(mm_status s);
MM_API const char* mm_last_error(void);
/* Library version string, e.g. "mm_b200 0.1 sm_100a". */
MM_API const char* mm_version(void);

/* Optional allocator hook for the library's scratch and hierarchy storage.
 * alloc(bytes, stream, ctx) must return device memory usable on `stream`;
 * free_(ptr, stream, ctx) releases it.  NULL, NULL restores the default
 * (cudaMallocAsync / cudaFreeAsync, stream-ordered). */
MM_API mm_status mm_set_allocator(void* (*alloc)(size_t, mm_stream_t, void*),
                           void (*free_)(void*, mm_stream_t, void*), void* ctx);

/* Validate an S set on the device (syncs): row_ptr monotone within [0, nnz],
 * 0 <= col < n, no self entry, d > 0 finite, w >= 0 finite, rho_i > 0 for every
 * row (P:106 connected graphs; reading Q22).  Returns MM_ERR_INVALID_INPUT with
 * the first offending row and the reasons in mm_last_error().  Duplicate
 * entries are not detected.  The sweep entry points do not validate (cost). */
MM_API mm_status mm_validate_sset(const mm_sset* S, mm_stream_t stream);

/* Scratch bytes mm_sweep needs for n vertices (host out). ap = NULL: exact. */
MM_API mm_status mm_sweep_workspace(int32_t n, int dim, const mm_approx* ap, size_t* bytes);

/* One Jacobi sweep, Eq.(2) (ap = NULL: exact entropy term over all j notin S_i,
 * P:178) or Eq.(3) (ap != NULL: same-cluster exact terms over P, nu-weighted
 * representatives over H excluding H(i), minus the S_i terms).
 * q >= 0 is the repulsion exponent: r(i,j) = (x_i - x_j)/|x_i - x_j|^(q+2)
 * (q = 0 is the paper's r-value).  The representatives are the
 * unweighted means of x_in over each H class (Q11/Q12).
 * x_out must not alias x_in.  ws/ws_bytes: caller scratch of at least
 * mm_sweep_workspace() bytes, 256-B aligned (else MM_ERR_INVALID_ARGUMENT),
 * or NULL/0 to let the library allocate it stream-ordered.  stats (device, nullable) receives mm_sweep_stats.  async.
 * Eq.(3) evaluation order (results equal up to FP32 rounding, DESIGN.md
 * Q26-Q28): targets and representatives are visited in spatial order and
 * representatives grouped by mass; tiles far from a warp's targets drop the
 * FP64 lo part of the centroids.  Environment (read once per process, tests
 * and experiments): MM_FAR_TILES=0 keeps hi/lo everywhere, MM_FAR_PAIRS /
 * MM_REORDER_PAIRS set the n k thresholds of the far-tile path (1e9) and of
 * per-sweep re-sorting (1e11). */
MM_API mm_status mm_sweep(const mm_sset* S, int dim, float alpha, float q, const mm_approx* ap,
                   const float* x_in, float* x_out, mm_sweep_stats* stats,
                   void* ws, size_t ws_bytes, mm_stream_t stream);

/* K Jacobi sweeps ("a single update step of the coordinates of all
 * vertices using Eq.(2)" per iteration; "the current iteration uses the
 * coordinates that have been computed in the previous iteration"), each one
 * what mm_sweep computes, from x_in to x_out (must not alias).  With ap the
 * representatives are refreshed before every sweep (Q12).  A level that
 * qualifies (n <= 32,768 for Eq.(3), <= 4,096 exact; MM_SMALL_N caps it)
 * runs all K sweeps in the persistent small-level kernel, as mm_layout does;
 * otherwise the K sweeps are one CUDA graph of the tiled kernels.
 * stats (device, nullable) receives the LAST sweep's mm_sweep_stats.  K = 0
 * copies.  Returns MM_ERR_NONFINITE if a non-finite coordinate appeared.
 * syncs `stream` (and serialises with mm_layout like it). */
MM_API mm_status mm_sweeps(const mm_sset* S, int dim, float alpha, float q, const mm_approx* ap,
                           const float* x_in, float* x_out, int32_t K, mm_sweep_stats* stats, mm_stream_t stream);

/* Maxent-stress energy Eq.(1) in the S form with readings Q3/Q4:
 * out[0] = stress = 1/2 sum_i sum_{j in S_i} w (|x_i-x_j| - d)^2
 * out[1] = entropy = 1/2 sum_i sum_{j notin S_i, j != i} phi_q(|x_i - x_j|),
 *          phi_0(r) = -ln r, phi_q(r) = r^-q / q
 * out[2] = stress + alpha * entropy.  out is HOST double[3].
 * FP32 per pair, FP64 accumulation, fixed summation order (deterministic):
 * the per-CTA FP64 partials are copied to the host and summed there in CTA
 * order (a few thousand doubles; this is part of the sync, not a fallback).
 * A coincident non-S pair returns MM_ERR_NONFINITE.  syncs. */
MM_API mm_status mm_energy(const mm_sset* S, int dim, double alpha, double q, const float* x,
                    double* out, mm_stream_t stream);

/* Build the hierarchy: handshake heavy-edge matching by rating
 * omega_uv / (c_u c_v) (exact int64 compare; ties: higher SplitMix64 hash of
 * (seed, level, round, min, max), then lower id; <= max_rounds rounds), leader
 * ranking, contraction, coarse S^l (Q7, needs dim), until
 * n_l <= n_stop or a contraction would keep > 90% of the vertices or
 * max_levels levels exist (Q17).  c: device int32[n] node weights or NULL =
 * unit.  Integer results are bit-identical to the oracle's.  Syncs once per
 * level (to read n_{l+1}).  *out is released with mm_hierarchy_free. */
MM_API mm_status mm_build_hierarchy(const mm_graph* g, const int32_t* c, int dim, uint64_t seed,
                             int32_t n_stop, int32_t max_levels, int32_t max_rounds,
                             mm_hierarchy** out, mm_stream_t stream);
/* The paper's SCLaP hierarchy in the synchronous reading R6 of
 * level h = 1, 2, ... clusters with size bound U = max(max c,
 * min(b^h, n/f)) in lp_rounds label-propagation rounds (f0 = 20, b = 2 in the
 * paper; f <- 0.7 f after a contraction that is not 10% smaller), then
 * contracts (coarse id = rank of the distinct labels).  Integer-exact: bit-
 * identical to the oracle.  Stops at n_stop, max_levels or 10 ineffective
 * decays.  Syncs a few times per round. */
MM_API mm_status mm_build_hierarchy_sclap(const mm_graph* g, const int32_t* c, int dim, uint64_t seed,
                                          int32_t n_stop, int32_t max_levels, int32_t lp_rounds, double f0, double b,
                                          mm_hierarchy** out, mm_stream_t stream);
MM_API int32_t mm_hierarchy_num_levels(const mm_hierarchy* h);
MM_API mm_status mm_hierarchy_level(const mm_hierarchy* h, int32_t level, mm_level_view* out /*host*/);
MM_API void mm_hierarchy_free(mm_hierarchy* h);
/* Copy level `level` of the hierarchy into HOST arrays (any may be NULL to
 * skip): row_ptr int64[n+1], col int32[nnz], omega int32[nnz], c int32[n],
 * parent int32[n] (not at the coarsest level), d/w float[nnz] (not at level 0).
 * syncs `stream`. */
MM_API mm_status mm_hierarchy_copy_level(const mm_hierarchy* h, int32_t level, int64_t* row_ptr, int32_t* col,
                                         int32_t* omega, int32_t* c, int32_t* parent, float* d, float* w,
                                         mm_stream_t stream);

/* Prolongation of one level (the step mm_layout runs between levels):
 * x[u] = xc[parent[u]] + delta_u for u < n_fine.
 *   c_coarse == NULL: reading Q15 (BASELINE.json configs[2]): delta_u,k =
 *     1e-3 (2 U - 1), U = the counter RNG of (seed, jitter tag, level, u, k).
 *   c_coarse != NULL: the paper's disc (reading R7): angle 2 pi U0,
 *     distance c(parent)^(1/dim) U1 (dim 3: direction from z = 2 U2 - 1).
 * parent: device int32[n_fine] (ids < the coarse level's size, not checked);
 * xc: device coarse coordinates; c_coarse: device int32 coarse node weights;
 * x: device output [n_fine] in the coordinate layout (must not alias xc).
 * level = the FINE level's index (the RNG key).  async. */
MM_API mm_status mm_prolong(int32_t n_fine, int dim, const int32_t* parent, const float* xc,
                            const int32_t* c_coarse, uint64_t seed, int32_t level, float* x, mm_stream_t stream);

/* Multilevel layout.  h = 0: single level, x_init (device, required) is
 * iterated sweeps[0] exact sweeps (Eq.(2)).  h > 0: hierarchy (n_stop, seed),
 * box init of the coarsest level L (Q14), sweeps[min(L, nsweeps-1)] exact
 * sweeps there, then for l = L-1..0: prolongation (Q15) and
 * sweeps[min(l, nsweeps-1)] Eq.(3) sweeps with h' = min(h, L-l) (Q13); coarse
 * levels use S^l (Q7), level 0 uses S.  sweeps: HOST int32[nsweeps].
 * x_out: device, the finest layout.  rep: HOST report (nullable); its energy
 * leaves out pairs at distance exactly 0 and counts them (coincident_pairs),
 * whereas mm_energy rejects them.  syncs. */
MM_API mm_status mm_layout(const mm_graph* g, const mm_sset* S, int dim, float alpha, float q, int h,
                    const int32_t* sweeps, int32_t nsweeps, uint64_t seed, int32_t n_stop,
                    const float* x_init, float* x_out, mm_layout_report* rep, mm_stream_t stream);

/* Layout with the paper's schedule instead of fixed alpha / sweep counts.
 * Per optimized level (R1: the schedule restarts on every level): rounds at
 * alpha = alpha0, factor*alpha, ... clamped to alpha_min (R2), each of at most
 * `a` sweeps and cut short once the relative change |x'-x|/|x| < eps; at
 * alpha_min sweeps continue until the relative change < eps or max_final_iters
 * (R3).  flags = 0: one level from x_init (exact Eq.(2)).  MM_LAYOUT_MULTILEVEL:
 * hierarchy (n_stop, seed), box init of the coarsest level, prolongation, exact
 * sweeps when h = 0, else Eq.(3) with h' = min(h, L-l).  MM_LAYOUT_DYNAMIC: the
 * paper's update algorithm — hierarchy stopped after h levels, only the finest
 * level is optimized, from x_init (device, required), starting at alpha_min;
 * the representatives are the cluster midpoints of the current layout.
 * The report's energy is Eq.(1) at alpha_min (the paper's final penalty level,
 * P:324); rep->sweeps_level holds the sweeps run per level.  Syncs (once per
 * sweep: each schedule decision reads the sweep's relative change). */
MM_API mm_status mm_layout_schedule(const mm_graph* g, const mm_sset* S, int dim, float q, int h,
                                    const mm_schedule* sch, uint64_t seed, int32_t n_stop, int32_t flags,
                                    const float* x_init, float* x_out, mm_layout_report* rep, mm_stream_t stream);

/* Full stress, the paper's quality metric:
 * F(x) = sum over unordered pairs u<v of w_uv (|x_u - x_v| - d_uv)^2 with d_uv
 * the shortest-path (hop) distance in g and w = d^-2, and the optimal scale
 * s* = argmin_s F(s x) = A/B (A = sum w d l, B = sum w l^2; reading R5).
 * out: HOST double[4] = {F(x), s*, F(s* x), number of pairs}.  One BFS per
 * source (n BFS traversals, O(n m) work); n <= 1,638,400 (visited bitset in
 * shared memory).  FP64 sums; their order follows the BFS claim order, so the
 * last bits may vary between runs.  syncs. */
MM_API mm_status mm_full_stress(const mm_graph* g, int dim, const float* x, double* out, mm_stream_t stream);

/* ------------------------------------------------------------------ instrumentation */
/* Total kernels launched by this library since load (host counter). */
MM_API int64_t mm_launch_count(void);
/* Which kernel (b) an exact sweep of n vertices in `dim` dimensions uses:
 * 0 = one-sided tiled kernel (every ordered pair evaluated), 1 = symmetric
 * kernel (every unordered pair evaluated once and applied to both vertices,
 * DESIGN.md §5).  Host-only query (no GPU work; needs a current device for the
 * SM count); environment MM_SYM=0 forces 0, MM_SYM=2 forces 1. */
MM_API int mm_exact_kernel_variant(int32_t n, int dim);
/* When enabled, every kernel launch is bracketed by CUDA events on its
 * stream; mm_profile_read syncs those events and returns, per kernel name,
 * the launch count and summed device milliseconds. */
typedef struct {
    char name[48];
    int64_t launches;
    double total_ms;
} mm_kernel_profile;
MM_API mm_status mm_profile_enable(int on);
MM_API mm_status mm_profile_reset(void);
/* writes up to max entries into out (host); *count = number of kernel names */
MM_API mm_status mm_profile_read(mm_kernel_profile* out, int32_t max, int32_t* count);
/* the device milliseconds of the LAST (up to max) timed launches of kernel
 * `name` since mm_profile_reset, in launch order, into ms (host); *count =
 * how many.  E.g. the finest level of a layout runs last, so its K sweeps'
 * launches are the last K of each per-sweep kernel.  syncs their events. */
MM_API mm_status mm_profile_last(const char* name, int32_t max, double* ms, int32_t* count);

#ifdef __cplusplus
}
#endif
#endif /* MM_H */
