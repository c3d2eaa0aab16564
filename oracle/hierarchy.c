/* ORACLE (test infrastructure only) — multilevel hierarchy, integer-exact.
 *
 * Contraction follows PAPER.md P:225-232: "each block of the clustering is
 * contracted into a single node.  The weight of the node is set to the sum of
 * the weight of all nodes in the original block.  There is an edge between two
 * nodes u' and v' ... if the two corresponding blocks ... are connected by at
 * least one edge.  The weight of an edge (u',v') is set to the sum of the
 * weight of edges that run between block u' and block v'."  Repeated
 * recursively.
 *
 * The default clustering is BASELINE.json's "seeded heavy-edge matching"
 * (the paper's SCLaP, is sclap.c + or_build_hierarchy_sclap), read as Q16:
 * a synchronous handshake.  In round r every unmatched u picks the unmatched
 * neighbour v maximising the rating omega_uv / (c_u c_v) — compared exactly
 * as omega_a * c_b  vs  omega_b * c_a in 64-bit integers — ties broken by the
 * higher hash mix(mix(mix(mix(seed ^ TAG_MATCH) ^ level) ^ r) ^ (min<<32|max)),
 * then by the lower id; u and v match when they picked each other.  At most
 * max_rounds rounds, or until a round adds no match.  Coarse ids are the rank
 * of the cluster leader min(u, mate(u)) in ascending id order.
 * Stop rule Q17: stop when n_l <= n_stop, when a contraction would keep more
 * than 90% of the vertices (that level is discarded), or at max_levels. */
#include <stdlib.h>
#include <string.h>

#include "mm_oracle.h"

typedef struct {
    int32_t n;
    int64_t nnz;
    int64_t* rp;
    int32_t* col;
    int64_t* omega;
    int64_t* c;
    int32_t* parent; /* to level l+1; NULL at the coarsest */
    int32_t rounds;
} or_level;

struct or_hierarchy {
    int32_t L; /* number of levels */
    or_level* lv;
};

static void free_level(or_level* l) {
    free(l->rp); free(l->col); free(l->omega); free(l->c); free(l->parent);
    memset(l, 0, sizeof(*l));
}

static uint64_t match_hash(uint64_t seed, int32_t level, int32_t round, int32_t u, int32_t v) {
    const uint64_t lo = (uint64_t)(uint32_t)(u < v ? u : v), hi = (uint64_t)(uint32_t)(u < v ? v : u);
    uint64_t k = or_mix64(seed ^ OR_TAG_MATCH);
    k = or_mix64(k ^ (uint64_t)level);
    k = or_mix64(k ^ (uint64_t)round);
    return or_mix64(k ^ ((lo << 32) | hi));
}

/* handshake matching on level graph g; writes mate[] (-1 = unmatched) */
static int32_t match_level(const or_level* g, uint64_t seed, int32_t level, int32_t max_rounds,
                           int32_t* mate, int32_t* cand) {
    const int32_t n = g->n;
    for (int32_t u = 0; u < n; ++u) mate[u] = -1;
    int32_t r = 0;
    for (; r < max_rounds; ++r) {
        for (int32_t u = 0; u < n; ++u) {
            cand[u] = -1;
            if (mate[u] >= 0) continue;
            int32_t best = -1;
            int64_t wb = 0, cb = 0;
            uint64_t hb = 0;
            for (int64_t e = g->rp[u]; e < g->rp[u + 1]; ++e) {
                const int32_t v = g->col[e];
                if (v == u || mate[v] >= 0) continue;
                const int64_t wv = g->omega[e], cv = g->c[v];
                const uint64_t hv = match_hash(seed, level, r, u, v);
                int better;
                if (best < 0) {
                    better = 1;
                } else {
                    const int64_t lhs = wv * cb, rhs = wb * cv; /* wv/cv > wb/cb ? */
                    if (lhs != rhs) better = lhs > rhs;
                    else if (hv != hb) better = hv > hb;
                    else better = v < best;
                }
                if (better) { best = v; wb = wv; cb = cv; hb = hv; }
            }
            cand[u] = best;
        }
        int32_t added = 0;
        for (int32_t u = 0; u < n; ++u) {
            if (mate[u] >= 0 || cand[u] < 0) continue;
            const int32_t v = cand[u];
            if (cand[v] == u) { mate[u] = v; ++added; }
        }
        if (added == 0) { ++r; break; }
    }
    return r; /* rounds executed */
}

typedef struct { int32_t col; int64_t w; } centry;
static int contract_labels(or_level* g, const int32_t* lead, or_level* out);

/* matching: leader = min(u, mate(u)) */
static int contract_level(or_level* g, const int32_t* mate, or_level* out) {
    int32_t* lead = (int32_t*)malloc(sizeof(int32_t) * (size_t)(g->n > 0 ? g->n : 1));
    if (!lead) return OR_ENOMEM;
    for (int32_t u = 0; u < g->n; ++u) lead[u] = (mate[u] >= 0 && mate[u] < u) ? mate[u] : u;
    const int rc = contract_labels(g, lead, out);
    free(lead);
    return rc;
}
static int cmp_centry(const void* a, const void* b) {
    const centry* x = (const centry*)a; const centry* y = (const centry*)b;
    return (x->col > y->col) - (x->col < y->col);
}

/* contract g by cluster labels (lead[u] in [0, n) names u's cluster) into
 * out; coarse ids = rank of the distinct label values in ascending order (for
 * the matching, lead = min(u, mate(u)): the rank of the cluster leader);
 * sets g->parent */
static int contract_labels(or_level* g, const int32_t* lead, or_level* out) {
    const int32_t n = g->n;
    int32_t* cid = (int32_t*)calloc((size_t)(n > 0 ? n : 1), sizeof(int32_t));
    g->parent = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    if (!cid || !g->parent) { free(cid); return OR_ENOMEM; }
    for (int32_t u = 0; u < n; ++u) cid[lead[u]] = 1; /* label used */
    int32_t nc = 0;
    for (int32_t L = 0; L < n; ++L) cid[L] = cid[L] ? nc++ : -1;
    for (int32_t u = 0; u < n; ++u) g->parent[u] = cid[lead[u]];
    free(cid);
    out->n = nc;
    out->c = (int64_t*)calloc((size_t)(nc > 0 ? nc : 1), sizeof(int64_t));
    out->rp = (int64_t*)calloc((size_t)nc + 1, sizeof(int64_t));
    if (!out->c || !out->rp) return OR_ENOMEM;
    for (int32_t u = 0; u < n; ++u) out->c[g->parent[u]] += g->c[u];
    /* bucket crossing edges by coarse source, then sort + merge each row */
    int64_t* cnt = (int64_t*)calloc((size_t)nc + 1, sizeof(int64_t));
    if (!cnt) return OR_ENOMEM;
    for (int32_t u = 0; u < n; ++u)
        for (int64_t e = g->rp[u]; e < g->rp[u + 1]; ++e)
            if (g->parent[u] != g->parent[g->col[e]]) cnt[g->parent[u] + 1] += 1;
    for (int32_t p = 0; p < nc; ++p) cnt[p + 1] += cnt[p];
    const int64_t tot = cnt[nc];
    centry* buf = (centry*)malloc(sizeof(centry) * (size_t)(tot > 0 ? tot : 1));
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nc > 0 ? nc : 1));
    if (!buf || !fill) { free(cnt); free(buf); free(fill); return OR_ENOMEM; }
    for (int32_t p = 0; p < nc; ++p) fill[p] = cnt[p];
    for (int32_t u = 0; u < n; ++u)
        for (int64_t e = g->rp[u]; e < g->rp[u + 1]; ++e) {
            const int32_t pu = g->parent[u], pv = g->parent[g->col[e]];
            if (pu == pv) continue; /* intra-cluster edges vanish */
            buf[fill[pu]].col = pv;
            buf[fill[pu]].w = g->omega[e];
            fill[pu] += 1;
        }
    int64_t m = 0;
    for (int32_t p = 0; p < nc; ++p) {
        const int64_t b = cnt[p], e = cnt[p + 1];
        qsort(buf + b, (size_t)(e - b), sizeof(centry), cmp_centry);
        for (int64_t t = b; t < e; ++t)
            if (t == b || buf[t].col != buf[t - 1].col) ++m;
    }
    out->nnz = m;
    out->col = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
    out->omega = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m > 0 ? m : 1));
    if (!out->col || !out->omega) { free(cnt); free(buf); free(fill); return OR_ENOMEM; }
    int64_t pos = 0;
    for (int32_t p = 0; p < nc; ++p) {
        out->rp[p] = pos;
        const int64_t b = cnt[p], e = cnt[p + 1];
        for (int64_t t = b; t < e; ++t) {
            if (t == b || buf[t].col != buf[t - 1].col) {
                out->col[pos] = buf[t].col;
                out->omega[pos] = buf[t].w;
                ++pos;
            } else {
                out->omega[pos - 1] += buf[t].w;
            }
        }
    }
    out->rp[nc] = pos;
    free(cnt); free(buf); free(fill);
    return 0;
}

int or_build_hierarchy(int32_t n, const int64_t* rp, const int32_t* col,
                       const int64_t* omega, const int64_t* c,
                       uint64_t seed, int32_t n_stop, int32_t max_levels, int32_t max_rounds,
                       or_hierarchy** out) {
    if (n <= 0 || !rp || !col || !out || max_levels < 1 || max_rounds < 1) return OR_EINVAL;
    or_hierarchy* H = (or_hierarchy*)calloc(1, sizeof(or_hierarchy));
    if (!H) return OR_ENOMEM;
    H->lv = (or_level*)calloc((size_t)max_levels, sizeof(or_level));
    if (!H->lv) { free(H); return OR_ENOMEM; }
    or_level* l0 = &H->lv[0];
    l0->n = n;
    l0->nnz = rp[n];
    l0->rp = (int64_t*)malloc(sizeof(int64_t) * ((size_t)n + 1));
    l0->col = (int32_t*)malloc(sizeof(int32_t) * (size_t)(l0->nnz > 0 ? l0->nnz : 1));
    l0->omega = (int64_t*)malloc(sizeof(int64_t) * (size_t)(l0->nnz > 0 ? l0->nnz : 1));
    l0->c = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    if (!l0->rp || !l0->col || !l0->omega || !l0->c) { or_hier_free(H); return OR_ENOMEM; }
    memcpy(l0->rp, rp, sizeof(int64_t) * ((size_t)n + 1));
    memcpy(l0->col, col, sizeof(int32_t) * (size_t)l0->nnz);
    for (int64_t e = 0; e < l0->nnz; ++e) l0->omega[e] = omega ? omega[e] : 1;
    for (int32_t u = 0; u < n; ++u) l0->c[u] = c ? c[u] : 1;
    H->L = 1;
    int32_t* mate = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    int32_t* cand = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    if (!mate || !cand) { free(mate); free(cand); or_hier_free(H); return OR_ENOMEM; }
    while (H->L < max_levels) {
        or_level* g = &H->lv[H->L - 1];
        if (g->n <= n_stop) break;
        g->rounds = match_level(g, seed, H->L - 1, max_rounds, mate, cand);
        or_level next;
        memset(&next, 0, sizeof(next));
        const int rc = contract_level(g, mate, &next);
        if (rc) { free_level(&next); free(mate); free(cand); or_hier_free(H); return rc; }
        if ((int64_t)10 * next.n > (int64_t)9 * g->n) { /* less than 10% smaller: discard */
            free_level(&next);
            free(g->parent);
            g->parent = NULL;
            break;
        }
        H->lv[H->L] = next;
        H->L += 1;
    }
    free(mate); free(cand);
    *out = H;
    return 0;
}

/* SCLaP hierarchy (reading R6): level h = 1, 2, ... uses
 * U = max(max c, W), W = min(b^h, n0 / f); after a contraction that is not
 * more than 10% smaller, f <- 0.7 f (the level is kept); stop at n <= n_stop,
 * max_levels, or 10 consecutive ineffective decays, or when nothing merges. */
int or_sclap_labels(int32_t n, const int64_t* rp, const int32_t* col, const int64_t* omega, const int64_t* c,
                    int64_t U, int32_t rounds, uint64_t seed, int32_t level, int32_t* lab);

int or_build_hierarchy_sclap(int32_t n, const int64_t* rp, const int32_t* col, const int64_t* omega,
                             const int64_t* c, uint64_t seed, int32_t n_stop, int32_t max_levels, int32_t rounds,
                             double f0, double b, or_hierarchy** out) {
    return or_build_hierarchy_sclap_mode(n, rp, col, omega, c, seed, n_stop, max_levels, rounds, f0, b, 0, out);
}

/* seq = 1: the paper's sequential label propagation (R6s, or_sclap_labels_seq);
 * seq = 0: the synchronous reading R6 (or_sclap_labels) */
int or_build_hierarchy_sclap_mode(int32_t n, const int64_t* rp, const int32_t* col, const int64_t* omega,
                                  const int64_t* c, uint64_t seed, int32_t n_stop, int32_t max_levels,
                                  int32_t rounds, double f0, double b, int seq, or_hierarchy** out) {
    if (n <= 0 || !rp || !col || !out || max_levels < 1 || rounds < 1 || !(f0 > 0.0) || !(b > 1.0)) return OR_EINVAL;
    or_hierarchy* H = NULL;
    /* level 0 via the matching builder with max_levels = 1 (copies the graph) */
    int rc = or_build_hierarchy(n, rp, col, omega, c, seed, n, 1, 1, &H);
    if (rc) return rc;
    or_level* tmp = (or_level*)realloc(H->lv, sizeof(or_level) * (size_t)max_levels);
    if (!tmp) { or_hier_free(H); return OR_ENOMEM; }
    H->lv = tmp;
    memset(H->lv + 1, 0, sizeof(or_level) * (size_t)(max_levels - 1));
    int32_t* lab = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    if (!lab) { or_hier_free(H); return OR_ENOMEM; }
    double f = f0;
    int decays = 0;
    while (H->L < max_levels) {
        or_level* g = &H->lv[H->L - 1];
        if (g->n <= n_stop) break;
        const int32_t h = H->L; /* first coarsening uses h = 1 */
        int64_t cmax = 0;
        for (int32_t u = 0; u < g->n; ++u) if (g->c[u] > cmax) cmax = g->c[u];
        double W = 1.0;
        for (int32_t t = 0; t < h && W < 1e18; ++t) W *= b;
        if ((double)n / f < W) W = (double)n / f;
        const int64_t Wi = (int64_t)W; /* floor: cluster weights are integers */
        const int64_t U = cmax > Wi ? cmax : Wi;
        rc = seq ? or_sclap_labels_seq(g->n, g->rp, g->col, g->omega, g->c, U, rounds, seed, h - 1, lab)
                 : or_sclap_labels(g->n, g->rp, g->col, g->omega, g->c, U, rounds, seed, h - 1, lab);
        if (rc) break;
        g->rounds = rounds;
        or_level next;
        memset(&next, 0, sizeof(next));
        rc = contract_labels(g, lab, &next);
        if (rc) { free(next.rp); free(next.col); free(next.omega); free(next.c); break; }
        if (next.n == g->n) { /* nothing merged: stop, discard */
            free(next.rp); free(next.col); free(next.omega); free(next.c);
            free(g->parent);
            g->parent = NULL;
            if (++decays >= 10) break;
            f *= 0.7;
            continue;
        }
        if ((int64_t)10 * next.n > (int64_t)9 * g->n) {
            f *= 0.7;
            ++decays;
        } else {
            decays = 0;
        }
        H->lv[H->L] = next;
        H->L += 1;
        if (decays >= 10) break;
    }
    free(lab);
    if (rc) { or_hier_free(H); return rc; }
    *out = H;
    return 0;
}

int32_t or_hier_num_levels(const or_hierarchy* h) { return h ? h->L : 0; }

int or_hier_level(const or_hierarchy* h, int32_t l, int32_t* n, int64_t* nnz,
                  const int64_t** rp, const int32_t** col, const int64_t** omega,
                  const int64_t** c, const int32_t** parent, int32_t* rounds) {
    if (!h || l < 0 || l >= h->L) return OR_EINVAL;
    const or_level* g = &h->lv[l];
    *n = g->n; *nnz = g->nnz; *rp = g->rp; *col = g->col; *omega = g->omega; *c = g->c;
    *parent = (l + 1 < h->L) ? g->parent : NULL;
    *rounds = g->rounds;
    return 0;
}

void or_hier_free(or_hierarchy* h) {
    if (!h) return;
    for (int32_t l = 0; l < h->L; ++l) free_level(&h->lv[l]);
    free(h->lv);
    free(h);
}
