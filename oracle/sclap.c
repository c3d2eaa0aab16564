/* ORACLE (test infrastructure only) — SCLaP coarsening,
 * integer-exact.  Two functions:
 *   or_sclap_labels_seq  the paper's label propagation as written (reading
 *                        R6s below): nodes visited one at a time in a random
 *                        order, each move applied immediately;
 *   or_sclap_labels      the synchronous reading R6 of DESIGN.md that the GPU
 *                        implements (a parallel rule; checked against the
 *                        sequential one for validity and quality in tests).
 *
 * label propagation "starts with a singleton clustering
 * ... in each round the algorithm visits all nodes ... and assigns each node to
 * the predominant cluster in its neighborhood"; SCLaP "introduces an upper
 * bound U := max(max_v c(v), W) on the cluster sizes ... nodes are assigned to
 * the predominant cluster that is not overloaded after the label change";
 * "W = min(b^h, |V|/f) ... h is the level in the hierarchy"; "If the
 * contracted graph is not more than 10% smaller than the graph on the current
 * level, we decrease the value of f and set it to 0.7f"; "SCLaP performs at
 * most l rounds".  Contraction P:225-232 (shared with the matching hierarchy).
 *
 * R6 (a deterministic, parallel-friendly reading of the sequential random
 * order): round r works on the labels and cluster weights at its start.
 *  1. score_v(L) = sum of omega(v,u) over neighbours u with label L; s0 = score
 *     of v's own label (0 if no neighbour shares it).
 *  2. v requests the label L maximising (score desc, hash(seed,level,r,v,L)
 *     desc, L asc) among labels L < label(v) with cw(L) + c(v) <= U, if
 *     score_v(L) > s0 (strict improvement; "L < label(v)" forbids swaps).
 *  3. each target label accepts the longest prefix of its requests ordered by
 *     (gain desc, hash desc, v asc) whose weights keep cw(L) <= U.
 *  4. accepted nodes take the label; weights are recomputed.  Stop after l
 *     rounds or a round without moves.
 * Coarse ids = rank of the distinct labels in ascending order. */
#include <stdlib.h>
#include <string.h>

#include "mm_oracle.h"

#define OR_TAG_LP 0x4c505250ULL /* "LPRP" */

static uint64_t lp_hash(uint64_t seed, int32_t level, int32_t round, int32_t v, int32_t L) {
    uint64_t k = or_mix64(seed ^ OR_TAG_LP);
    k = or_mix64(k ^ (uint64_t)level);
    k = or_mix64(k ^ (uint64_t)round);
    return or_mix64(k ^ (((uint64_t)(uint32_t)v << 32) | (uint32_t)L));
}

typedef struct { int32_t v, L; int64_t gain; uint64_t h; int64_t c; } lp_req;
static int cmp_req(const void* a, const void* b) {
    const lp_req* x = (const lp_req*)a; const lp_req* y = (const lp_req*)b;
    if (x->L != y->L) return x->L < y->L ? -1 : 1;
    if (x->gain != y->gain) return x->gain > y->gain ? -1 : 1;
    if (x->h != y->h) return x->h > y->h ? -1 : 1;
    return (x->v > y->v) - (x->v < y->v);
}
typedef struct { int32_t L; int64_t w; } lw;
static int cmp_lw(const void* a, const void* b) {
    const lw* x = (const lw*)a; const lw* y = (const lw*)b;
    return (x->L > y->L) - (x->L < y->L);
}

/* R6s, the paper's sequential label propagation: "starts with a
 * singleton clustering", "works in rounds", "in each round the algorithm
 * visits all nodes in random order and assigns each node to the predominant
 * cluster in its neighborhood"; SCLaP: "nodes are assigned to the
 * predominant cluster that is not overloaded after the label change", i.e.
 * cw(L) + c(v) <= U for L != label(v).  Silences, read here: the random order
 * of round r is a Fisher-Yates shuffle driven by the counter RNG of (seed,
 * "LPSQ", level, r, i); "predominant" = largest sum of edge weights omega to
 * the cluster; a node leaves its cluster only for a strictly larger score
 * (ties with its own label keep it; ties among other labels: higher hash of
 * (seed, level, r, v, L), then the lower label); labels and cluster weights
 * are updated immediately, so later nodes of the round see the move.  Stop
 * after `rounds` rounds (the paper's l) or a round without moves. */
#define OR_TAG_LPSQ 0x4c505351ULL /* "LPSQ" */
int or_sclap_labels_seq(int32_t n, const int64_t* rp, const int32_t* col, const int64_t* omega, const int64_t* c,
                        int64_t U, int32_t rounds, uint64_t seed, int32_t level, int32_t* lab) {
    int64_t* cw = (int64_t*)calloc((size_t)(n > 0 ? n : 1), sizeof(int64_t));
    int64_t* acc = (int64_t*)calloc((size_t)(n > 0 ? n : 1), sizeof(int64_t));
    int32_t* touched = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    if (!cw || !acc || !touched || !order) { free(cw); free(acc); free(touched); free(order); return OR_ENOMEM; }
    for (int32_t v = 0; v < n; ++v) { lab[v] = v; cw[v] = c[v]; }
    for (int32_t r = 0; r < rounds; ++r) {
        /* random visiting order of this round */
        const uint64_t k0 = or_mix64(or_mix64(or_mix64(seed ^ OR_TAG_LPSQ) ^ (uint64_t)level) ^ (uint64_t)r);
        for (int32_t i = 0; i < n; ++i) order[i] = i;
        for (int32_t i = n - 1; i > 0; --i) {
            const int32_t j = (int32_t)(or_mix64(k0 ^ (uint64_t)i) % (uint64_t)(i + 1));
            const int32_t t = order[i]; order[i] = order[j]; order[j] = t;
        }
        int32_t moved = 0;
        for (int32_t t = 0; t < n; ++t) {
            const int32_t v = order[t];
            int32_t m = 0;
            for (int64_t e = rp[v]; e < rp[v + 1]; ++e) {
                const int32_t u = col[e];
                if (u == v) continue;
                const int32_t L = lab[u];
                if (acc[L] == 0) touched[m++] = L;
                acc[L] += omega[e];
            }
            const int32_t own = lab[v];
            const int64_t s0 = acc[own];
            int32_t best = -1;
            int64_t bs = 0;
            uint64_t bh = 0;
            for (int32_t q = 0; q < m; ++q) {
                const int32_t L = touched[q];
                const int64_t s = acc[L];
                if (L == own || cw[L] + c[v] > U) continue;
                const uint64_t h = lp_hash(seed, level, r, v, L);
                if (best < 0 || s > bs || (s == bs && (h > bh || (h == bh && L < best)))) {
                    best = L; bs = s; bh = h;
                }
            }
            for (int32_t q = 0; q < m; ++q) acc[touched[q]] = 0;
            if (best >= 0 && bs > s0) {
                cw[own] -= c[v];
                cw[best] += c[v];
                lab[v] = best;
                ++moved;
            }
        }
        if (moved == 0) break;
    }
    free(cw); free(acc); free(touched); free(order);
    return 0;
}

/* One SCLaP clustering of graph (n, rp, col, omega, c) with bound U; labels out. */
int or_sclap_labels(int32_t n, const int64_t* rp, const int32_t* col, const int64_t* omega, const int64_t* c,
                    int64_t U, int32_t rounds, uint64_t seed, int32_t level, int32_t* lab) {
    int64_t* cw = (int64_t*)calloc((size_t)n, sizeof(int64_t));
    lp_req* req = (lp_req*)malloc(sizeof(lp_req) * (size_t)(n > 0 ? n : 1));
    int64_t dmax = 0;
    for (int32_t v = 0; v < n; ++v) if (rp[v + 1] - rp[v] > dmax) dmax = rp[v + 1] - rp[v];
    lw* sc = (lw*)malloc(sizeof(lw) * (size_t)(dmax > 0 ? dmax : 1));
    if (!cw || !req || !sc) { free(cw); free(req); free(sc); return OR_ENOMEM; }
    for (int32_t v = 0; v < n; ++v) { lab[v] = v; cw[v] = c[v]; }
    for (int32_t r = 0; r < rounds; ++r) {
        int32_t nreq = 0;
        for (int32_t v = 0; v < n; ++v) {
            /* scores of neighbour labels (start-of-round labels) */
            int64_t m = 0;
            for (int64_t e = rp[v]; e < rp[v + 1]; ++e) {
                if (col[e] == v) continue;
                sc[m].L = lab[col[e]];
                sc[m].w = omega[e];
                ++m;
            }
            qsort(sc, (size_t)m, sizeof(lw), cmp_lw);
            int64_t s0 = 0;
            int32_t best = -1;
            int64_t bs = 0;
            uint64_t bh = 0;
            for (int64_t t = 0; t < m;) {
                const int32_t L = sc[t].L;
                int64_t s = 0;
                while (t < m && sc[t].L == L) s += sc[t++].w;
                if (L == lab[v]) { s0 = s; continue; }
                if (L >= lab[v] || cw[L] + c[v] > U) continue;
                const uint64_t h = lp_hash(seed, level, r, v, L);
                if (best < 0 || s > bs || (s == bs && (h > bh || (h == bh && L < best)))) {
                    best = L; bs = s; bh = h;
                }
            }
            if (best >= 0 && bs > s0) {
                req[nreq].v = v; req[nreq].L = best; req[nreq].gain = bs - s0; req[nreq].h = bh; req[nreq].c = c[v];
                ++nreq;
            }
        }
        if (nreq == 0) break;
        qsort(req, (size_t)nreq, sizeof(lp_req), cmp_req);
        int32_t moved = 0;
        for (int32_t t = 0; t < nreq;) {
            const int32_t L = req[t].L;
            int64_t acc = cw[L];
            int ok = 1;
            for (; t < nreq && req[t].L == L; ++t) {
                if (ok && acc + req[t].c <= U) {
                    acc += req[t].c;
                    req[t].gain = -1; /* accepted marker */
                } else {
                    ok = 0; /* longest prefix only */
                }
            }
        }
        for (int32_t t = 0; t < nreq; ++t)
            if (req[t].gain == -1) { lab[req[t].v] = req[t].L; ++moved; }
        memset(cw, 0, sizeof(int64_t) * (size_t)n);
        for (int32_t v = 0; v < n; ++v) cw[lab[v]] += c[v];
        if (moved == 0) break;
    }
    free(cw); free(req); free(sc);
    return 0;
}
