/* Input-generator helper (NOT method arithmetic): for every vertex u of a
 * symmetric CSR graph with sorted adjacency rows, find the `cap` lowest-id
 * vertices at hop distance exactly 2.  This builds the config-4 stress pair
 * set S = E ∪ {capped hop-2} (BASELINE.json configs[3]: "S = edges plus
 * 2-hop pairs capped at 64 per vertex by lowest vertex id").  Used by
 * workloads/sset.py and shared by the oracle tests and the GPU tests alike,
 * so it holds no part of Eq.(2)/(3).
 *
 * Method: a k-way merge (binary min-heap) over the sorted neighbour lists
 * N(v), v ∈ N(u); the merge pops ids in ascending order, skipping u, N(u)
 * and repeats, and stops after `cap` accepted ids. */
#include <stdint.h>
#include <stdlib.h>

typedef struct { int32_t id; int32_t src; int64_t pos; } hent;

static void sift_down(hent* h, int32_t n, int32_t i) {
    for (;;) {
        int32_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < n && h[l].id < h[m].id) m = l;
        if (r < n && h[r].id < h[m].id) m = r;
        if (m == i) return;
        hent t = h[i]; h[i] = h[m]; h[m] = t; i = m;
    }
}

/* out: int32 [n*cap] (row u at u*cap), cnt: int32 [n] */
int gen_capped2hop(int32_t n, const int64_t* rp, const int32_t* col, int32_t cap,
                   int32_t* out, int32_t* cnt) {
    int32_t* stamp = (int32_t*)calloc((size_t)n, sizeof(int32_t));
    int64_t dmax = 0;
    for (int32_t u = 0; u < n; ++u) if (rp[u + 1] - rp[u] > dmax) dmax = rp[u + 1] - rp[u];
    hent* heap = (hent*)malloc(sizeof(hent) * (size_t)(dmax + 1));
    if (!stamp || !heap) { free(stamp); free(heap); return -1; }
    for (int32_t u = 0; u < n; ++u) {
        const int32_t tag = u + 1;  /* 1-based stamps; 0 = never stamped */
        stamp[u] = tag;
        for (int64_t k = rp[u]; k < rp[u + 1]; ++k) stamp[col[k]] = tag;
        int32_t hn = 0;
        for (int64_t k = rp[u]; k < rp[u + 1]; ++k) {
            const int32_t v = col[k];
            if (rp[v] < rp[v + 1]) { heap[hn].id = col[rp[v]]; heap[hn].src = v; heap[hn].pos = rp[v]; ++hn; }
        }
        for (int32_t i = hn / 2 - 1; i >= 0; --i) sift_down(heap, hn, i);
        int32_t m = 0;
        int32_t* o = out + (int64_t)u * cap;
        while (hn > 0 && m < cap) {
            const int32_t x = heap[0].id;
            if (stamp[x] != tag) { stamp[x] = tag; o[m++] = x; }  /* accept; stamp dedups */
            const int32_t v = heap[0].src;
            const int64_t p = heap[0].pos + 1;
            if (p < rp[v + 1]) { heap[0].id = col[p]; heap[0].pos = p; }
            else { heap[0] = heap[--hn]; }
            sift_down(heap, hn, 0);
        }
        cnt[u] = m;
    }
    free(stamp); free(heap);
    return 0;
}
