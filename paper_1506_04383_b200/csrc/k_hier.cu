// k_hier.cu — kernels (d): handshake heavy-edge matching, contraction,
// coarse S^l, grouping maps into CSR, centroid/mass refresh, prolongation and
// the coarsest-level initial layout.
//
// Contraction: "each block of the clustering is
// contracted into a single node.  The weight of the node is set to the sum of
// the weight of all nodes in the original block ... The weight of an edge
// (u',v') is set to the sum of the weight of edges that run between block u'
// and block v'."  The clustering is BASELINE.json's seeded heavy-edge
// matching, read as Q16: synchronous handshake rounds; rating
// omega_uv / (c_u c_v) compared exactly in int64; ties -> higher SplitMix64
// hash of (seed, level, round, min, max) -> lower id; coarse id = rank of the
// leader min(u, mate(u)).  All integer work, so the result is bit-identical to
// the oracle's.
//
// Centroids (Q10-Q12): nu(v') = number of current-level
// members, x'_v' = their unweighted mean; members are visited in ascending
// id order from a CSR built by a stable sort, so the FP32 sum is deterministic.
// Prolongation (Q15, BASELINE.json configs[2]): x_u = x_{P(u)} + 1e-3 (2U - 1)
// per component, U from the counter RNG keyed (seed, JITTER, level, u*dim+k).
#include "k_perm.cuh"
#include "k_sort.cuh"

#include "k_hier.cuh"

namespace mm {

namespace {

__device__ __forceinline__ uint64_t match_hash(uint64_t seed, int32_t level, int32_t round, int32_t u, int32_t v) {
    const uint64_t lo = (uint64_t)(uint32_t)min(u, v), hi = (uint64_t)(uint32_t)max(u, v);
    uint64_t k = mix64(seed ^ kTagMatch);
    k = mix64(k ^ (uint64_t)level);
    k = mix64(k ^ (uint64_t)round);
    return mix64(k ^ ((lo << 32) | hi));
}

// Candidate order of the handshake (Q16): higher rating omega/(c_u c_v)
// (exact: w_a c_b vs w_b c_a in int64), then higher hash, then lower id.
struct Cand {
    int32_t v;
    int32_t w;
    int32_t c;
    uint64_t h;
};
__device__ __forceinline__ bool cand_better(const Cand& a, const Cand& b) {
    if (a.v < 0) return false;
    if (b.v < 0) return true;
    const int64_t lhs = (int64_t)a.w * b.c, rhs = (int64_t)b.w * a.c;
    if (lhs != rhs) return lhs > rhs;
    if (a.h != b.h) return a.h > b.h;
    return a.v < b.v;
}

// G lanes per vertex (G from the mean degree): the group scans the row
// strided, then a shuffle reduction under the (total) candidate order picks
// the best unmatched neighbour.  All lanes reach the shuffles.
template <int G>
__global__ void k_match_pick(int32_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                             const int32_t* __restrict__ omega, const int32_t* __restrict__ c,
                             const int32_t* __restrict__ mate, int32_t* __restrict__ cand, uint64_t seed,
                             int32_t level, int32_t round) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int32_t u = (int32_t)(t / G);
    const int lg = (int)(t & (G - 1));
    Cand best{-1, 0, 1, 0};
    const bool active = u < n && mate[u] < 0;
    if (active) {
        const int64_t e1 = rp[u + 1];
        for (int64_t e = rp[u] + lg; e < e1; e += G) {
            const int32_t v = col[e];
            if (v == u || mate[v] >= 0) continue;
            const Cand cv{v, omega ? omega[e] : 1, c[v], match_hash(seed, level, round, u, v)};
            if (cand_better(cv, best)) best = cv;
        }
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
        Cand other;
        other.v = __shfl_xor_sync(0xffffffffu, best.v, o, G);
        other.w = __shfl_xor_sync(0xffffffffu, best.w, o, G);
        other.c = __shfl_xor_sync(0xffffffffu, best.c, o, G);
        other.h = __shfl_xor_sync(0xffffffffu, best.h, o, G);
        if (cand_better(other, best)) best = other;
    }
    if (u < n && lg == 0) cand[u] = active ? best.v : -1;
}

// ---------------------------------------------------------------------------
// All handshake rounds of one level in ONE cooperative launch (every CTA
// resident; grid barriers between the phases): per round, pick (G lanes per
// unmatched vertex, as k_match_pick) -> barrier -> confirm (mutual picks match,
// counted) -> barrier -> every CTA reads the count and continues while a round
// added a match and fewer than max_rounds ran.  Same rounds, same hashes, same
// decisions as the host loop of k_match_pick / k_match_confirm launches.
// Arrays written inside the launch (mate, cand, the counters) are read
// through L2 (ld.global.cg), never the non-coherent path.
struct MatchSync {
    unsigned count;
    unsigned gen;
};
__device__ MatchSync g_match_sync;

__device__ __forceinline__ void match_grid_barrier(unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* gen = &g_match_sync.gen;
        const unsigned g = *gen;
        __threadfence();
        if (atomicAdd(&g_match_sync.count, 1u) == nblocks - 1) {
            g_match_sync.count = 0;
            __threadfence();
            atomicAdd(&g_match_sync.gen, 1u);
        } else {
            while (*gen == g) __nanosleep(40);
        }
        __threadfence();
    }
    __syncthreads();
}

template <int G>
__global__ void __launch_bounds__(256) k_match_level(int32_t n, const int64_t* __restrict__ rp,
                                                     const int32_t* __restrict__ col, const int32_t* __restrict__ omega,
                                                     const int32_t* __restrict__ c, int32_t* mate, int32_t* cand,
                                                     uint64_t seed, int32_t level, int32_t max_rounds,
                                                     int32_t* added /* [2], zeroed */, int32_t* rounds_out) {
    const unsigned NB = gridDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)NB * blockDim.x;
    const int lg = (int)(t0 & (G - 1));
    const int64_t ngroups = nt / G;
    const int64_t iters = ((int64_t)n + ngroups - 1) / ngroups;
    __shared__ int32_t s_cnt;
    int32_t round = 0;
    for (;;) {
        // ---- pick: G lanes per vertex, uniform trip count (the shuffles need every lane)
        for (int64_t r = 0; r < iters; ++r) {
            const int64_t uu = t0 / G + r * ngroups;
            const int32_t u = (int32_t)(uu < n ? uu : n - 1);
            Cand best{-1, 0, 1, 0};
            const bool active = uu < n && __ldcg(mate + u) < 0;
            if (active) {
                const int64_t e1 = rp[u + 1];
                for (int64_t e = rp[u] + lg; e < e1; e += G) {
                    const int32_t v = col[e];
                    if (v == u || __ldcg(mate + v) >= 0) continue;
                    const Cand cv{v, omega ? omega[e] : 1, c[v], match_hash(seed, level, round, u, v)};
                    if (cand_better(cv, best)) best = cv;
                }
            }
#pragma unroll
            for (int o = G / 2; o > 0; o >>= 1) {
                Cand other;
                other.v = __shfl_xor_sync(0xffffffffu, best.v, o, G);
                other.w = __shfl_xor_sync(0xffffffffu, best.w, o, G);
                other.c = __shfl_xor_sync(0xffffffffu, best.c, o, G);
                other.h = __shfl_xor_sync(0xffffffffu, best.h, o, G);
                if (cand_better(other, best)) best = other;
            }
            if (uu < n && lg == 0) cand[u] = active ? best.v : -1;
        }
        match_grid_barrier(NB);
        // the next round's counter: every CTA read it (as round - 1's) before this barrier
        if (blockIdx.x == 0 && threadIdx.x == 0) added[(round + 1) & 1] = 0;
        // ---- confirm: mutual picks match
        if (threadIdx.x == 0) s_cnt = 0;
        __syncthreads();
        int32_t hit = 0;
        for (int64_t u = t0; u < n; u += nt) {
            if (__ldcg(mate + u) < 0) {
                const int32_t v = __ldcg(cand + u);
                if (v >= 0 && __ldcg(cand + v) == (int32_t)u) {
                    mate[u] = v;
                    ++hit;
                }
            }
        }
        hit = __reduce_add_sync(0xffffffffu, hit);
        if ((threadIdx.x & 31) == 0 && hit) atomicAdd(&s_cnt, hit);
        __syncthreads();
        if (threadIdx.x == 0 && s_cnt) atomicAdd(added + (round & 1), s_cnt);
        match_grid_barrier(NB);
        const int32_t a = __ldcg(added + (round & 1));
        ++round;
        if (a == 0 || round >= max_rounds) break;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *rounds_out = round;
}

__global__ void k_match_confirm(int32_t n, const int32_t* __restrict__ cand, int32_t* __restrict__ mate,
                                int32_t* __restrict__ added) {
    const int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    int32_t hit = 0;
    if (u < n && mate[u] < 0) {
        const int32_t v = cand[u];
        if (v >= 0 && cand[v] == u) {
            mate[u] = v;
            hit = 1;
        }
    }
    hit = __reduce_add_sync(0xffffffffu, hit);
    if ((threadIdx.x & 31) == 0 && hit) atomicAdd(added, hit);
}

__global__ void k_leader_flag(int32_t n, const int32_t* __restrict__ mate, int32_t* __restrict__ flag) {
    const int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n) return;
    const int32_t m = mate[u];
    flag[u] = (m < 0 || u < m) ? 1 : 0;
}

// cid = exclusive scan of flags; parent[u] = cid[leader(u)]; leader_of[p]; c'
__global__ void k_parent(int32_t n, const int32_t* __restrict__ mate, const int32_t* __restrict__ cid,
                         const int32_t* __restrict__ c, int32_t* __restrict__ parent, int32_t* __restrict__ c_next) {
    const int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n) return;
    const int32_t m = mate[u];
    const int32_t lead = (m >= 0 && m < u) ? m : u;
    const int32_t p = cid[lead];
    parent[u] = p;
    if (lead == u) c_next[p] = c[u] + (m >= 0 ? c[m] : 0);
}

// keys (parent[u] * nc + parent[v]) for crossing entries; intra-cluster -> sentinel nc*nc
// (one warp per row: coarse Chung-Lu levels have rows of 10^4-10^5 entries)
// row id of every CSR entry: one warp per row writes u over [rp[u], rp[u+1])
// (stores only, so heavy rows cost little)
__global__ void k_row_ids(int32_t n, const int64_t* __restrict__ rp, int32_t* __restrict__ row) {
    const int32_t u = (int32_t)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (u >= n) return;
    const int64_t e1 = rp[u + 1];
    for (int64_t e = rp[u] + lane; e < e1; e += 32) row[e] = u;
}

// edge-parallel: key = parent(u) * nc + parent(v) for crossing entries, sentinel nc^2 otherwise
__global__ void k_edge_keys(int64_t m, const int32_t* __restrict__ row, const int32_t* __restrict__ col,
                            const int32_t* __restrict__ omega, const int32_t* __restrict__ parent, int64_t nc,
                            uint64_t* __restrict__ keys, int32_t* __restrict__ vals) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m) return;
    const int64_t pu = __ldg(parent + __ldg(row + e)), pv = __ldg(parent + __ldg(col + e));
    keys[e] = (pu != pv) ? (uint64_t)(pu * nc + pv) : (uint64_t)(nc * nc);
    vals[e] = omega ? __ldg(omega + e) : 1;
}

__global__ void k_run_heads(int64_t m, const uint64_t* __restrict__ keys, uint64_t sentinel, int32_t* __restrict__ head) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m) return;
    const uint64_t k = keys[t];
    head[t] = (k != sentinel && (t == 0 || keys[t - 1] != k)) ? 1 : 0;
}

// for each run head: write coarse col / omega (sum over the run) and the row id
__global__ void k_run_emit(int64_t m, const uint64_t* __restrict__ keys, const int32_t* __restrict__ vals,
                           const int32_t* __restrict__ head, const int32_t* __restrict__ pos, int64_t nc,
                           int32_t* __restrict__ ccol, int32_t* __restrict__ comega, int32_t* __restrict__ urow) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= m || !head[t]) return;
    const uint64_t k = keys[t];
    int32_t s = 0;
    for (int64_t r = t; r < m && keys[r] == k; ++r) s += vals[r];
    const int32_t p = pos[t];
    ccol[p] = (int32_t)(k % (uint64_t)nc);
    comega[p] = s;
    urow[p] = (int32_t)(k / (uint64_t)nc);
}

// row_ptr[p] = first unique entry with row >= p (binary search; no atomics)
__global__ void k_rowptr_search(int32_t nc, const int32_t* __restrict__ urow, int64_t m2, int64_t* __restrict__ rp) {
    const int32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p > nc) return;
    int64_t lo = 0, hi = m2;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (urow[mid] < p) lo = mid + 1; else hi = mid;
    }
    rp[p] = lo;
}

// coarse S^l = E^l (Q7), edge-parallel over the m2 unique entries: d = s(c_u) + s(c_v),
// s(c) = c^(1/dim), w = d^-2
__global__ void k_coarse_sset(int64_t m, const int32_t* __restrict__ urow, const int32_t* __restrict__ col,
                              const int32_t* __restrict__ c, int dim, float* __restrict__ d, float* __restrict__ w) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= m) return;
    const float cu = (float)__ldg(c + __ldg(urow + e)), cv = (float)__ldg(c + __ldg(col + e));
    const float su = dim == 2 ? sqrtf(cu) : cbrtf(cu);
    const float sv = dim == 2 ? sqrtf(cv) : cbrtf(cv);
    const float dd = su + sv;
    d[e] = dd;
    w[e] = 1.0f / (dd * dd);
}

__global__ void k_iota(int32_t n, int32_t* __restrict__ a) {
    const int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) a[t] = t;
}

__global__ void k_fill_i32(int64_t n, int32_t v, int32_t* __restrict__ a) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) a[t] = v;
}

__global__ void k_count(int32_t n, const int32_t* __restrict__ key, int32_t* __restrict__ cnt) {
    const int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) atomicAdd(cnt + key[t], 1);
}

__global__ void k_compose(int32_t n, const int32_t* __restrict__ a, const int32_t* __restrict__ map,
                          int32_t* __restrict__ out) {
    const int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) out[t] = map[a[t]];
}

// Representative x'_v' = unweighted mean of the members (Q11),
// accumulated in FP64 and stored as hi + lo floats (hi = fl32(mean),
// lo = fl32(mean - hi)); rep_hi.w = nu(v') (Q10).  G lanes per
// representative (G from the mean cluster size: 2 at h = 2, 32 at h = 7):
// lane l sums members l, l+G, ... in order, then a fixed shuffle tree.
template <int DIM, int G>
// mem == nullptr: members are the contiguous ranges themselves (renumbered
// level, k_perm.cuh); sbound (nullable): the member range of each slot
__global__ void k_centroid(int32_t k, const int32_t* __restrict__ mptr, const int32_t* __restrict__ mem,
                           const float* __restrict__ x, const int32_t* __restrict__ rord,
                           const float4* __restrict__ frame, float4* __restrict__ rep_hi,
                           float4* __restrict__ rep_lo, const int2* __restrict__ sbound) {
    const int64_t tg = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int32_t slot = (int32_t)(tg / G);
    const int lg = (int)(tg & (G - 1));
    double sx = 0.0, sy = 0.0, sz = 0.0;
    int32_t b = 0, e = 0;
    if (slot < k) {
        if (sbound != nullptr) {
            const int2 be = __ldg(sbound + slot);
            b = be.x;
            e = be.y;
        } else {
            const int32_t v = rord != nullptr ? __ldg(rord + slot) : slot;
            b = mptr[v];
            e = mptr[v + 1];
        }
        for (int32_t t = b + lg; t < e; t += G) {
            const float4 p = load_x<DIM>(x, mem != nullptr ? __ldg(mem + t) : t);
            sx += p.x;
            sy += p.y;
            sz += p.z;
        }
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
        sx += __shfl_xor_sync(0xffffffffu, sx, o, G);
        sy += __shfl_xor_sync(0xffffffffu, sy, o, G);
        if constexpr (DIM == 3) sz += __shfl_xor_sync(0xffffffffu, sz, o, G);
    }
    if (slot >= k || lg != 0) return;
    const double nu = (double)(e - b);
    // relative to the frame origin (Q28; exact FP64 subtraction of an FP32 value)
    const float4 f = frame != nullptr ? *frame : make_float4(0.f, 0.f, 0.f, 0.f);
    const double mx = sx / nu - (double)f.x, my = sy / nu - (double)f.y, mz = DIM == 3 ? sz / nu - (double)f.z : 0.0;
    const float hx = (float)mx, hy = (float)my, hz = (float)mz;
    rep_hi[slot] = make_float4(hx, hy, hz, (float)nu);
    rep_lo[slot] = make_float4((float)(mx - hx), (float)(my - hy), (float)(mz - hz), 0.f);
}

// ---- orders for kernel (c) (Q26/Q27), computed once per level -----
// float <-> order-preserving unsigned (for atomic min/max of a bounding box)
__device__ __forceinline__ uint32_t f2ord(float f) {
    const uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}
__global__ void k_box_init(uint32_t* box) {
    if (threadIdx.x < 3) box[threadIdx.x] = 0xffffffffu;
    else if (threadIdx.x < 8) box[threadIdx.x] = 0u;  // [6]: ticket of k_frame_fused
}
template <int DIM>
__global__ void k_bbox(int32_t n, const float* __restrict__ x, uint32_t* __restrict__ box) {
    float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const float4 p = load_x<DIM>(x, i);
        const float v[3] = {p.x, p.y, p.z};
#pragma unroll
        for (int c = 0; c < DIM; ++c) {
            mn[c] = fminf(mn[c], v[c]);
            mx[c] = fmaxf(mx[c], v[c]);
        }
    }
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mn[c] = fminf(mn[c], __shfl_xor_sync(0xffffffffu, mn[c], o));
            mx[c] = fmaxf(mx[c], __shfl_xor_sync(0xffffffffu, mx[c], o));
        }
        if ((threadIdx.x & 31) == 0 && mn[c] <= mx[c]) {  // min/max: order-independent, deterministic
            atomicMin(box + c, f2ord(mn[c]));
            atomicMax(box + 3 + c, f2ord(mx[c]));
        }
    }
}
// Frame origin c (Q28): per axis, a float c with c/2 <= x <= 2c (or 2c <= x <= c/2)
// for every coordinate of the box, so that x - c is exact in FP32 (Sterbenz);
// 0 when no such c exists (a box that reaches 0 or spans a factor > 3)
template <int DIM>
__global__ void k_frame(const uint32_t* __restrict__ box, float4* __restrict__ frame) {
    if (threadIdx.x != 0) return;
    float c[3] = {0.f, 0.f, 0.f};
    for (int a = 0; a < DIM; ++a) {
        const float lo = ord2f(box[a]), hi = ord2f(box[3 + a]);
        if (!(lo <= hi)) continue;  // empty or non-finite box
        const float m = 0.5f * lo + 0.5f * hi;
        const bool ok = (lo > 0.f && 0.5f * m <= lo && hi <= 2.0f * m) || (hi < 0.f && 0.5f * m >= hi && lo >= 2.0f * m);
        c[a] = ok ? m : 0.f;
    }
    *frame = make_float4(c[0], c[1], c[2], 0.f);
}
__device__ __forceinline__ uint32_t spread2(uint32_t v) {  // 16 bits -> even bits
    v &= 0xffffu;
    v = (v | (v << 8)) & 0x00ff00ffu;
    v = (v | (v << 4)) & 0x0f0f0f0fu;
    v = (v | (v << 2)) & 0x33333333u;
    v = (v | (v << 1)) & 0x55555555u;
    return v;
}
__device__ __forceinline__ uint32_t spread3(uint32_t v) {  // 10 bits -> every third bit
    v &= 0x3ffu;
    v = (v | (v << 16)) & 0x030000ffu;
    v = (v | (v << 8)) & 0x0300f00fu;
    v = (v | (v << 4)) & 0x030c30c3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}
// Morton (Z-order) key of p quantised to the box: 16 bits per axis (2-D), 10 (3-D)
template <int DIM>
__device__ __forceinline__ uint32_t morton_key(const float4& p, const uint32_t* box) {
    const int B = DIM == 2 ? 16 : 10;
    const float cells = (float)(1u << B);
    const float v[3] = {p.x, p.y, p.z};
    uint32_t q[3] = {0, 0, 0};
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
        const float lo = ord2f(box[c]), hi = ord2f(box[3 + c]);
        const float ext = hi - lo;
        float t = ext > 0.f ? (v[c] - lo) / ext * cells : 0.f;
        t = fminf(fmaxf(t, 0.f), cells - 1.f);
        q[c] = (uint32_t)t;  // NaN -> 0
    }
    return DIM == 2 ? (spread2(q[0]) | (spread2(q[1]) << 1))
                    : (spread3(q[0]) | (spread3(q[1]) << 1) | (spread3(q[2]) << 2));
}
template <int DIM>
__global__ void k_target_keys(int32_t n, const float* __restrict__ x, const uint32_t* __restrict__ box,
                              uint32_t* __restrict__ key) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) key[i] = morton_key<DIM>(load_x<DIM>(x, i), box);
}
// bounding box + frame origin in one launch: per-block min/max -> atomics on box;
// the last block (ticket box[6]) derives the frame and re-arms box / ticket for
// the next launch (box must be armed once by k_box_init)
template <int DIM>
__global__ void k_frame_fused(int32_t n, const float* __restrict__ x, uint32_t* __restrict__ box,
                              float4* __restrict__ frame) {
    float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const float4 p = load_x<DIM>(x, i);
        const float v[3] = {p.x, p.y, p.z};
#pragma unroll
        for (int c = 0; c < DIM; ++c) {
            mn[c] = fminf(mn[c], v[c]);
            mx[c] = fmaxf(mx[c], v[c]);
        }
    }
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mn[c] = fminf(mn[c], __shfl_xor_sync(0xffffffffu, mn[c], o));
            mx[c] = fmaxf(mx[c], __shfl_xor_sync(0xffffffffu, mx[c], o));
        }
        if ((threadIdx.x & 31) == 0 && mn[c] <= mx[c]) {
            atomicMin(box + c, f2ord(mn[c]));
            atomicMax(box + 3 + c, f2ord(mx[c]));
        }
    }
    __threadfence();
    __syncthreads();
    __shared__ bool last;
    if (threadIdx.x == 0) last = atomicAdd(box + 6, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last || threadIdx.x != 0) return;
    __threadfence();
    uint32_t b[6];
    for (int c = 0; c < 6; ++c) b[c] = atomicAdd(box + c, 0u);  // coherent reads
    float cc[3] = {0.f, 0.f, 0.f};
    for (int a = 0; a < DIM; ++a) {
        const float lo = ord2f(b[a]), hi = ord2f(b[3 + a]);
        if (!(lo <= hi)) continue;
        const float m = 0.5f * lo + 0.5f * hi;
        const bool ok = (lo > 0.f && 0.5f * m <= lo && hi <= 2.0f * m) || (hi < 0.f && 0.5f * m >= hi && lo >= 2.0f * m);
        cc[a] = ok ? m : 0.f;
    }
    *frame = make_float4(cc[0], cc[1], cc[2], 0.f);
    for (int c = 0; c < 3; ++c) {
        box[c] = 0xffffffffu;
        box[3 + c] = 0u;
    }
    box[6] = 0u;
}
// representative keys from its (frame-relative) centroid
template <int DIM>
__global__ void k_rep_keys_c(int32_t k, const int32_t* __restrict__ mptr, const float4* __restrict__ rep_hi,
                             const float4* __restrict__ frame, const uint32_t* __restrict__ box,
                             uint64_t* __restrict__ key) {
    const int32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= k) return;
    const float4 f = *frame, h = rep_hi[v];
    const float4 p = make_float4(h.x + f.x, h.y + f.y, h.z + f.z, 0.f);
    key[v] = ((uint64_t)(uint32_t)(mptr[v + 1] - mptr[v]) << 32) | morton_key<DIM>(p, box);
}
// rpos = inverse of rord; tile_nu[t] = the common mass of slots [tile t, tile t + tile - 1] or 0
// sbound (nullable): member range [mptr[r], mptr[r+1]) of the rep at each slot, so
// that the centroid refresh reads it coalesced
__global__ void k_rep_slots(int32_t k, const int32_t* __restrict__ rord, const uint64_t* __restrict__ key_sorted,
                            int32_t* __restrict__ rpos, int32_t* __restrict__ tile_nu, int tile,
                            const int32_t* __restrict__ mptr, int2* __restrict__ sbound) {
    const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= k) return;
    const int32_t r = rord[s];
    rpos[r] = s;
    if (sbound != nullptr) sbound[s] = make_int2(mptr[r], mptr[r + 1]);
    if (s % tile == 0) {
        const int32_t last = min(s + tile - 1, k - 1);
        const uint32_t a = (uint32_t)(key_sorted[s] >> 32), b = (uint32_t)(key_sorted[last] >> 32);
        tile_nu[s / tile] = a == b ? (int32_t)a : 0;
    }
}
__global__ void k_scatter_inv(int32_t n, const int32_t* __restrict__ perm, int32_t* __restrict__ inv) {
    const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s < n) inv[perm[s]] = s;
}
// per source tile of kernel (c): box of the representatives' hi coordinates
// {min x, min y, min z, max |coordinate|}, {max x, max y, max z, 0}
template <int DIM>
__global__ void k_tile_box(int32_t k, const float4* __restrict__ rep_hi, float4* __restrict__ tile_box) {
    const int32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
    if (s < k) {
        const float4 p = rep_hi[s];
        mn[0] = mx[0] = p.x;
        mn[1] = mx[1] = p.y;
        if (DIM == 3) mn[2] = mx[2] = p.z;
    }
    __shared__ float red[8][6];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mn[c] = fminf(mn[c], __shfl_xor_sync(0xffffffffu, mn[c], o));
            mx[c] = fmaxf(mx[c], __shfl_xor_sync(0xffffffffu, mx[c], o));
        }
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        for (int c = 0; c < 3; ++c) {
            red[w][c] = mn[c];
            red[w][3 + c] = mx[c];
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int ww = 1; ww < (int)(blockDim.x >> 5); ++ww)
            for (int c = 0; c < 3; ++c) {
                red[0][c] = fminf(red[0][c], red[ww][c]);
                red[0][3 + c] = fmaxf(red[0][3 + c], red[ww][3 + c]);
            }
        float X = 0.f;
        for (int c = 0; c < DIM; ++c) X = fmaxf(X, fmaxf(fabsf(red[0][c]), fabsf(red[0][3 + c])));
        if (DIM == 2) red[0][2] = red[0][5] = 0.f;
        tile_box[2 * blockIdx.x] = make_float4(red[0][0], red[0][1], red[0][2], X);
        tile_box[2 * blockIdx.x + 1] = make_float4(red[0][3], red[0][4], red[0][5], 0.f);
    }
}

template <int DIM>
__global__ void k_prolong(int32_t n, const int32_t* __restrict__ parent, const float* __restrict__ xc,
                          uint64_t seed, int32_t level, float* __restrict__ x) {
    const int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n) return;
    const float4 pc = load_x<DIM>(xc, parent[u]);
    const uint64_t k0 = mix64(mix64(seed ^ kTagJitter) ^ (uint64_t)level);
    float o[3];
    const float pv[3] = {pc.x, pc.y, pc.z};
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
        const float U = uniform24(mix64(k0 ^ ((uint64_t)u * DIM + c)));
        o[c] = pv[c] + 1e-3f * (2.0f * U - 1.0f);
    }
    store_x<DIM>(x, u, make_float4(o[0], o[1], DIM == 3 ? o[2] : 0.f, 0.f));
}

template <int DIM>
__global__ void k_init_box(int32_t n, const double* __restrict__ dsum, int64_t nnz, uint64_t seed, int32_t level,
                           float* __restrict__ x) {
    const int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n) return;
    const double dbar = nnz > 0 ? *dsum / (double)nnz : 1.0;
    const float box = (float)(dbar * (DIM == 2 ? sqrt((double)n) : cbrt((double)n)));
    const uint64_t k0 = mix64(mix64(seed ^ kTagInit) ^ (uint64_t)level);
    float o[3];
#pragma unroll
    for (int c = 0; c < DIM; ++c) o[c] = box * uniform24(mix64(k0 ^ ((uint64_t)u * DIM + c)));
    store_x<DIM>(x, u, make_float4(o[0], o[1], DIM == 3 ? o[2] : 0.f, 0.f));
}

// ---- label-based contraction (SCLaP, R6): coarse id = rank of the distinct labels
__global__ void k_label_flags(int32_t n, const int32_t* __restrict__ lab, int32_t* __restrict__ flag) {
    const int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u < n) flag[lab[u]] = 1;  // benign race: every writer stores 1
}
__global__ void k_label_parent(int32_t n, const int32_t* __restrict__ lab, const int32_t* __restrict__ cid,
                               const int32_t* __restrict__ c, int32_t* __restrict__ parent,
                               int32_t* __restrict__ c_next) {
    const int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n) return;
    const int32_t p = cid[lab[u]];
    parent[u] = p;
    atomicAdd(c_next + p, c[u]);  // integer: order-free
}

// the paper's disc prolongation (reading R7): angle U0 * 2pi, radius
// c(v')^(1/dim) * U1; dim 3 direction from z = 2 U2 - 1
template <int DIM>
__global__ void k_prolong_disc(int32_t n, const int32_t* __restrict__ parent, const float* __restrict__ xc,
                               const int32_t* __restrict__ c_coarse, uint64_t seed, int32_t level,
                               float* __restrict__ x) {
    const int32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n) return;
    const int32_t p = parent[u];
    const float4 pc = load_x<DIM>(xc, p);
    const uint64_t k0 = mix64(mix64(seed ^ kTagDisc) ^ (uint64_t)level);
    const float U0 = uniform24(mix64(k0 ^ ((uint64_t)u * 3 + 0)));
    const float U1 = uniform24(mix64(k0 ^ ((uint64_t)u * 3 + 1)));
    const float U2 = uniform24(mix64(k0 ^ ((uint64_t)u * 3 + 2)));
    const float cp = (float)c_coarse[p];
    const float r = (DIM == 2 ? sqrtf(cp) : cbrtf(cp)) * U1;
    float sn, cs;
    sincosf(6.28318530717958647692f * U0, &sn, &cs);
    if (DIM == 2) {
        store_x<DIM>(x, u, make_float4(pc.x + r * cs, pc.y + r * sn, 0.f, 0.f));
    } else {
        const float z = 2.0f * U2 - 1.0f, sz = sqrtf(fmaxf(0.f, 1.0f - z * z));
        store_x<DIM>(x, u, make_float4(pc.x + r * sz * cs, pc.y + r * sz * sn, pc.z + r * z, 0.f));
    }
}

__global__ void k_max_i32(int32_t n, const int32_t* __restrict__ a, int32_t* __restrict__ out) {
    int32_t m = 0;
    for (int32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) m = max(m, a[t]);
    m = __reduce_max_sync(0xffffffffu, m);
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// FP64 sum of a float array (one block, fixed order)
__global__ void k_sum_f32(int64_t m, const float* __restrict__ a, double* __restrict__ out) {
    __shared__ double red[32];
    double s = 0.0;
    for (int64_t t = threadIdx.x; t < m; t += blockDim.x) s += (double)a[t];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        *out = t;
    }
}

inline int nblk(int64_t n, int b = 256) { return (int)((n + b - 1) / b); }

// lanes per vertex for the matching scan: about 2 row entries per lane
// (MM_MATCH_G overrides, experiments)
int match_group(int32_t n, int64_t nnz) {
    static const int forced = [] {
        const char* e = getenv("MM_MATCH_G");
        return e ? atoi(e) : 0;
    }();
    if (forced == 2 || forced == 4 || forced == 8 || forced == 16 || forced == 32) return forced;
    const double mean = n > 0 ? (double)nnz / n : 0.0;
    int g = 2;
    while (g < 32 && 2.0 * (2 * g) <= mean) g *= 2;
    return g;
}

}  // namespace

// ------------------------------------------------------------------ host side

cudaError_t run_match_round(int32_t n, int64_t nnz, const int64_t* rp, const int32_t* col, const int32_t* omega,
                            const int32_t* c, int32_t* mate, int32_t* cand, uint64_t seed, int32_t level,
                            int32_t round, int32_t* added, cudaStream_t st) {
    {
        LaunchScope ls("match_pick", st);
        const int G = match_group(n, nnz);
        const int nb = nblk((int64_t)n * G);
        switch (G) {
            case 2: k_match_pick<2><<<nb, 256, 0, st>>>(n, rp, col, omega, c, mate, cand, seed, level, round); break;
            case 4: k_match_pick<4><<<nb, 256, 0, st>>>(n, rp, col, omega, c, mate, cand, seed, level, round); break;
            case 8: k_match_pick<8><<<nb, 256, 0, st>>>(n, rp, col, omega, c, mate, cand, seed, level, round); break;
            case 16: k_match_pick<16><<<nb, 256, 0, st>>>(n, rp, col, omega, c, mate, cand, seed, level, round); break;
            default: k_match_pick<32><<<nb, 256, 0, st>>>(n, rp, col, omega, c, mate, cand, seed, level, round); break;
        }
    }
    {
        LaunchScope ls("match_confirm", st);
        k_match_confirm<<<nblk(n), 256, 0, st>>>(n, cand, mate, added);
    }
    return cudaGetLastError();
}

template <int G>
cudaError_t match_level_t(int32_t n, const int64_t* rp, const int32_t* col, const int32_t* omega, const int32_t* c,
                          int32_t* mate, int32_t* cand, uint64_t seed, int32_t level, int32_t max_rounds,
                          int32_t* added, int32_t* rounds_out, cudaStream_t st) {
    static const int grid = [] {
        int dev = 0, sms = 148, occ = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_match_level<G>, 256, 0);
        return sms * std::max(occ, 1);
    }();
    void* params[] = {&n, &rp, &col, &omega, &c, &mate, &cand, &seed, &level, &max_rounds, &added, &rounds_out};
    return cudaLaunchCooperativeKernel((const void*)k_match_level<G>, dim3(grid), dim3(256), params, 0, st);
}

cudaError_t run_match_level(int32_t n, int64_t nnz, const int64_t* rp, const int32_t* col, const int32_t* omega,
                            const int32_t* c, int32_t* mate, int32_t* cand, uint64_t seed, int32_t level,
                            int32_t max_rounds, int32_t* added, int32_t* rounds_out, cudaStream_t st) {
    LaunchScope ls("match_level", st);
    cudaError_t e = cudaMemsetAsync(added, 0, 2 * sizeof(int32_t), st);
    if (e != cudaSuccess) return e;
    switch (match_group(n, nnz)) {
        case 2: return match_level_t<2>(n, rp, col, omega, c, mate, cand, seed, level, max_rounds, added, rounds_out, st);
        case 4: return match_level_t<4>(n, rp, col, omega, c, mate, cand, seed, level, max_rounds, added, rounds_out, st);
        case 8: return match_level_t<8>(n, rp, col, omega, c, mate, cand, seed, level, max_rounds, added, rounds_out, st);
        case 16: return match_level_t<16>(n, rp, col, omega, c, mate, cand, seed, level, max_rounds, added, rounds_out, st);
        default: return match_level_t<32>(n, rp, col, omega, c, mate, cand, seed, level, max_rounds, added, rounds_out, st);
    }
}

cudaError_t launch_fill(int64_t n, int32_t v, int32_t* a, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    LaunchScope ls("fill", st);
    k_fill_i32<<<nblk(n), 256, 0, st>>>(n, v, a);
    return cudaGetLastError();
}

// scratch of the hand-written scan / sort (k_perm.cu, k_sort.cu) used below
size_t scan_temp_bytes(int32_t n) { return perm_scan_tmp_bytes((int64_t)n + 1); }

size_t sort_temp_bytes_u64(int64_t m) { return radix_sort_tmp_bytes<uint64_t>(m); }

size_t sort_temp_bytes_i32(int32_t n) { return radix_sort_tmp_bytes<uint32_t>(n); }

// exclusive sum of n items (out[0..n-1]), as the scans of the contraction need
cudaError_t exclusive_scan_i32(const int32_t* in, int32_t* out, int32_t n, void* tmp, size_t tmp_bytes,
                               cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    if (tmp_bytes < perm_scan_tmp_bytes(n)) return cudaErrorInvalidValue;
    return scan_i32_excl<int32_t>(in, out, (int64_t)n - 1, tmp, st);
}

cudaError_t contract_leaders(int32_t n, const int32_t* mate, const int32_t* c, int32_t* flag, int32_t* cid,
                             int32_t* parent, int32_t* c_next, void* tmp, size_t tmp_bytes, cudaStream_t st) {
    {
        LaunchScope ls("leader_flag", st);
        k_leader_flag<<<nblk(n), 256, 0, st>>>(n, mate, flag);
    }
    cudaError_t e = exclusive_scan_i32(flag, cid, n, tmp, tmp_bytes, st);
    if (e != cudaSuccess) return e;
    LaunchScope ls("parent", st);
    k_parent<<<nblk(n), 256, 0, st>>>(n, mate, cid, c, parent, c_next);
    return cudaGetLastError();
}

cudaError_t contract_edges(int32_t n, int64_t nnz, const int64_t* rp, const int32_t* col, const int32_t* omega,
                           const int32_t* parent, int32_t nc, uint64_t* keys, uint64_t* keys_alt, int32_t* vals,
                           int32_t* vals_alt, int32_t* head, int32_t* pos, int32_t* ccol_tmp,
                           int32_t* comega_tmp, int32_t* rowcnt, void* tmp, size_t tmp_bytes, cudaStream_t st) {
    cudaError_t e;
    {
        // head is free until run_heads: it carries the row id of every entry
        LaunchScope ls("row_ids", st);
        k_row_ids<<<nblk((int64_t)n * 32), 256, 0, st>>>(n, rp, head);
    }
    {
        LaunchScope ls("edge_keys", st);
        k_edge_keys<<<nblk(nnz), 256, 0, st>>>(nnz, head, col, omega, parent, nc, keys, vals);
    }
    const uint64_t sentinel = (uint64_t)nc * (uint64_t)nc;
    int end_bit = 1;
    while (end_bit < 64 && (sentinel >> end_bit) != 0) ++end_bit;
    e = radix_sort_pairs<uint64_t>(keys, keys_alt, vals, vals_alt, nnz, 0, end_bit, tmp, tmp_bytes, st, "sort_edges");
    if (e != cudaSuccess) return e;
    {
        LaunchScope ls("run_heads", st);
        k_run_heads<<<nblk(nnz), 256, 0, st>>>(nnz, keys_alt, sentinel, head);
    }
    e = exclusive_scan_i32(head, pos, (int32_t)nnz, tmp, tmp_bytes, st);
    if (e != cudaSuccess) return e;
    (void)rowcnt;
    LaunchScope ls("run_emit", st);
    // vals (pre-sort values) is dead after the sort: reuse it for the row ids
    k_run_emit<<<nblk(nnz), 256, 0, st>>>(nnz, keys_alt, vals_alt, head, pos, nc, ccol_tmp, comega_tmp, vals);
    return cudaGetLastError();
}

cudaError_t rowptr_from_rows(int32_t nc, const int32_t* urow, int64_t m2, int64_t* rp, cudaStream_t st) {
    LaunchScope ls("rowptr", st);
    k_rowptr_search<<<nblk((int64_t)nc + 1), 256, 0, st>>>(nc, urow, m2, rp);
    return cudaGetLastError();
}

cudaError_t launch_coarse_sset(int64_t m, const int32_t* urow, const int32_t* col, const int32_t* c, int dim,
                               float* d, float* w, cudaStream_t st) {
    if (m <= 0) return cudaSuccess;
    LaunchScope ls("coarse_sset", st);
    k_coarse_sset<<<nblk(m), 256, 0, st>>>(m, urow, col, c, dim, d, w);
    return cudaGetLastError();
}

cudaError_t group_by_key(int32_t n, const int32_t* key, int32_t k, int32_t* ptr, int32_t* members,
                         int32_t* key_sorted, int32_t* iota, int32_t* cnt, void* tmp, size_t tmp_bytes,
                         cudaStream_t st) {
    cudaError_t e;
    {
        LaunchScope ls("iota", st);
        k_iota<<<nblk(n), 256, 0, st>>>(n, iota);
    }
    int end_bit = 1;
    while (end_bit < 31 && ((k - 1) >> end_bit) != 0) ++end_bit;
    // keys are non-negative ids < k: sorted as unsigned
    e = radix_sort_pairs<uint32_t>(reinterpret_cast<const uint32_t*>(key), reinterpret_cast<uint32_t*>(key_sorted), iota,
                                   members, n, 0, end_bit, tmp, tmp_bytes, st, "sort_group");
    if (e != cudaSuccess) return e;
    e = launch_fill(k + 1, 0, cnt, st);
    if (e != cudaSuccess) return e;
    {
        LaunchScope ls("count", st);
        k_count<<<nblk(n), 256, 0, st>>>(n, key, cnt);
    }
    // exclusive scan over k+1 entries: ptr[k] = n
    return exclusive_scan_i32(cnt, ptr, k + 1, tmp, tmp_bytes, st);
}

cudaError_t launch_compose(int32_t n, const int32_t* a, const int32_t* map, int32_t* out, cudaStream_t st) {
    LaunchScope ls("compose", st);
    k_compose<<<nblk(n), 256, 0, st>>>(n, a, map, out);
    return cudaGetLastError();
}

cudaError_t launch_frame_fused(int dim, int32_t n, const float* x, uint32_t* box, float4* frame, cudaStream_t st) {
    LaunchScope ls("frame", st);
    const int nb = std::max(1, std::min(nblk(n), 2 * 148));
    if (dim == 2) k_frame_fused<2><<<nb, 256, 0, st>>>(n, x, box, frame);
    else k_frame_fused<3><<<nb, 256, 0, st>>>(n, x, box, frame);
    return cudaGetLastError();
}

cudaError_t launch_frame(int dim, int32_t n, const float* x, uint32_t* box, float4* frame, cudaStream_t st) {
    LaunchScope ls("frame", st);
    k_box_init<<<1, 32, 0, st>>>(box);
    const int nb = std::max(1, std::min(nblk(n), 4 * 148));
    if (dim == 2) {
        k_bbox<2><<<nb, 256, 0, st>>>(n, x, box);
        k_frame<2><<<1, 32, 0, st>>>(box, frame);
    } else {
        k_bbox<3><<<nb, 256, 0, st>>>(n, x, box);
        k_frame<3><<<1, 32, 0, st>>>(box, frame);
    }
    return cudaGetLastError();
}

cudaError_t approx_orders(int dim, int32_t n, int32_t k, const int32_t* mptr, const int32_t* mem, const float* x,
                          int tile, const int32_t* iota, uint32_t* box, float4* frame, float4* rep_hi,
                          float4* rep_lo, uint32_t* tkey, uint32_t* tkey_sorted, int32_t* tperm, int32_t* tpos,
                          uint64_t* rkey, uint64_t* rkey_sorted, int32_t* rord, int32_t* rpos, int32_t* tile_nu,
                          void* tmp, size_t tmp_bytes, cudaStream_t st, int2* sbound) {
    if (k <= 0 || n <= 0) return cudaSuccess;
    cudaError_t e = launch_frame(dim, n, x, box, frame, st);
    if (e != cudaSuccess) return e;
    // centroids by representative id (the sort keys); the sweep rewrites them by slot
    e = launch_centroid(dim, n, k, mptr, mem, x, nullptr, frame, rep_hi, rep_lo, nullptr, tile, st, nullptr,
                        "centroid_keys");
    if (e != cudaSuccess) return e;
    {
        LaunchScope ls("order_keys", st);
        if (dim == 2) {
            k_target_keys<2><<<nblk(n), 256, 0, st>>>(n, x, box, tkey);
            k_rep_keys_c<2><<<nblk(k), 256, 0, st>>>(k, mptr, rep_hi, frame, box, rkey);
        } else {
            k_target_keys<3><<<nblk(n), 256, 0, st>>>(n, x, box, tkey);
            k_rep_keys_c<3><<<nblk(k), 256, 0, st>>>(k, mptr, rep_hi, frame, box, rkey);
        }
    }
    // stable: equal keys keep id order
    e = radix_sort_pairs<uint32_t>(tkey, tkey_sorted, iota, tperm, n, 0, 32, tmp, tmp_bytes, st, "sort_order");
    if (e != cudaSuccess) return e;
    e = radix_sort_pairs<uint64_t>(rkey, rkey_sorted, iota, rord, k, 0, 64, tmp, tmp_bytes, st, "sort_order");
    if (e != cudaSuccess) return e;
    LaunchScope ls("order_slots", st);
    k_scatter_inv<<<nblk(n), 256, 0, st>>>(n, tperm, tpos);
    k_rep_slots<<<nblk(k), 256, 0, st>>>(k, rord, rkey_sorted, rpos, tile_nu, tile, mptr, sbound);
    k_box_init<<<1, 32, 0, st>>>(box);  // armed for launch_frame_fused
    return cudaGetLastError();
}

cudaError_t launch_centroid(int dim, int32_t n, int32_t k, const int32_t* mptr, const int32_t* mem, const float* x,
                            const int32_t* rord, const float4* frame, float4* rep_hi, float4* rep_lo,
                            float4* tile_box, int tile, cudaStream_t st, const int2* sbound, const char* name) {
    if (tile_box != nullptr && k > 0) {
        const cudaError_t e = launch_centroid(dim, n, k, mptr, mem, x, rord, frame, rep_hi, rep_lo, nullptr, tile,
                                              st, sbound, name);
        if (e != cudaSuccess) return e;
        LaunchScope ls("tile_box", st);
        const int nt = (k + tile - 1) / tile;
        if (dim == 2) k_tile_box<2><<<nt, tile, 0, st>>>(k, rep_hi, tile_box);
        else k_tile_box<3><<<nt, tile, 0, st>>>(k, rep_hi, tile_box);
        return cudaGetLastError();
    }
    LaunchScope ls(name, st);
    // lanes per representative: about 4 members per lane
    const double mean = k > 0 ? (double)n / k : 1.0;
    int G = 1;
    while (G < 32 && 4.0 * (2 * G) <= mean) G *= 2;
    const int nb = nblk((int64_t)k * G);
#define MM_C(D)                                                                               \
    switch (G) {                                                                              \
        case 1: k_centroid<D, 1><<<nb, 256, 0, st>>>(k, mptr, mem, x, rord, frame, rep_hi, rep_lo, sbound); break;   \
        case 2: k_centroid<D, 2><<<nb, 256, 0, st>>>(k, mptr, mem, x, rord, frame, rep_hi, rep_lo, sbound); break;   \
        case 4: k_centroid<D, 4><<<nb, 256, 0, st>>>(k, mptr, mem, x, rord, frame, rep_hi, rep_lo, sbound); break;   \
        case 8: k_centroid<D, 8><<<nb, 256, 0, st>>>(k, mptr, mem, x, rord, frame, rep_hi, rep_lo, sbound); break;   \
        case 16: k_centroid<D, 16><<<nb, 256, 0, st>>>(k, mptr, mem, x, rord, frame, rep_hi, rep_lo, sbound); break; \
        default: k_centroid<D, 32><<<nb, 256, 0, st>>>(k, mptr, mem, x, rord, frame, rep_hi, rep_lo, sbound); break; \
    }
    if (dim == 2) { MM_C(2) } else { MM_C(3) }
#undef MM_C
    return cudaGetLastError();
}

cudaError_t launch_prolong(int dim, int32_t n, const int32_t* parent, const float* xc, uint64_t seed,
                           int32_t level, float* x, cudaStream_t st) {
    LaunchScope ls("prolong", st);
    if (dim == 2) k_prolong<2><<<nblk(n), 256, 0, st>>>(n, parent, xc, seed, level, x);
    else k_prolong<3><<<nblk(n), 256, 0, st>>>(n, parent, xc, seed, level, x);
    return cudaGetLastError();
}

cudaError_t launch_init_box(int dim, int32_t n, const float* d, int64_t nnz, double* dsum, uint64_t seed,
                            int32_t level, float* x, cudaStream_t st) {
    {
        LaunchScope ls("sum_d", st);
        k_sum_f32<<<1, 1024, 0, st>>>(nnz, d, dsum);
    }
    LaunchScope ls("init_box", st);
    if (dim == 2) k_init_box<2><<<nblk(n), 256, 0, st>>>(n, dsum, nnz, seed, level, x);
    else k_init_box<3><<<nblk(n), 256, 0, st>>>(n, dsum, nnz, seed, level, x);
    return cudaGetLastError();
}

}  // namespace mm

namespace mm {

cudaError_t contract_labels_gpu(int32_t n, const int32_t* lab, const int32_t* c, int32_t* flag, int32_t* cid,
                                int32_t* parent, int32_t* c_next, int32_t* nc_out_dev, void* tmp, size_t tmp_bytes,
                                cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(flag, 0, sizeof(int32_t) * ((size_t)n + 1), st);
    if (e != cudaSuccess) return e;
    {
        LaunchScope ls("label_flags", st);
        k_label_flags<<<nblk(n), 256, 0, st>>>(n, lab, flag);
    }
    // exclusive scan over n + 1 entries: cid[n] = number of clusters
    e = exclusive_scan_i32(flag, cid, n + 1, tmp, tmp_bytes, st);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(c_next, 0, sizeof(int32_t) * (size_t)n, st);
    if (e != cudaSuccess) return e;
    {
        LaunchScope ls("label_parent", st);
        k_label_parent<<<nblk(n), 256, 0, st>>>(n, lab, cid, c, parent, c_next);
    }
    return cudaMemcpyAsync(nc_out_dev, cid + n, sizeof(int32_t), cudaMemcpyDeviceToDevice, st);
}

cudaError_t launch_prolong_disc(int dim, int32_t n, const int32_t* parent, const float* xc, const int32_t* c_coarse,
                                uint64_t seed, int32_t level, float* x, cudaStream_t st) {
    LaunchScope ls("prolong_disc", st);
    if (dim == 2) k_prolong_disc<2><<<nblk(n), 256, 0, st>>>(n, parent, xc, c_coarse, seed, level, x);
    else k_prolong_disc<3><<<nblk(n), 256, 0, st>>>(n, parent, xc, c_coarse, seed, level, x);
    return cudaGetLastError();
}

cudaError_t launch_max_i32(int32_t n, const int32_t* a, int32_t* out, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(int32_t), st);
    if (e != cudaSuccess) return e;
    LaunchScope ls("max_c", st);
    k_max_i32<<<std::max(1, std::min(nblk(n), 1184)), 256, 0, st>>>(n, a, out);
    return cudaGetLastError();
}

}  // namespace mm
