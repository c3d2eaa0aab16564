// api.cu — the C-ABI of libmm_b200.so (include/mm.h): argument checks, the
// stream-ordered allocator hook, workspace layout, launch bookkeeping and the
// host drivers (mm_sweep, mm_energy, mm_build_hierarchy, mm_layout).
// Every step of the hot path runs in the kernels of k_repulse.cu, k_gather.cu
// and k_hier.cu; the host only sequences launches and reads sizes.
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "k_fullstress.cuh"
#include "k_hier.cuh"
#include "k_small.cuh"
#include "k_perm.cuh"
#include "k_sclap.cuh"
#include "k_repulse.cuh"

// ------------------------------------------------------------------ errors
namespace {
thread_local std::string g_err;

void set_err(const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
}

mm_status cuda_fail(cudaError_t e, const char* where) {
    set_err("%s: %s", where, cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? MM_ERR_OUT_OF_MEMORY : MM_ERR_CUDA;
}

#define MM_CU(expr, where)                              \
    do {                                                \
        cudaError_t _e = (expr);                        \
        if (_e != cudaSuccess) return cuda_fail(_e, where); \
    } while (0)

// ------------------------------------------------------------------ allocator
void* (*g_alloc)(size_t, mm_stream_t, void*) = nullptr;
void (*g_free)(void*, mm_stream_t, void*) = nullptr;
void* g_alloc_ctx = nullptr;

// Keep freed blocks in the device's stream-ordered pool (the default release
// threshold 0 returns them to the driver at every synchronisation, and the
// next cudaMallocAsync would map fresh pages).
void keep_pool_warm() {
    static const bool done = [] {
        int dev = 0;
        cudaMemPool_t pool;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        return true;
    }();
    (void)done;
    cudaGetLastError();
}

void* dev_alloc(size_t bytes, cudaStream_t st) {
    if (bytes == 0) bytes = 16;
    if (g_alloc) return g_alloc(bytes, (mm_stream_t)st, g_alloc_ctx);
    keep_pool_warm();
    void* p = nullptr;
    if (cudaMallocAsync(&p, bytes, st) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return p;
}
void dev_free(void* p, cudaStream_t st) {
    if (!p) return;
    if (g_free) g_free(p, (mm_stream_t)st, g_alloc_ctx);
    else cudaFreeAsync(p, st);
}

// A bump allocator over one device block (workspace carving, 256-B aligned).
struct Carver {
    char* base;
    size_t cap, off = 0;
    bool ok = true;
    Carver(void* b, size_t c) : base((char*)b), cap(c) {}
    template <class T>
    T* take(size_t count) {
        size_t bytes = ((count * sizeof(T)) + 255) & ~(size_t)255;
        if (off + bytes > cap) {
            ok = false;
            return nullptr;
        }
        T* p = reinterpret_cast<T*>(base + off);
        off += bytes;
        return p;
    }
};
size_t al(size_t bytes) { return (bytes + 255) & ~(size_t)255; }

struct DevBuf {
    void* p = nullptr;
    cudaStream_t st = nullptr;
    DevBuf() = default;
    DevBuf(size_t bytes, cudaStream_t s) : st(s) { p = dev_alloc(bytes, s); }
    ~DevBuf() { dev_free(p, st); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

// ------------------------------------------------------------------ host trace (MM_TRACE=1)
bool trace_on() {
    static const bool on = [] {
        const char* e = getenv("MM_TRACE");
        return e && e[0] && e[0] != '0';
    }();
    return on;
}
void trace(const char* what) {
    if (!trace_on()) return;
    static auto t0 = std::chrono::steady_clock::now();
    const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    fprintf(stderr, "[mm_trace %12.1f us] %s\n", us, what);
}

// ------------------------------------------------------------------ profiling
std::atomic<int64_t> g_launches{0};
std::atomic<int> g_prof_on{0};
std::mutex g_prof_mu;
struct PendingEv {
    const char* name;
    cudaEvent_t a, b;
};
std::vector<PendingEv> g_pending;
std::vector<cudaEvent_t> g_event_pool;  // reused timing events (creation is not free)
std::map<std::string, std::pair<int64_t, double>> g_prof;
std::vector<std::pair<const char*, float>> g_prof_list;  // every timed launch, in launch order

cudaEvent_t pool_get() {  // caller holds g_prof_mu
    if (!g_event_pool.empty()) {
        cudaEvent_t e = g_event_pool.back();
        g_event_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    return e;
}

}  // namespace

namespace mm {
LaunchScope::LaunchScope(const char* n, cudaStream_t s) : name(n), stream(s), slot(-1) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (!g_prof_on.load(std::memory_order_relaxed)) return;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return;
    std::lock_guard<std::mutex> g(g_prof_mu);
    PendingEv ev{n, pool_get(), pool_get()};
    if (!ev.a || !ev.b) return;
    cudaEventRecord(ev.a, s);
    g_pending.push_back(ev);
    slot = (int)g_pending.size() - 1;
}
LaunchScope::~LaunchScope() {
    if (slot < 0) return;
    std::lock_guard<std::mutex> g(g_prof_mu);
    if (slot < (int)g_pending.size()) cudaEventRecord(g_pending[slot].b, stream);
}
}  // namespace mm

using namespace mm;

// ------------------------------------------------------------------ helpers
namespace {

int stride_of(int dim) { return dim == 2 ? 2 : 4; }

mm_status check_sset(const mm_sset* S, const char* who) {
    if (!S) { set_err("%s: S is NULL", who); return MM_ERR_INVALID_ARGUMENT; }
    if (S->n <= 0) { set_err("%s: S->n must be > 0 (got %d)", who, S->n); return MM_ERR_INVALID_ARGUMENT; }
    if (S->nnz < 0) { set_err("%s: S->nnz < 0", who); return MM_ERR_INVALID_ARGUMENT; }
    if (!S->row_ptr || (S->nnz > 0 && (!S->col || !S->d || !S->w))) {
        set_err("%s: S has a NULL array", who);
        return MM_ERR_INVALID_ARGUMENT;
    }
    return MM_OK;
}

mm_status check_dim_q(int dim, double q, const char* who) {
    if (dim != 2 && dim != 3) { set_err("%s: dim must be 2 or 3 (got %d)", who, dim); return MM_ERR_UNSUPPORTED; }
    if (!(q >= 0.0) || !isfinite(q)) { set_err("%s: q must be finite and >= 0", who); return MM_ERR_UNSUPPORTED; }
    return MM_OK;
}

mm_status check_x(const float* x, int dim, const char* what, const char* who) {
    if (!x) { set_err("%s: %s is NULL", who, what); return MM_ERR_INVALID_ARGUMENT; }
    const uintptr_t a = dim == 2 ? 8 : 16;
    if (((uintptr_t)x) % a) { set_err("%s: %s must be %d-byte aligned", who, what, (int)a); return MM_ERR_INVALID_ARGUMENT; }
    return MM_OK;
}

// Buffers for one sweep (all device); sized by plan_sweep_bytes.
struct SweepBufs {
    float* part = nullptr;
    float* jpart = nullptr;  // symmetric exact mode: j-side sums [TB-1][n]
    double* stat_partial = nullptr;
    int32_t* flags = nullptr;
    float4* rep_hi = nullptr;
    float4* rep_lo = nullptr;
    int32_t* mptr = nullptr;
    int32_t* mem = nullptr;
    int32_t* cptr = nullptr;
    int32_t* child = nullptr;
    int32_t* key_sorted = nullptr;
    int32_t* iota = nullptr;
    int32_t* cnt = nullptr;
    int32_t* rord = nullptr;     // representatives in mass order (Q26): slot -> rep id
    int32_t* rpos = nullptr;     // rep id -> slot
    int32_t* tile_nu = nullptr;  // [ceil(k / kCoarseTile)] common mass of a tile, or 0
    int32_t* tperm = nullptr;    // targets in spatial order (Q27): slot -> vertex
    int32_t* tpos = nullptr;     // vertex -> slot
    float4* tile_box = nullptr;  // [2 ceil(k / kCoarseTile)] per-tile box of the representatives
    uint64_t* rkey = nullptr;    // [2k] representative sort keys (scratch)
    uint32_t* box = nullptr;     // [8] layout box (scratch)
    float4* frame = nullptr;     // [1] kernel (c)'s frame origin (Q28)
    int32_t* sib = nullptr;      // renumbered level: per-vertex sibling (k_perm.cuh), else NULL
    int2* sbound = nullptr;      // member range of the rep at each slot (written with the orders)
    bool contig = false;         // renumbered level: members of a rep are a contiguous range (mem = identity)
    bool reorder = false;        // recompute kernel (c)'s orders before every sweep
    bool far = false;            // kernel (c) with per-sweep frame and tile boxes (lo-free far tiles, Q27/Q28)
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
};

// scratch of the hand-written sorts / scans of one sweep's maps and orders
size_t cub_tmp_bytes(int32_t n) {
    return std::max({sort_temp_bytes_i32(n), sort_temp_bytes_u64(n), scan_temp_bytes(n + 2)}) + 256;
}

// Exact sweeps use the symmetric kernel (each unordered pair once)
// unless MM_SYM=0, its j-side buffer would exceed 2 GiB, or the triangular
// schedule has too few units per CTA; MM_SYM=2 forces it (tests).
bool use_sym(int32_t n, int dim) {
    static const int env = [] {
        const char* v = getenv("MM_SYM");
        return (v && v[0] == '0') ? 0 : (v && v[0] == '2') ? 2 : 1;  // 2: force (tests)
    }();
    if (!env) return false;
    const int64_t tb = (n + 1023) / 1024;
    if ((tb - 1) * (int64_t)n * stride_of(dim) * 4 > (int64_t(1) << 31)) return false;
    // the triangular schedule has 4 TB(TB+1)/2 units (block pair x source
    // sub-tile): with fewer units than CTAs part of the GPU idles and the
    // one-sided kernel is faster (measured: n = 16K already favours symmetric)
    const SymPlan sp = plan_repulse_sym(n, dim);
    return env == 2 || sp.ts.U >= sp.full_grid;
}

int part_slots(int32_t n, int dim, int32_t n_src, bool approx) {
    RepulsePlan p = plan_repulse(n, n_src, dim, approx, true);
    RepulsePlan p2 = plan_repulse(n, n_src, dim, approx, false);
    int slots = std::max(p.slots, p2.slots);
    if (!approx && use_sym(n, dim)) slots = std::max(slots, plan_repulse_sym(n, dim).slots);
    return slots;
}

// per-CTA FP64 partials: the gather's [blocks][3] (bound: G = 32) or the
// small-level kernel's [2][grid][4], whichever is larger
size_t stat_partial_doubles(int32_t n) {
    return std::max((size_t)gather_blocks(n, 1e9) * 3, (size_t)small_level_partials(n) * 4);
}

size_t sweep_bytes(int32_t n, int dim, int32_t k, bool approx, double mean_row) {
    const int32_t n_src = approx ? k : n;
    const int slots = part_slots(n, dim, n_src, approx);
    size_t b = al((size_t)slots * n * stride_of(dim) * sizeof(float));
    if (!approx && use_sym(n, dim))
        b += al((size_t)sym_jpart_rows(plan_repulse_sym(n, dim)) * n * stride_of(dim) * sizeof(float));
    (void)mean_row;
    b += al(stat_partial_doubles(n) * sizeof(double));
    b += al(sizeof(int32_t) * 4);
    if (approx) {
        b += 2 * al((size_t)k * sizeof(float4)) + al((size_t)(k + 1) * 4) + al((size_t)n * 4);
        b += al((size_t)(n + 1) * 4) + al((size_t)n * 4);
        b += al((size_t)n * 4) * 2 + al((size_t)(std::max(n, k) + 2) * 4);
        b += 2 * al((size_t)k * 4) + al((size_t)k * 8) + al((size_t)(k / kCoarseTile + 1) * 4);
        b += 2 * al((size_t)n * 4) + al((size_t)(k / kCoarseTile + 1) * 32) + al((size_t)k * 16) + al(32) + al(16);
        b += al(cub_tmp_bytes(n));
    }
    return b + 4096;
}

bool carve_sweep(Carver& cv, int32_t n, int dim, int32_t k, bool approx, double mean_row, SweepBufs& sb) {
    const int32_t n_src = approx ? k : n;
    sb.part = cv.take<float>((size_t)part_slots(n, dim, n_src, approx) * n * stride_of(dim));
    if (!approx && use_sym(n, dim))
        sb.jpart = cv.take<float>((size_t)sym_jpart_rows(plan_repulse_sym(n, dim)) * n * stride_of(dim));
    (void)mean_row;
    sb.stat_partial = cv.take<double>(stat_partial_doubles(n));
    sb.flags = cv.take<int32_t>(4);
    if (approx) {
        sb.rep_hi = cv.take<float4>(k);
        sb.rep_lo = cv.take<float4>(k);
        sb.mptr = cv.take<int32_t>(k + 1);
        sb.mem = cv.take<int32_t>(n);
        sb.cptr = cv.take<int32_t>(n + 1);
        sb.child = cv.take<int32_t>(n);
        sb.key_sorted = cv.take<int32_t>(n);
        sb.iota = cv.take<int32_t>(n);
        sb.cnt = cv.take<int32_t>(std::max(n, k) + 2);
        sb.rord = cv.take<int32_t>(k);
        sb.sbound = cv.take<int2>(k);
        sb.rpos = cv.take<int32_t>(k);
        sb.tile_nu = cv.take<int32_t>(k / kCoarseTile + 1);
        sb.tperm = cv.take<int32_t>(n);
        sb.tpos = cv.take<int32_t>(n);
        sb.tile_box = cv.take<float4>((size_t)2 * (k / kCoarseTile + 1));
        sb.rkey = cv.take<uint64_t>((size_t)2 * k);
        sb.box = cv.take<uint32_t>(8);
        sb.frame = cv.take<float4>(1);
        sb.tmp_bytes = cub_tmp_bytes(n);
        sb.tmp = cv.take<char>(sb.tmp_bytes);
    }
    return cv.ok;
}

// Q27 switch: kernel (c) drops the lo correction on tiles far from a warp's
// targets (MM_FAR_TILES=0 keeps hi/lo differencing everywhere; experiments)
bool far_tiles() {
    static const bool on = [] {
        const char* v = getenv("MM_FAR_TILES");
        return !(v && v[0] == '0');
    }();
    return on;
}

// Kernel (c)'s orders from the positions x: targets in Morton order, representatives
// by (mass, Morton) so that it scales whole tiles by nu (Q26) and drops the lo
// correction on tiles far from a warp's targets (Q27).  group_by_key left
// iota = 0..n-1 (k <= n); cnt / key_sorted are free scratch after prepare_approx.
cudaError_t coarse_orders(int32_t n, int dim, const mm_approx* ap, const float* x, const SweepBufs& sb,
                          cudaStream_t st) {
    return approx_orders(dim, n, ap->k, sb.mptr, sb.contig ? nullptr : sb.mem, x, kCoarseTile, sb.iota, sb.box,
                         sb.frame, sb.rep_hi,
                         sb.rep_lo, reinterpret_cast<uint32_t*>(sb.cnt), reinterpret_cast<uint32_t*>(sb.key_sorted),
                         sb.tperm,
                         sb.tpos, sb.rkey, sb.rkey + ap->k, sb.rord, sb.rpos, sb.tile_nu, sb.tmp, sb.tmp_bytes, st,
                         sb.contig ? sb.sbound : nullptr);
}

// Re-sort before every sweep when kernel (c)'s work (n k pairs) dwarfs the two
// sorts; otherwise once per level / mm_sweep call (MM_REORDER_PAIRS overrides)
bool reorder_every_sweep(int32_t n, int32_t k) {
    static const double thr = [] {
        const char* v = getenv("MM_REORDER_PAIRS");
        return v ? atof(v) : 1e11;  // measured: cfg4's finest level +2%, cfg3 (2e10) loses 5%
    }();
    return (double)n * (double)k >= thr;
}

// The far-tile machinery costs two small launches per sweep (frame, tile boxes):
// below this many pairs per sweep (kernel (c) well under ~0.3 ms) it does not pay
// (MM_FAR_PAIRS overrides; measured in the MulMent_7/10 schedules, small k)
double far_min_pairs() {
    static const double thr = [] {
        const char* v = getenv("MM_FAR_PAIRS");
        return v ? atof(v) : 1e9;
    }();
    return thr;
}

// Locality renumbering of an Eq.(3) level on the tiled path (k_perm.cuh;
// MM_RENUMBER=0 disables it: experiments, A/B)
// mode 1: representative-slot order (members contiguous); 2: Morton order of
// the level's starting positions (kernel (c)'s target order)
int renumber_mode() {
    static const int m = [] {
        const char* v = getenv("MM_RENUMBER");
        return v ? atoi(v) : 1;
    }();
    return m;
}
bool renumber_enabled() { return renumber_mode() != 0; }

size_t renumber_bytes(int32_t n, int64_t nnz, int32_t k) {
    return 6 * al((size_t)n * 4) + 2 * al((size_t)(k + 1) * 4) + al((size_t)(n + 1) * 8) + 3 * al((size_t)nnz * 4) +
           al(perm_scan_tmp_bytes((int64_t)std::max(n, k) + 1)) + 1024;
}

// Group maps into CSRs (members of each representative, children of each parent).
cudaError_t prepare_approx(int32_t n, int dim, const mm_approx* ap, const float* x, SweepBufs& sb, cudaStream_t st) {
    cudaError_t e = group_by_key(n, ap->ancestor, ap->k, sb.mptr, sb.mem, sb.key_sorted, sb.iota, sb.cnt, sb.tmp,
                                 sb.tmp_bytes, st);
    if (e != cudaSuccess) return e;
    e = group_by_key(n, ap->parent, n, sb.cptr, sb.child, sb.key_sorted, sb.iota, sb.cnt, sb.tmp, sb.tmp_bytes, st);
    if (e != cudaSuccess) return e;
    sb.reorder = reorder_every_sweep(n, ap->k);
    sb.far = far_tiles() && (double)n * (double)ap->k >= far_min_pairs();
    return coarse_orders(n, dim, ap, x, sb, st);
}

// One sweep with all buffers prepared (graph-capturable: no allocation, no sync).
cudaError_t sweep_core(const mm_sset* S, int dim, float alpha, float q, const mm_approx* ap, const float* x_in,
                       float* x_out, mm_sweep_stats* stats, const SweepBufs& sb, cudaStream_t st,
                       const double* alpha_dev = nullptr) {
    const int32_t n = S->n;
    const double mean_row = (double)S->nnz / (double)n;
    const bool qpow = q != 0.0f;
    cudaError_t e = cudaSuccess;
    RepulsePlan p;
    SymPlan sp;
    if (ap) {
        // frame origin of this sweep's positions (Q28); with per-sweep orders it comes with them
        if (sb.reorder) e = coarse_orders(n, dim, ap, x_in, sb, st);
        else if (sb.far) e = launch_frame_fused(dim, n, x_in, sb.box, sb.frame, st);
        if (e != cudaSuccess) return e;
        const float4* frame = sb.far ? sb.frame : nullptr;
        e = launch_centroid(dim, n, ap->k, sb.mptr, sb.contig ? nullptr : sb.mem, x_in, sb.rord, frame, sb.rep_hi,
                            sb.rep_lo, sb.far ? sb.tile_box : nullptr, kCoarseTile, st,
                            sb.contig ? sb.sbound : nullptr);
        if (e != cudaSuccess) return e;
        p = plan_repulse(n, ap->k, dim, true, qpow);
        CoarseOrder co;
        co.tperm = sb.tperm;
        co.tile_nu = sb.tile_nu;
        co.tile_box = sb.far ? sb.tile_box : nullptr;
        co.frame = frame;
        e = launch_repulse(dim, qpow, true, q, n, x_in, ap->k, sb.rep_hi, sb.rep_lo, co, p, sb.part, st);
    } else if (sb.jpart) {
        sp = plan_repulse_sym(n, dim);
        e = launch_repulse_sym(dim, qpow, q, n, x_in, sp, sb.part, sb.jpart, st);
    } else {
        p = plan_repulse(n, n, dim, false, qpow);
        e = launch_repulse(dim, qpow, false, q, n, x_in, n, nullptr, nullptr, CoarseOrder{}, p, sb.part, st);
    }
    if (e != cudaSuccess) return e;
    GatherArgs ga;
    ga.n = n;
    ga.rp = S->row_ptr;
    ga.col = S->col;
    ga.d = S->d;
    ga.w = S->w;
    ga.x = x_in;
    ga.alpha = alpha;
    ga.alpha_dev = alpha_dev;
    ga.q = q;
    ga.part = sb.part;
    ga.sch = p.sch;
    ga.tpb = repulse_targets_per_block(dim);
    ga.jpart = nullptr;
    if (!ap && sb.jpart) {
        ga.jpart = sb.jpart;
        ga.tri = sp.ts;
        ga.tpb = 1024;
    }
    if (ap) {
        ga.anc = ap->ancestor;
        ga.rpos = sb.rpos;
        ga.tpos = sb.tpos;
        ga.frame = sb.far ? sb.frame : nullptr;
        ga.rep_hi = sb.rep_hi;
        ga.rep_lo = sb.rep_lo;
    }
    ga.parent = ap ? ap->parent : nullptr;
    ga.child_ptr = ap ? sb.cptr : nullptr;
    ga.child = ap ? sb.child : nullptr;
    ga.sib = ap ? sb.sib : nullptr;
    ga.x_out = x_out;
    ga.stat_partial = sb.stat_partial;
    ga.flags = sb.flags;
    ga.ticket = sb.flags + 1;
    ga.stats = stats;
    return launch_gather(dim, ga, mean_row, st);
}

// Energy with caller-provided stream; syncs.  Pairs at distance exactly 0 are
// skipped in both the all-pairs and the S sums and counted: *coinc_out (nullable)
// receives the number of coincident non-S ORDERED pairs.  strict: such pairs
// make Eq.(1) undefined (ln 0) and return MM_ERR_NONFINITE (mm_energy); the
// layout report instead records the count next to the finite remainder.
mm_status energy_core(const mm_sset* S, int dim, double alpha, double q, const float* x, double* out,
                      cudaStream_t st, bool strict, int64_t* coinc_out) {
    const int32_t n = S->n;
    const double mean_row = (double)S->nnz / (double)n;
    EntropyPlan ep = plan_entropy(n);
    const int nb_all = ep.nblocks, nb_s = gather_blocks(n, mean_row);
    const size_t bytes = al((size_t)nb_all * 8) + al((size_t)nb_s * 16) + al(16);
    DevBuf buf(bytes, st);
    if (!buf.p) { set_err("mm_energy: out of device memory (%zu B)", bytes); return MM_ERR_OUT_OF_MEMORY; }
    Carver cv(buf.p, bytes);
    double* pa = cv.take<double>(nb_all);
    double* ps = cv.take<double>((size_t)nb_s * 2);
    int32_t* coinc = cv.take<int32_t>(4);
    MM_CU(cudaMemsetAsync(coinc, 0, 16, st), "mm_energy memset");
    MM_CU(launch_entropy_all(dim, q, n, x, ep, pa, coinc, st), "mm_energy entropy_pairs");
    MM_CU(launch_energy_s(dim, q, n, S->row_ptr, S->col, S->d, S->w, x, mean_row, ps, coinc + 1, st),
          "mm_energy energy_s");
    std::vector<double> ha(nb_all), hs((size_t)nb_s * 2);
    int32_t hc[2] = {0, 0};
    MM_CU(cudaMemcpyAsync(ha.data(), pa, (size_t)nb_all * 8, cudaMemcpyDeviceToHost, st), "mm_energy d2h");
    MM_CU(cudaMemcpyAsync(hs.data(), ps, (size_t)nb_s * 16, cudaMemcpyDeviceToHost, st), "mm_energy d2h");
    MM_CU(cudaMemcpyAsync(hc, coinc, 8, cudaMemcpyDeviceToHost, st), "mm_energy d2h");
    MM_CU(cudaStreamSynchronize(st), "mm_energy sync");
    double su = 0.0, ss = 0.0, sp = 0.0;
    for (int b = 0; b < nb_all; ++b) su += ha[b];
    for (int b = 0; b < nb_s; ++b) {
        ss += hs[(size_t)b * 2];
        sp += hs[(size_t)b * 2 + 1];
    }
    // sum over ordered non-S pairs / 2 = sum_{i<j} phi - 1/2 sum_S phi
    const double diff = su - 0.5 * sp;
    const double entropy = (q == 0.0) ? (-0.5 * M_LN2) * diff : diff / q;
    out[0] = 0.5 * ss;
    out[1] = entropy;
    out[2] = out[0] + alpha * out[1];
    const int64_t nonS = 2 * (int64_t)hc[0] - hc[1];
    if (coinc_out) *coinc_out = nonS;
    if (strict && nonS > 0) {
        set_err("mm_energy: %lld coincident non-S ordered pair(s): ln 0 is undefined (Eq.(1))", (long long)nonS);
        return MM_ERR_NONFINITE;
    }
    if (!isfinite(out[2])) {
        set_err("mm_energy: non-finite energy");
        return MM_ERR_NONFINITE;
    }
    return MM_OK;
}

}  // namespace

// ================================================================== C ABI
extern "C" {

const char* mm_status_string(mm_status s) {
    switch (s) {
        case MM_OK: return "MM_OK";
        case MM_ERR_INVALID_ARGUMENT: return "MM_ERR_INVALID_ARGUMENT";
        case MM_ERR_INVALID_INPUT: return "MM_ERR_INVALID_INPUT";
        case MM_ERR_NONFINITE: return "MM_ERR_NONFINITE";
        case MM_ERR_OUT_OF_MEMORY: return "MM_ERR_OUT_OF_MEMORY";
        case MM_ERR_CUDA: return "MM_ERR_CUDA";
        case MM_ERR_UNSUPPORTED: return "MM_ERR_UNSUPPORTED";
    }
    return "MM_ERR_UNKNOWN";
}

const char* mm_last_error(void) { return g_err.c_str(); }

const char* mm_version(void) { return "mm_b200 0.1 sm_100a"; }

mm_status mm_set_allocator(void* (*alloc)(size_t, mm_stream_t, void*), void (*free_)(void*, mm_stream_t, void*),
                           void* ctx) {
    if ((alloc == nullptr) != (free_ == nullptr)) {
        set_err("mm_set_allocator: alloc and free must both be set or both be NULL");
        return MM_ERR_INVALID_ARGUMENT;
    }
    g_alloc = alloc;
    g_free = free_;
    g_alloc_ctx = ctx;
    return MM_OK;
}

mm_status mm_sweep_workspace(int32_t n, int dim, const mm_approx* ap, size_t* bytes) {
    if (!bytes || n <= 0) { set_err("mm_sweep_workspace: bad arguments"); return MM_ERR_INVALID_ARGUMENT; }
    if (dim != 2 && dim != 3) { set_err("mm_sweep_workspace: dim must be 2 or 3"); return MM_ERR_UNSUPPORTED; }
    if (ap && ap->k <= 0) { set_err("mm_sweep_workspace: ap->k must be > 0"); return MM_ERR_INVALID_ARGUMENT; }
    *bytes = sweep_bytes(n, dim, ap ? ap->k : 0, ap != nullptr, 1.0);
    return MM_OK;
}

mm_status mm_sweep(const mm_sset* S, int dim, float alpha, float q, const mm_approx* ap, const float* x_in,
                   float* x_out, mm_sweep_stats* stats, void* ws, size_t ws_bytes, mm_stream_t stream) {
    mm_status s;
    if ((s = check_sset(S, "mm_sweep")) != MM_OK) return s;
    if ((s = check_dim_q(dim, q, "mm_sweep")) != MM_OK) return s;
    if ((s = check_x(x_in, dim, "x_in", "mm_sweep")) != MM_OK) return s;
    if ((s = check_x(x_out, dim, "x_out", "mm_sweep")) != MM_OK) return s;
    if (!isfinite(alpha)) { set_err("mm_sweep: alpha must be finite"); return MM_ERR_INVALID_ARGUMENT; }
    const int32_t n = S->n;
    const size_t xb = (size_t)n * stride_of(dim) * sizeof(float);
    const char *a0 = (const char*)x_in, *b0 = (const char*)x_out;
    if (a0 < b0 + xb && b0 < a0 + xb) { set_err("mm_sweep: x_out must not alias x_in"); return MM_ERR_INVALID_ARGUMENT; }
    if (ap) {
        if (ap->k <= 0 || ap->k > n || !ap->parent || !ap->ancestor) {
            set_err("mm_sweep: bad mm_approx (k=%d must be in [1, n], maps non-NULL)", ap ? ap->k : 0);
            return MM_ERR_INVALID_ARGUMENT;
        }
    }
    cudaStream_t st = (cudaStream_t)stream;
    const double mean_row = (double)S->nnz / (double)n;
    const size_t need = sweep_bytes(n, dim, ap ? ap->k : 0, ap != nullptr, mean_row);
    DevBuf own;
    void* base = ws;
    size_t cap = ws_bytes;
    if (!ws) {
        own.st = st;
        own.p = dev_alloc(need, st);
        if (!own.p) { set_err("mm_sweep: out of device memory (%zu B)", need); return MM_ERR_OUT_OF_MEMORY; }
        base = own.p;
        cap = need;
    } else if (ws_bytes < need) {
        set_err("mm_sweep: workspace too small (%zu < %zu B)", ws_bytes, need);
        return MM_ERR_INVALID_ARGUMENT;
    }
    if (ws && ((uintptr_t)ws & 255u) != 0) {
        set_err("mm_sweep: workspace must be 256-B aligned (got %p)", ws);
        return MM_ERR_INVALID_ARGUMENT;
    }
    Carver cv(base, cap);
    SweepBufs sb;
    if (!carve_sweep(cv, n, dim, ap ? ap->k : 0, ap != nullptr, mean_row, sb)) {
        set_err("mm_sweep: workspace carving failed");
        return MM_ERR_INVALID_ARGUMENT;
    }
    MM_CU(cudaMemsetAsync(sb.flags, 0, 4 * sizeof(int32_t), st), "mm_sweep memset");
    if (ap) MM_CU(prepare_approx(n, dim, ap, x_in, sb, st), "mm_sweep prepare_approx");
    MM_CU(sweep_core(S, dim, alpha, q, ap, x_in, x_out, stats, sb, st), "mm_sweep");
    return MM_OK;
}

mm_status mm_energy(const mm_sset* S, int dim, double alpha, double q, const float* x, double* out,
                    mm_stream_t stream) {
    mm_status s;
    if ((s = check_sset(S, "mm_energy")) != MM_OK) return s;
    if ((s = check_dim_q(dim, q, "mm_energy")) != MM_OK) return s;
    if ((s = check_x(x, dim, "x", "mm_energy")) != MM_OK) return s;
    if (!out) { set_err("mm_energy: out is NULL"); return MM_ERR_INVALID_ARGUMENT; }
    return energy_core(S, dim, alpha, q, x, out, (cudaStream_t)stream, true, nullptr);
}

int64_t mm_launch_count(void) { return g_launches.load(); }

int mm_exact_kernel_variant(int32_t n, int dim) {
    if (n < 1 || (dim != 2 && dim != 3)) return 0;
    return use_sym(n, dim) ? 1 : 0;
}

mm_status mm_profile_enable(int on) {
    g_prof_on.store(on ? 1 : 0);
    return MM_OK;
}

mm_status mm_profile_reset(void) {
    std::lock_guard<std::mutex> g(g_prof_mu);
    for (auto& p : g_pending) {
        cudaEventSynchronize(p.b);
        g_event_pool.push_back(p.a);
        g_event_pool.push_back(p.b);
    }
    g_pending.clear();
    g_prof.clear();
    g_prof_list.clear();
    return MM_OK;
}

namespace {
// folds the pending launch events into the per-name totals and the ordered list (holds g_prof_mu)
void prof_fold() {
    for (auto& p : g_pending) {
        cudaError_t e = cudaEventSynchronize(p.b);
        float ms = 0.f;
        if (e == cudaSuccess && cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
            auto& r = g_prof[p.name];
            r.first += 1;
            r.second += ms;
            g_prof_list.emplace_back(p.name, ms);
        } else {
            cudaGetLastError();
        }
        g_event_pool.push_back(p.a);
        g_event_pool.push_back(p.b);
    }
    g_pending.clear();
}
}  // namespace

mm_status mm_profile_last(const char* name, int32_t max, double* ms, int32_t* count) {
    if (!name || (max > 0 && !ms) || !count) { set_err("mm_profile_last: NULL argument"); return MM_ERR_INVALID_ARGUMENT; }
    std::lock_guard<std::mutex> g(g_prof_mu);
    prof_fold();
    int32_t c = 0;
    for (auto it = g_prof_list.rbegin(); it != g_prof_list.rend() && c < max; ++it)
        if (strcmp(it->first, name) == 0) ms[c++] = it->second;
    std::reverse(ms, ms + c);
    *count = c;
    return MM_OK;
}

mm_status mm_profile_read(mm_kernel_profile* out, int32_t max, int32_t* count) {
    std::lock_guard<std::mutex> g(g_prof_mu);
    prof_fold();
    int32_t i = 0;
    for (auto& kv : g_prof) {
        if (out && i < max) {
            memset(out[i].name, 0, sizeof(out[i].name));
            strncpy(out[i].name, kv.first.c_str(), sizeof(out[i].name) - 1);
            out[i].launches = kv.second.first;
            out[i].total_ms = kv.second.second;
        }
        ++i;
    }
    if (count) *count = i;
    return MM_OK;
}

}  // extern "C"

// ================================================================== hierarchy
struct HLevel {
    int32_t n = 0;
    int64_t nnz = 0;
    int64_t* rp = nullptr;
    int32_t* col = nullptr;
    int32_t* omega = nullptr;
    int32_t* c = nullptr;
    int32_t* parent = nullptr;
    float* d = nullptr;
    float* w = nullptr;
    int32_t rounds = 0;
};

struct mm_hierarchy {
    std::vector<HLevel> lv;
};

namespace {

void free_level(HLevel& l) {
    dev_free(l.rp, nullptr);
    dev_free(l.col, nullptr);
    dev_free(l.omega, nullptr);
    dev_free(l.c, nullptr);
    dev_free(l.parent, nullptr);
    dev_free(l.d, nullptr);
    dev_free(l.w, nullptr);
    l = HLevel();
}

template <class T>
T* alloc_n(size_t count, cudaStream_t st) {
    return (T*)dev_alloc(sizeof(T) * (count > 0 ? count : 1), st);
}

// clustering of the hierarchy: heavy-edge matching (Q16, default) or SCLaP (R6)
struct HierMode {
    bool sclap = false;
    int32_t lp_rounds = 3;
    double f0 = 20.0, b = 2.0;
};

// Calls that drive the device-resident synchronisation state (the grid
// barriers of k_match_level and k_small_level, the schedule loop's
// g_sched_state) hold this lock from their first launch until their final
// stream synchronisation, so concurrent calls from several host threads (any
// streams) cannot interleave on that state.  Recursive: mm_layout builds its
// hierarchy through build_hierarchy_impl.
std::recursive_mutex g_state_mu;

mm_status build_hierarchy_impl(const mm_graph* g, const int32_t* c, int dim, uint64_t seed, int32_t n_stop,
                               int32_t max_levels, int32_t max_rounds, mm_hierarchy** out, cudaStream_t st,
                               const HierMode& mode = HierMode()) {
    std::lock_guard<std::recursive_mutex> state_lock(g_state_mu);
    const int32_t n0 = g->n;
    const int64_t nnz0 = g->nnz;
    mm_hierarchy* H = new mm_hierarchy();
    auto fail = [&](mm_status s) {
        cudaStreamSynchronize(st);
        for (auto& l : H->lv) free_level(l);
        delete H;
        return s;
    };
    HLevel l0;
    l0.n = n0;
    l0.nnz = nnz0;
    l0.rp = alloc_n<int64_t>((size_t)n0 + 1, st);
    l0.col = alloc_n<int32_t>(nnz0, st);
    l0.omega = alloc_n<int32_t>(nnz0, st);
    l0.c = alloc_n<int32_t>(n0, st);
    H->lv.push_back(l0);
    if (!l0.rp || !l0.col || !l0.omega || !l0.c) { set_err("mm_build_hierarchy: out of memory"); return fail(MM_ERR_OUT_OF_MEMORY); }
    if (cudaMemcpyAsync(l0.rp, g->row_ptr, sizeof(int64_t) * ((size_t)n0 + 1), cudaMemcpyDeviceToDevice, st) ||
        (nnz0 > 0 && cudaMemcpyAsync(l0.col, g->col, sizeof(int32_t) * nnz0, cudaMemcpyDeviceToDevice, st))) {
        set_err("mm_build_hierarchy: copy failed");
        return fail(MM_ERR_CUDA);
    }
    if (g->omega) {
        if (nnz0 > 0 && cudaMemcpyAsync(l0.omega, g->omega, sizeof(int32_t) * nnz0, cudaMemcpyDeviceToDevice, st)) {
            set_err("mm_build_hierarchy: copy failed");
            return fail(MM_ERR_CUDA);
        }
    } else if (launch_fill(nnz0, 1, l0.omega, st) != cudaSuccess) {
        set_err("mm_build_hierarchy: fill failed");
        return fail(MM_ERR_CUDA);
    }
    if (c) {
        if (cudaMemcpyAsync(l0.c, c, sizeof(int32_t) * n0, cudaMemcpyDeviceToDevice, st)) {
            set_err("mm_build_hierarchy: copy failed");
            return fail(MM_ERR_CUDA);
        }
    } else if (launch_fill(n0, 1, l0.c, st) != cudaSuccess) {
        set_err("mm_build_hierarchy: fill failed");
        return fail(MM_ERR_CUDA);
    }
    // scratch sized by level 0 (levels only shrink)
    const int64_t m0 = std::max<int64_t>(nnz0, 1);
    const size_t tmpb = std::max(sort_temp_bytes_u64(m0), scan_temp_bytes((int32_t)std::max<int64_t>(m0, n0 + 2))) + 256;
    const size_t bytes = al((size_t)n0 * 4 + 8) * 6 + al(64) + al((size_t)m0 * 8) * 2 + al((size_t)m0 * 4) * 6 +
                         al(((size_t)n0 + 2) * 4) * 2 + al(tmpb) + 4096;
    DevBuf scratch(bytes, st);
    if (!scratch.p) { set_err("mm_build_hierarchy: out of memory (%zu B scratch)", bytes); return fail(MM_ERR_OUT_OF_MEMORY); }
    Carver cv(scratch.p, bytes);
    int32_t* mate = cv.take<int32_t>(n0);
    int32_t* cand = cv.take<int32_t>(n0);  // SCLaP: the labels
    int32_t* flag = cv.take<int32_t>((size_t)n0 + 2);
    int32_t* cid = cv.take<int32_t>((size_t)n0 + 2);
    int32_t* cnext = cv.take<int32_t>(n0);
    int32_t* spare = cv.take<int32_t>(n0);
    (void)spare;
    int32_t* added = cv.take<int32_t>(16);
    uint64_t* keys = cv.take<uint64_t>(m0);
    uint64_t* keys_alt = cv.take<uint64_t>(m0);
    int32_t* vals = cv.take<int32_t>(m0);
    int32_t* vals_alt = cv.take<int32_t>(m0);
    int32_t* head = cv.take<int32_t>(m0);
    int32_t* pos = cv.take<int32_t>(m0);
    int32_t* ccol = cv.take<int32_t>(m0);
    int32_t* comega = cv.take<int32_t>(m0);
    int32_t* rowcnt = cv.take<int32_t>((size_t)n0 + 2);
    int32_t* excl = cv.take<int32_t>((size_t)n0 + 2);
    void* tmp = cv.take<char>(tmpb);
    if (!cv.ok) { set_err("mm_build_hierarchy: scratch carving failed"); return fail(MM_ERR_INVALID_ARGUMENT); }

    double f = mode.f0;
    int decays = 0;
    while ((int32_t)H->lv.size() < max_levels) {
        const size_t li = H->lv.size() - 1;
        const HLevel cur = H->lv[li];
        if (cur.n <= n_stop) break;
        int32_t nc = 0;
        int32_t* parent = nullptr;
        if (mode.sclap) {
            // U = max(max c, W), W = min(b^h, n0 / f), h = 1 for the first coarsening
            const int32_t h = (int32_t)li + 1;
            int32_t cmax = 0;
            if (launch_max_i32(cur.n, cur.c, added, st) || cudaMemcpyAsync(&cmax, added, 4, cudaMemcpyDeviceToHost, st) ||
                cudaStreamSynchronize(st)) {
                set_err("mm_build_hierarchy: max c failed");
                return fail(MM_ERR_CUDA);
            }
            double W = 1.0;
            for (int32_t t = 0; t < h && W < 1e18; ++t) W *= mode.b;
            W = std::min(W, (double)n0 / f);
            const long long U = std::max<long long>(cmax, (long long)W);
            int32_t used = 0;
            cudaError_t e = sclap_labels_gpu(cur.n, cur.nnz, cur.rp, cur.col, cur.omega, cur.c, U, mode.lp_rounds,
                                             seed, (int32_t)li, cand, &used, st, dev_alloc, dev_free);
            if (e != cudaSuccess) {
                set_err("mm_build_hierarchy: SCLaP failed: %s", cudaGetErrorString(e));
                return fail(e == cudaErrorMemoryAllocation ? MM_ERR_OUT_OF_MEMORY : MM_ERR_CUDA);
            }
            H->lv[li].rounds = mode.lp_rounds;
            parent = alloc_n<int32_t>(cur.n, st);
            if (!parent) { set_err("mm_build_hierarchy: out of memory"); return fail(MM_ERR_OUT_OF_MEMORY); }
            if (contract_labels_gpu(cur.n, cand, cur.c, flag, cid, parent, cnext, added, tmp, tmpb, st) ||
                cudaMemcpyAsync(&nc, added, 4, cudaMemcpyDeviceToHost, st) || cudaStreamSynchronize(st)) {
                dev_free(parent, st);
                set_err("mm_build_hierarchy: label contraction failed: %s", cudaGetErrorString(cudaGetLastError()));
                return fail(MM_ERR_CUDA);
            }
            if (nc == cur.n) {  // nothing merged: decay f and retry this level (at most 10 times)
                dev_free(parent, st);
                f *= 0.7;
                if (++decays >= 10) break;
                continue;
            }
            if ((int64_t)10 * nc > (int64_t)9 * cur.n) {  // "not more than 10% smaller": f <- 0.7 f
                f *= 0.7;
                ++decays;
            } else {
                decays = 0;
            }
        } else {
        if (launch_fill(cur.n, -1, mate, st) != cudaSuccess) { set_err("mm_build_hierarchy: fill"); return fail(MM_ERR_CUDA); }
        int32_t rounds = max_rounds;
        bool device_loop = false;
        {
            // all rounds in one cooperative launch (host loop below if it cannot be resident)
            const cudaError_t e = max_rounds > 0 ? run_match_level(cur.n, cur.nnz, cur.rp, cur.col, cur.omega, cur.c, mate,
                                                                   cand, seed, (int32_t)li, max_rounds, added,
                                                                   added + 2, st)
                                                 : cudaErrorNotSupported;
            if (e == cudaSuccess) {
                device_loop = true;
                if (cudaMemcpyAsync(&rounds, added + 2, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
                    cudaStreamSynchronize(st) != cudaSuccess) {
                    set_err("mm_build_hierarchy: matching rounds d2h");
                    return fail(MM_ERR_CUDA);
                }
            } else {
                cudaGetLastError();
                if (e != cudaErrorCooperativeLaunchTooLarge && e != cudaErrorNotSupported) {
                    set_err("mm_build_hierarchy: matching: %s", cudaGetErrorString(e));
                    return fail(MM_ERR_CUDA);
                }
            }
        }
        for (int32_t r = 0; r < max_rounds && !device_loop; ++r) {
            int32_t h_added = 0;
            if (cudaMemsetAsync(added, 0, 4, st) ||
                run_match_round(cur.n, cur.nnz, cur.rp, cur.col, cur.omega, cur.c, mate, cand, seed, (int32_t)li, r, added, st) ||
                cudaMemcpyAsync(&h_added, added, 4, cudaMemcpyDeviceToHost, st) || cudaStreamSynchronize(st)) {
                cudaError_t e = cudaGetLastError();
                set_err("mm_build_hierarchy: matching round failed: %s", cudaGetErrorString(e));
                return fail(MM_ERR_CUDA);
            }
            if (h_added == 0) {
                rounds = r + 1;
                break;
            }
        }
        H->lv[li].rounds = rounds;
        parent = alloc_n<int32_t>(cur.n, st);
        if (!parent) { set_err("mm_build_hierarchy: out of memory"); return fail(MM_ERR_OUT_OF_MEMORY); }
        int32_t last[2] = {0, 0};
        if (contract_leaders(cur.n, mate, cur.c, flag, cid, parent, cnext, tmp, tmpb, st) ||
            cudaMemcpyAsync(&last[0], cid + cur.n - 1, 4, cudaMemcpyDeviceToHost, st) ||
            cudaMemcpyAsync(&last[1], flag + cur.n - 1, 4, cudaMemcpyDeviceToHost, st) || cudaStreamSynchronize(st)) {
            dev_free(parent, st);
            set_err("mm_build_hierarchy: contraction failed: %s", cudaGetErrorString(cudaGetLastError()));
            return fail(MM_ERR_CUDA);
        }
        nc = last[0] + last[1];
        if ((int64_t)10 * nc > (int64_t)9 * cur.n) {  // Q17: less than 10% smaller -> discard, stop
            dev_free(parent, st);
            break;
        }
        }
        int64_t m2 = 0;
        if (cur.nnz > 0) {
            int32_t lastp[2] = {0, 0};
            if (contract_edges(cur.n, cur.nnz, cur.rp, cur.col, cur.omega, parent, nc, keys, keys_alt, vals, vals_alt,
                               head, pos, ccol, comega, rowcnt, tmp, tmpb, st) ||
                cudaMemcpyAsync(&lastp[0], pos + cur.nnz - 1, 4, cudaMemcpyDeviceToHost, st) ||
                cudaMemcpyAsync(&lastp[1], head + cur.nnz - 1, 4, cudaMemcpyDeviceToHost, st) ||
                cudaStreamSynchronize(st)) {
                dev_free(parent, st);
                set_err("mm_build_hierarchy: edge contraction failed: %s", cudaGetErrorString(cudaGetLastError()));
                return fail(MM_ERR_CUDA);
            }
            m2 = (int64_t)lastp[0] + lastp[1];
        }
        HLevel nx;
        nx.n = nc;
        nx.nnz = m2;
        nx.rp = alloc_n<int64_t>((size_t)nc + 1, st);
        nx.col = alloc_n<int32_t>(m2, st);
        nx.omega = alloc_n<int32_t>(m2, st);
        nx.c = alloc_n<int32_t>(nc, st);
        nx.d = alloc_n<float>(m2, st);
        nx.w = alloc_n<float>(m2, st);
        H->lv[li].parent = parent;
        H->lv.push_back(nx);
        if (!nx.rp || !nx.col || !nx.omega || !nx.c || !nx.d || !nx.w) {
            set_err("mm_build_hierarchy: out of memory");
            return fail(MM_ERR_OUT_OF_MEMORY);
        }
        if (rowptr_from_rows(nc, vals, m2, nx.rp, st) ||
            (m2 > 0 && cudaMemcpyAsync(nx.col, ccol, 4 * m2, cudaMemcpyDeviceToDevice, st)) ||
            (m2 > 0 && cudaMemcpyAsync(nx.omega, comega, 4 * m2, cudaMemcpyDeviceToDevice, st)) ||
            cudaMemcpyAsync(nx.c, cnext, 4 * (size_t)nc, cudaMemcpyDeviceToDevice, st) ||
            launch_coarse_sset(m2, vals, nx.col, nx.c, dim, nx.d, nx.w, st)) {
            set_err("mm_build_hierarchy: level assembly failed: %s", cudaGetErrorString(cudaGetLastError()));
            return fail(MM_ERR_CUDA);
        }
        if (mode.sclap && decays >= 10) break;
    }
    if (cudaStreamSynchronize(st) != cudaSuccess) {
        set_err("mm_build_hierarchy: %s", cudaGetErrorString(cudaGetLastError()));
        return fail(MM_ERR_CUDA);
    }
    *out = H;
    return MM_OK;
}

mm_status check_graph(const mm_graph* g, const char* who) {
    if (!g || g->n <= 0 || g->nnz < 0 || !g->row_ptr || (g->nnz > 0 && !g->col)) {
        set_err("%s: bad mm_graph (n > 0, nnz >= 0, row_ptr/col non-NULL required)", who);
        return MM_ERR_INVALID_ARGUMENT;
    }
    if (g->nnz > INT32_MAX) { set_err("%s: nnz > 2^31-1 unsupported", who); return MM_ERR_UNSUPPORTED; }
    return MM_OK;
}

}  // namespace

extern "C" {

mm_status mm_build_hierarchy(const mm_graph* g, const int32_t* c, int dim, uint64_t seed, int32_t n_stop,
                             int32_t max_levels, int32_t max_rounds, mm_hierarchy** out, mm_stream_t stream) {
    mm_status s;
    if ((s = check_graph(g, "mm_build_hierarchy")) != MM_OK) return s;
    if (dim != 2 && dim != 3) { set_err("mm_build_hierarchy: dim must be 2 or 3"); return MM_ERR_UNSUPPORTED; }
    if (!out || n_stop < 1 || max_levels < 1 || max_levels > MM_MAX_LEVELS || max_rounds < 1) {
        set_err("mm_build_hierarchy: bad arguments (out non-NULL, n_stop >= 1, 1 <= max_levels <= %d, max_rounds >= 1)",
                MM_MAX_LEVELS);
        return MM_ERR_INVALID_ARGUMENT;
    }
    *out = nullptr;
    return build_hierarchy_impl(g, c, dim, seed, n_stop, max_levels, max_rounds, out, (cudaStream_t)stream);
}

mm_status mm_build_hierarchy_sclap(const mm_graph* g, const int32_t* c, int dim, uint64_t seed, int32_t n_stop,
                                   int32_t max_levels, int32_t lp_rounds, double f0, double b, mm_hierarchy** out,
                                   mm_stream_t stream) {
    mm_status s;
    if ((s = check_graph(g, "mm_build_hierarchy_sclap")) != MM_OK) return s;
    if (dim != 2 && dim != 3) { set_err("mm_build_hierarchy_sclap: dim must be 2 or 3"); return MM_ERR_UNSUPPORTED; }
    if (!out || n_stop < 1 || max_levels < 1 || max_levels > MM_MAX_LEVELS || lp_rounds < 1 || !(f0 > 0.0) ||
        !(b > 1.0)) {
        set_err("mm_build_hierarchy_sclap: bad arguments (out, n_stop >= 1, 1 <= max_levels <= %d, lp_rounds >= 1, "
                "f0 > 0, b > 1)", MM_MAX_LEVELS);
        return MM_ERR_INVALID_ARGUMENT;
    }
    *out = nullptr;
    HierMode m;
    m.sclap = true;
    m.lp_rounds = lp_rounds;
    m.f0 = f0;
    m.b = b;
    return build_hierarchy_impl(g, c, dim, seed, n_stop, max_levels, 64, out, (cudaStream_t)stream, m);
}

int32_t mm_hierarchy_num_levels(const mm_hierarchy* h) { return h ? (int32_t)h->lv.size() : 0; }

mm_status mm_hierarchy_level(const mm_hierarchy* h, int32_t level, mm_level_view* out) {
    if (!h || !out || level < 0 || level >= (int32_t)h->lv.size()) {
        set_err("mm_hierarchy_level: bad arguments");
        return MM_ERR_INVALID_ARGUMENT;
    }
    const HLevel& l = h->lv[level];
    out->n = l.n;
    out->nnz = l.nnz;
    out->row_ptr = l.rp;
    out->col = l.col;
    out->omega = l.omega;
    out->c = l.c;
    out->parent = l.parent;
    out->d = l.d;
    out->w = l.w;
    out->rounds = l.rounds;
    return MM_OK;
}

mm_status mm_hierarchy_copy_level(const mm_hierarchy* h, int32_t level, int64_t* row_ptr, int32_t* col,
                                  int32_t* omega, int32_t* c, int32_t* parent, float* d, float* w, mm_stream_t stream) {
    if (!h || level < 0 || level >= (int32_t)h->lv.size()) {
        set_err("mm_hierarchy_copy_level: bad arguments");
        return MM_ERR_INVALID_ARGUMENT;
    }
    const HLevel& l = h->lv[level];
    cudaStream_t st = (cudaStream_t)stream;
    const auto cp = [&](void* dst, const void* src, size_t bytes) {
        return (dst && src && bytes) ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st) : cudaSuccess;
    };
    MM_CU(cp(row_ptr, l.rp, sizeof(int64_t) * ((size_t)l.n + 1)), "mm_hierarchy_copy_level");
    MM_CU(cp(col, l.col, sizeof(int32_t) * l.nnz), "mm_hierarchy_copy_level");
    MM_CU(cp(omega, l.omega, sizeof(int32_t) * l.nnz), "mm_hierarchy_copy_level");
    MM_CU(cp(c, l.c, sizeof(int32_t) * l.n), "mm_hierarchy_copy_level");
    MM_CU(cp(parent, l.parent, sizeof(int32_t) * l.n), "mm_hierarchy_copy_level");
    MM_CU(cp(d, l.d, sizeof(float) * l.nnz), "mm_hierarchy_copy_level");
    MM_CU(cp(w, l.w, sizeof(float) * l.nnz), "mm_hierarchy_copy_level");
    MM_CU(cudaStreamSynchronize(st), "mm_hierarchy_copy_level");
    return MM_OK;
}

void mm_hierarchy_free(mm_hierarchy* h) {
    if (!h) return;
    cudaDeviceSynchronize();
    for (auto& l : h->lv) free_level(l);
    delete h;
}

}  // extern "C"

// ================================================================== layout driver
namespace {

bool graphs_enabled() {
    const char* e = getenv("MM_NO_GRAPHS");
    return !(e && e[0] && e[0] != '0') && !g_prof_on.load();
}

// Instantiated CUDA graphs of K-sweep sequences, keyed by every value the
// captured launches depend on (pointers, sizes, parameters).  A hit relaunches
// the executable graph; capture + instantiate is paid once per distinct key.
struct GraphKey {
    const void* p[24];
    int64_t v[8];
    float f[2];
    int32_t kind = 0;      // 0: K fixed sweeps; 1: device-driven schedule loop of one level
    int32_t si[3] = {0, 0, 0};
    double sd[4] = {0, 0, 0, 0};
    bool operator==(const GraphKey& o) const { return memcmp(this, &o, sizeof(GraphKey)) == 0; }
};
struct GraphEntry {
    GraphKey key;
    cudaGraphExec_t exec;
    int64_t kernels;
    uint64_t stamp;
};
std::mutex g_graph_mu;
std::vector<GraphEntry> g_graphs;
uint64_t g_graph_clock = 0;
constexpr size_t kGraphCacheMax = 16;

// cache lookup: on a hit the launch counter advances by the graph's kernels
// (for a schedule graph: one body pass per lookup, an undercount)
cudaGraphExec_t graph_cache_find(const GraphKey& key) {
    std::lock_guard<std::mutex> g(g_graph_mu);
    for (auto& e : g_graphs) {
        if (e.key == key) {
            e.stamp = ++g_graph_clock;
            g_launches.fetch_add(e.kernels, std::memory_order_relaxed);
            return e.exec;
        }
    }
    return nullptr;
}

void graph_cache_insert(const GraphKey& key, cudaGraphExec_t exec, int64_t kernels) {
    std::lock_guard<std::mutex> g(g_graph_mu);
    if (g_graphs.size() >= kGraphCacheMax) {
        size_t victim = 0;
        for (size_t i = 1; i < g_graphs.size(); ++i)
            if (g_graphs[i].stamp < g_graphs[victim].stamp) victim = i;
        cudaDeviceSynchronize();  // the victim may still be running
        cudaGraphExecDestroy(g_graphs[victim].exec);
        g_graphs.erase(g_graphs.begin() + victim);
    }
    g_graphs.push_back(GraphEntry{key, exec, kernels, ++g_graph_clock});
}

GraphKey make_key(const mm_sset* S, int dim, float alpha, float q, const mm_approx* ap, const float* src,
                  const float* bufA, const float* bufB, int32_t K, const mm_sweep_stats* stats, const SweepBufs& sb,
                  cudaStream_t st) {
    GraphKey k;
    memset(&k, 0, sizeof(k));
    (void)st;  // an executable graph may be launched into any stream
    const void* ps[24] = {S->row_ptr, S->col, S->d, S->w, src, bufA, bufB, stats, sb.part, sb.stat_partial,
                          sb.flags, sb.rep_hi, sb.rep_lo, sb.mptr, ap ? ap->ancestor : nullptr, sb.child, sb.jpart,
                          sb.rord, sb.rpos, sb.tile_nu, sb.tperm, sb.tpos, sb.tile_box, sb.frame};
    memcpy(k.p, ps, sizeof(ps));
    k.v[0] = S->n;
    k.v[1] = S->nnz;
    k.v[2] = dim;
    k.v[3] = K;
    k.v[4] = ap ? ap->k : -1;
    k.v[5] = (int64_t)(uintptr_t)(ap ? ap->parent : nullptr);
    k.v[6] = (int64_t)(uintptr_t)sb.cptr;
    k.v[7] = (int64_t)(uintptr_t)sb.mem;
    k.f[0] = alpha;
    k.f[1] = q;
    return k;
}

// Runs K sweeps ping-ponging between bufA/bufB starting from src; returns the
// buffer holding the result.  With graphs enabled the sequence is captured
// once into a CUDA graph (cached) and relaunched.
cudaError_t run_sweeps(const mm_sset* S, int dim, float alpha, float q, const mm_approx* ap, const float* src,
                       float* bufA, float* bufB, int32_t K, mm_sweep_stats* stats, const SweepBufs& sb,
                       cudaStream_t st, const float** result) {
    if (K <= 0) {
        *result = src;
        return cudaSuccess;
    }
    // result buffer of the ping-pong (independent of capture)
    const float* cur = src;
    for (int32_t s = 0; s < K; ++s) cur = (cur == bufA) ? bufB : bufA;
    *result = cur;
    const bool use_graph = graphs_enabled() && K > 1 && st != nullptr;
    if (!use_graph) {
        const float* c = src;
        for (int32_t s = 0; s < K; ++s) {
            float* dst = (c == bufA) ? bufB : bufA;
            cudaError_t err = sweep_core(S, dim, alpha, q, ap, c, dst, stats, sb, st);
            if (err != cudaSuccess) return err;
            c = dst;
        }
        return cudaSuccess;
    }
    const GraphKey key = make_key(S, dim, alpha, q, ap, src, bufA, bufB, K, stats, sb, st);
    if (cudaGraphExec_t hit = graph_cache_find(key)) return cudaGraphLaunch(hit, st);
    const int64_t l0 = g_launches.load();
    cudaError_t err = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    if (err != cudaSuccess) return err;
    const float* c = src;
    for (int32_t s = 0; s < K && err == cudaSuccess; ++s) {
        float* dst = (c == bufA) ? bufB : bufA;
        err = sweep_core(S, dim, alpha, q, ap, c, dst, stats, sb, st);
        c = dst;
    }
    cudaGraph_t graph = nullptr;
    cudaError_t e2 = cudaStreamEndCapture(st, &graph);
    if (err == cudaSuccess) err = e2;
    cudaGraphExec_t exec = nullptr;
    if (err == cudaSuccess) err = cudaGraphInstantiate(&exec, graph, 0);
    if (graph) cudaGraphDestroy(graph);
    if (err != cudaSuccess) {
        if (exec) cudaGraphExecDestroy(exec);
        return err;
    }
    err = cudaGraphLaunch(exec, st);
    graph_cache_insert(key, exec, g_launches.load() - l0);
    return err;
}

}  // namespace

namespace {

// ------------------------------------------------------------------ per-level runners
// A runner performs the sweeps of one level, starting from `src` (read-only
// until consumed) and ping-ponging between A and B; it returns the buffer
// holding the result and the number of sweeps it ran.
struct Runner {
    virtual ~Runner() {}
    virtual mm_status run(const mm_sset* S, int dim, float q, const mm_approx* ap, const float* src, float* A, float* B,
                          mm_sweep_stats* dstats, const SweepBufs& sb, cudaStream_t ls, int32_t level,
                          bool start_at_min, const float** res, int32_t* sweeps) = 0;
};

// Small levels: all sweeps of the level in one persistent cooperative kernel
// (k_small.cu).  mode 0: K sweeps at alpha0 (no host wait; the result buffer
// follows from K's parity); mode 1: the schedule, decided on the device (one
// host wait for the sweep count).
mm_status run_small(const mm_sset* S, int dim, float q, const mm_approx* ap, const float* src, float* A, float* B,
                    mm_sweep_stats* dstats, const SweepBufs& sb, cudaStream_t ls, int mode, int32_t K, double alpha0,
                    const mm_schedule* sch, const float** res, int32_t* nsw) {
    const size_t xbytes = (size_t)S->n * stride_of(dim) * sizeof(float);
    float *x0, *x1;
    if (src == A) {
        x0 = A;
        x1 = B;
    } else {
        if (src != B) MM_CU(cudaMemcpyAsync(B, src, xbytes, cudaMemcpyDeviceToDevice, ls), "small level copy");
        x0 = B;
        x1 = A;
    }
    SmallArgs a;
    a.n = S->n;
    a.k = ap ? ap->k : 0;
    a.rp = S->row_ptr;
    a.col = S->col;
    a.d = S->d;
    a.w = S->w;
    a.x0 = x0;
    a.x1 = x1;
    a.q = q;
    if (ap) {
        a.anc = ap->ancestor;
        a.parent = ap->parent;
        a.mptr = sb.mptr;
        a.mem = sb.mem;
        a.cptr = sb.cptr;
        a.child = sb.child;
        a.rep_hi = sb.rep_hi;
        a.rep_lo = sb.rep_lo;
    }
    a.mode = mode;
    a.K = K;
    a.alpha0 = alpha0;
    if (sch) {
        a.alpha_min = sch->alpha_min;
        a.factor = sch->factor;
        a.eps = sch->eps;
        a.rounds = sch->a;
        a.max_final = sch->max_final_iters;
    }
    a.partial = sb.stat_partial;
    a.result = sb.flags;  // re-armed (memset) before the next level's sweeps
    a.stats = dstats;
    {
        const cudaError_t e = launch_small_level(dim, ap != nullptr, a, ls);
        if (e == cudaErrorCooperativeLaunchTooLarge || e == cudaErrorNotSupported) {
            // the grid cannot be co-resident here (e.g. the GPU is shared): the
            // caller runs the tiled path instead
            cudaGetLastError();
            return MM_ERR_UNSUPPORTED;
        }
        MM_CU(e, "small level");
    }
    if (mode == 0) {
        *res = (K & 1) ? x1 : x0;
        *nsw = K;
        return MM_OK;
    }
    int32_t h[3] = {0, 0, 0};
    MM_CU(cudaMemcpyAsync(h, sb.flags, sizeof(h), cudaMemcpyDeviceToHost, ls), "small level d2h");
    MM_CU(cudaStreamSynchronize(ls), "small level sync");
    if (h[1]) {
        set_err("mm_layout_schedule: non-finite coordinate produced");
        return MM_ERR_NONFINITE;
    }
    *res = h[2] ? x1 : x0;
    *nsw = h[0];
    return MM_OK;
}

// Fixed alpha and sweep counts (BASELINE.json configs): the K sweeps of a
// level are one cached CUDA graph (or, for a small level, one persistent kernel).
struct FixedRunner : Runner {
    float alpha;
    const int32_t* sweeps;
    int32_t nsweeps;
    mm_status run(const mm_sset* S, int dim, float q, const mm_approx* ap, const float* src, float* A, float* B,
                  mm_sweep_stats* dstats, const SweepBufs& sb, cudaStream_t ls, int32_t level, bool,
                  const float** res, int32_t* nsw) override {
        const int32_t K = sweeps[std::min(level, nsweeps - 1)];
        if (K >= 1 && small_level_ok(dim, S->n, ap ? ap->k : 0, ap != nullptr)) {
            const mm_status st = run_small(S, dim, q, ap, src, A, B, dstats, sb, ls, 0, K, alpha, nullptr, res, nsw);
            if (st != MM_ERR_UNSUPPORTED) return st;
        }
        MM_CU(run_sweeps(S, dim, alpha, q, ap, src, A, B, K, dstats, sb, ls, res), "mm_layout sweeps");
        *nsw = K;
        return MM_OK;
    }
};

// The paper's schedule (readings R1-R4): rounds of at
// most `a` sweeps per alpha, cut short when the relative change < eps, alpha
// <- max(factor alpha, alpha_min); at alpha_min until converged (or the cap).
// Each decision needs the relative change of the sweep just run: the fused
// stats are read back after every sweep (one small D2H + sync per sweep).
// ------------------------------------------------------------------ device-driven schedule loop
// The schedule of one level as ONE CUDA graph: a conditional WHILE
// node whose body runs a sweep, a one-thread decision kernel that applies the
// schedule's rules to the sweep's fused statistics in device memory, and a
// conditional IF node holding the second (ping-pong) sweep and decision.  The
// decisions are the host runner's, in the same double arithmetic, so the
// sweep count and every alpha are identical; the host waits once per level
// instead of once per sweep.
struct SchedDev {
    double alpha;
    int32_t it, max_it, fin, done, err, count, cur, pad;
};
__device__ SchedDev g_sched_state;

__global__ void k_sched_init(SchedDev* s, double alpha, double alpha_min, int32_t a, int32_t max_final) {
    s->alpha = alpha;
    s->it = 0;
    s->fin = alpha <= alpha_min;
    s->max_it = s->fin ? max_final : a;
    s->done = 0;
    s->err = 0;
    s->count = 0;
    s->cur = 0;
}

__global__ void k_sched_decide(SchedDev* s, const mm_sweep_stats* st, double alpha_min, double factor, double eps,
                               int32_t a, int32_t max_final, cudaGraphConditionalHandle h_while,
                               cudaGraphConditionalHandle h_if, int set_if) {
    if (!s->done) {
        s->count += 1;
        s->cur ^= 1;
        if (st->flags & 1) {
            s->err = 1;
            s->done = 1;
        } else {
            const double rel = st->x2 > 0 ? sqrt(st->dx2) / sqrt(st->x2) : INFINITY;
            s->it += 1;
            if (rel < eps || s->it >= s->max_it) {  // round over (converged or a sweeps done)
                if (s->fin) {
                    s->done = 1;
                } else {
                    s->alpha = fmax(s->alpha * factor, alpha_min);
                    s->it = 0;
                    s->fin = s->alpha <= alpha_min;
                    s->max_it = s->fin ? max_final : a;
                }
            }
        }
    }
    const unsigned go = s->done ? 0u : 1u;
    cudaGraphSetConditional(h_while, go);
    if (set_if) cudaGraphSetConditional(h_if, go);
}

struct ScheduleRunner : Runner {
    mm_schedule sch;
    mm_status run_graph(const mm_sset* S, int dim, float q, const mm_approx* ap, const float* src, float* A,
                        float* B, mm_sweep_stats* dstats, const SweepBufs& sb, cudaStream_t ls, bool start_at_min,
                        const float** res, int32_t* nsw) {
        const int st_w = stride_of(dim);
        const size_t xbytes = (size_t)S->n * st_w * sizeof(float);
        // the loop state lives in a fixed device symbol (layouts are serialised
        // by the driver's stream lock), so the graph can be cached and relaunched
        SchedDev* sd = nullptr;
        MM_CU(cudaGetSymbolAddress((void**)&sd, g_sched_state), "mm_layout_schedule state");
        const double alpha0 = start_at_min ? sch.alpha_min : sch.alpha0;
        {
            LaunchScope lsc("sched_init", ls);
            k_sched_init<<<1, 1, 0, ls>>>(sd, alpha0, sch.alpha_min, sch.a, sch.max_final_iters);
        }
        MM_CU(cudaGetLastError(), "mm_layout_schedule init");
        // ping-pong P -> Q -> P ...; a src outside {A, B} is copied into B first
        float* P;
        float* Q;
        if (src == A) {
            P = A;
            Q = B;
        } else {
            if (src != B) MM_CU(cudaMemcpyAsync(B, src, xbytes, cudaMemcpyDeviceToDevice, ls), "mm_layout_schedule copy");
            P = B;
            Q = A;
        }
        const double* ad = &sd->alpha;
        GraphKey key = make_key(S, dim, (float)alpha0, q, ap, P, A, B, 0, dstats, sb, ls);
        key.kind = 1;
        key.si[0] = sch.a;
        key.si[1] = sch.max_final_iters;
        key.sd[0] = sch.alpha_min;
        key.sd[1] = sch.factor;
        key.sd[2] = sch.eps;
        const int64_t c0 = g_launches.load();
        cudaGraphExec_t cached = graph_cache_find(key);  // adds one sweep's kernels (k_half)
        SchedDev h{};
        if (cached) {
            const int64_t k_half = g_launches.load() - c0;
            cudaError_t e = cudaGraphLaunch(cached, ls);
            if (e == cudaSuccess) e = cudaMemcpyAsync(&h, sd, sizeof(h), cudaMemcpyDeviceToHost, ls);
            if (e == cudaSuccess) e = cudaStreamSynchronize(ls);
            if (e != cudaSuccess) {
                set_err("mm_layout_schedule: schedule graph launch: %s", cudaGetErrorString(e));
                return MM_ERR_CUDA;
            }
            g_launches.fetch_add((int64_t)h.count * k_half - k_half, std::memory_order_relaxed);
            return finish(h, P, Q, res, nsw);
        }
        const int64_t l0 = g_launches.load();
        cudaGraph_t g = nullptr;
        cudaGraphExec_t exec = nullptr;
        cudaError_t e = cudaGraphCreate(&g, 0);
        cudaGraphConditionalHandle hw = 0, hi = 0;
        cudaGraphNodeParams wp = {};
        cudaGraphNode_t wn = nullptr;
        if (e == cudaSuccess) e = cudaGraphConditionalHandleCreate(&hw, g, 1, cudaGraphCondAssignDefault);
        if (e == cudaSuccess) {
            wp.type = cudaGraphNodeTypeConditional;
            wp.conditional.handle = hw;
            wp.conditional.type = cudaGraphCondTypeWhile;
            wp.conditional.size = 1;
            e = cudaGraphAddNode(&wn, g, nullptr, 0, &wp);
        }
        cudaGraph_t body = e == cudaSuccess ? wp.conditional.phGraph_out[0] : nullptr;
        if (e == cudaSuccess) e = cudaGraphConditionalHandleCreate(&hi, body, 0, cudaGraphCondAssignDefault);
        const double amin = sch.alpha_min, fac = sch.factor, eps = sch.eps;
        const int32_t a = sch.a, mf = sch.max_final_iters;
        cudaGraph_t cap = nullptr;
        if (e == cudaSuccess)
            e = cudaStreamBeginCaptureToGraph(ls, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
        if (e == cudaSuccess) {
            cudaError_t ec = sweep_core(S, dim, (float)alpha0, q, ap, P, Q, dstats, sb, ls, ad);
            if (ec == cudaSuccess) {
                LaunchScope lsc("sched_decide", ls);
                k_sched_decide<<<1, 1, 0, ls>>>(sd, dstats, amin, fac, eps, a, mf, hw, hi, 1);
                ec = cudaGetLastError();
            }
            // the IF node after the first decision, spliced into the capture
            cudaGraphNodeParams ip = {};
            cudaGraphNode_t in = nullptr;
            if (ec == cudaSuccess) {
                cudaStreamCaptureStatus cs;
                cudaGraph_t cg = nullptr;
                const cudaGraphNode_t* deps = nullptr;
                size_t nd = 0;
                ec = cudaStreamGetCaptureInfo(ls, &cs, nullptr, &cg, &deps, &nd);
                if (ec == cudaSuccess) {
                    ip.type = cudaGraphNodeTypeConditional;
                    ip.conditional.handle = hi;
                    ip.conditional.type = cudaGraphCondTypeIf;
                    ip.conditional.size = 1;
                    ec = cudaGraphAddNode(&in, cg, deps, nd, &ip);
                }
                if (ec == cudaSuccess) ec = cudaStreamUpdateCaptureDependencies(ls, &in, 1, cudaStreamSetCaptureDependencies);
            }
            e = cudaStreamEndCapture(ls, &cap);
            if (ec != cudaSuccess) e = ec;
            if (e == cudaSuccess) {
                e = cudaStreamBeginCaptureToGraph(ls, ip.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                                  cudaStreamCaptureModeThreadLocal);
                if (e == cudaSuccess) {
                    ec = sweep_core(S, dim, (float)alpha0, q, ap, Q, P, dstats, sb, ls, ad);
                    if (ec == cudaSuccess) {
                        LaunchScope lsc("sched_decide", ls);
                        k_sched_decide<<<1, 1, 0, ls>>>(sd, dstats, amin, fac, eps, a, mf, hw, hi, 0);
                        ec = cudaGetLastError();
                    }
                    e = cudaStreamEndCapture(ls, &cap);
                    if (ec != cudaSuccess) e = ec;
                }
            }
        }
        if (e == cudaSuccess) e = cudaGraphInstantiate(&exec, g, 0);
        if (g) cudaGraphDestroy(g);
        // kernels per sweep (+ its decision): the capture counted both halves once
        const int64_t k_half = (g_launches.load() - l0) / 2;
        if (e == cudaSuccess) e = cudaGraphLaunch(exec, ls);
        if (e == cudaSuccess) e = cudaMemcpyAsync(&h, sd, sizeof(h), cudaMemcpyDeviceToHost, ls);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ls);
        if (e != cudaSuccess) {
            if (exec) cudaGraphExecDestroy(exec);
            cudaGetLastError();
            set_err("mm_layout_schedule: device-driven schedule graph: %s", cudaGetErrorString(e));
            return MM_ERR_CUDA;
        }
        graph_cache_insert(key, exec, k_half);
        g_launches.fetch_add((int64_t)h.count * k_half - 2 * k_half, std::memory_order_relaxed);
        return finish(h, P, Q, res, nsw);
    }
    static mm_status finish(const SchedDev& h, float* P, float* Q, const float** res, int32_t* nsw) {
        if (h.err) {
            set_err("mm_layout_schedule: non-finite coordinate produced");
            return MM_ERR_NONFINITE;
        }
        *res = (h.count & 1) ? Q : P;
        *nsw = h.count;
        return MM_OK;
    }
    mm_status run(const mm_sset* S, int dim, float q, const mm_approx* ap, const float* src, float* A, float* B,
                  mm_sweep_stats* dstats, const SweepBufs& sb, cudaStream_t ls, int32_t, bool start_at_min,
                  const float** res, int32_t* nsw) override {
        // one graph per level, the host waiting once (MM_SCHED_GRAPH=0: host loop)
        static const bool dev_loop = [] {
            const char* e = getenv("MM_SCHED_GRAPH");
            return !(e && e[0] == '0');
        }();
        if (sch.a >= 1 && sch.max_final_iters >= 1 && small_level_ok(dim, S->n, ap ? ap->k : 0, ap != nullptr)) {
            const mm_status st = run_small(S, dim, q, ap, src, A, B, dstats, sb, ls, 1, 0,
                                           start_at_min ? sch.alpha_min : sch.alpha0, &sch, res, nsw);
            if (st != MM_ERR_UNSUPPORTED) return st;
        }
        if (dev_loop && graphs_enabled() && sch.a >= 1 && sch.max_final_iters >= 1)
            return run_graph(S, dim, q, ap, src, A, B, dstats, sb, ls, start_at_min, res, nsw);
        double alpha = start_at_min ? sch.alpha_min : sch.alpha0;
        const float* cur = src;
        int32_t count = 0;
        mm_sweep_stats hs;
        for (;;) {
            const bool final = alpha <= sch.alpha_min;
            const int32_t max_it = final ? sch.max_final_iters : sch.a;
            for (int32_t it = 0; it < max_it; ++it) {
                float* dst = (cur == A) ? B : A;
                MM_CU(sweep_core(S, dim, (float)alpha, q, ap, cur, dst, dstats, sb, ls), "mm_layout_schedule sweep");
                MM_CU(cudaMemcpyAsync(&hs, dstats, sizeof(hs), cudaMemcpyDeviceToHost, ls), "mm_layout_schedule d2h");
                MM_CU(cudaStreamSynchronize(ls), "mm_layout_schedule sync");
                cur = dst;
                ++count;
                if (hs.flags & 1) {
                    set_err("mm_layout_schedule: non-finite coordinate produced");
                    return MM_ERR_NONFINITE;
                }
                const double rel = hs.x2 > 0 ? sqrt(hs.dx2) / sqrt(hs.x2) : INFINITY;
                if (rel < sch.eps) break;
            }
            if (final) break;
            alpha = std::max(alpha * sch.factor, sch.alpha_min);
        }
        *res = cur;
        *nsw = count;
        return MM_OK;
    }
};

// Shared multilevel / single-level driver of mm_layout and mm_layout_schedule.
// flags: MM_LAYOUT_MULTILEVEL (hierarchy + prolongation, exact when h = 0,
// Eq.(3) with h' = min(h, L - l) otherwise), MM_LAYOUT_DYNAMIC (finest level
// only, from x_init, starting at alpha_min, hierarchy stopped after h levels).
mm_status layout_impl(const mm_graph* g, const mm_sset* S, int dim, float q, int h, Runner& run, double alpha_energy,
                      uint64_t seed, int32_t n_stop, int flags, const float* x_init, float* x_out,
                      mm_layout_report* rep, cudaStream_t us, const char* who) {
    mm_status s;
    const bool multilevel = (flags & MM_LAYOUT_MULTILEVEL) != 0, dynamic = (flags & MM_LAYOUT_DYNAMIC) != 0;
    const int32_t n0 = S->n;
    const int st_w = stride_of(dim);
    const size_t xbytes = (size_t)n0 * st_w * sizeof(float);
    cudaEvent_t ev = nullptr;
    // the driver's own non-blocking stream per device (persistent, so that
    // stream-ordered workspace reuse and the graph cache see the same addresses
    // call after call); the state lock serialises layouts (see g_state_mu)
    constexpr int kMaxDevices = 64;
    static cudaStream_t s_ls[kMaxDevices] = {};
    std::lock_guard<std::recursive_mutex> state_lock(g_state_mu);
    int dev = 0;
    MM_CU(cudaGetDevice(&dev), "mm_layout device");
    if (dev < 0 || dev >= kMaxDevices) { set_err("%s: device ordinal %d >= %d", who, dev, kMaxDevices); return MM_ERR_UNSUPPORTED; }
    if (!s_ls[dev]) MM_CU(cudaStreamCreateWithFlags(&s_ls[dev], cudaStreamNonBlocking), "mm_layout stream");
    cudaStream_t ls = s_ls[dev];
    struct StreamGuard {
        cudaStream_t s;
        cudaEvent_t e;
        ~StreamGuard() {
            if (s) cudaStreamSynchronize(s);
            if (e) cudaEventDestroy(e);
        }
    } guard{ls, nullptr};
    MM_CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "mm_layout event");
    guard.e = ev;
    MM_CU(cudaEventRecord(ev, us), "mm_layout event");
    MM_CU(cudaStreamWaitEvent(ls, ev, 0), "mm_layout wait");

    mm_layout_report R;
    memset(&R, 0, sizeof(R));
    trace("layout: begin");

    if (!multilevel && !dynamic) {
        const double mean_row = (double)S->nnz / n0;
        const size_t need = sweep_bytes(n0, dim, 0, false, mean_row) + al(xbytes) + al(sizeof(mm_sweep_stats));
        DevBuf buf(need, ls);
        if (!buf.p) { set_err("%s: out of device memory (%zu B)", who, need); return MM_ERR_OUT_OF_MEMORY; }
        Carver cv(buf.p, need);
        float* tmpx = cv.take<float>((size_t)n0 * st_w);
        mm_sweep_stats* dstats = cv.take<mm_sweep_stats>(1);
        SweepBufs sb;
        if (!carve_sweep(cv, n0, dim, 0, false, mean_row, sb)) { set_err("%s: carving failed", who); return MM_ERR_INVALID_ARGUMENT; }
        MM_CU(cudaMemsetAsync(sb.flags, 0, 4 * sizeof(int32_t), ls), "mm_layout memset");
        MM_CU(cudaMemsetAsync(dstats, 0, sizeof(mm_sweep_stats), ls), "mm_layout memset");
        const float* src = x_init;
        float *A = x_out, *B = tmpx;
        const char *pi = (const char*)x_init, *po = (const char*)x_out;
        if (pi == po) {  // in-place request: iterate from a copy (Jacobi needs two buffers)
            MM_CU(cudaMemcpyAsync(tmpx, x_init, xbytes, cudaMemcpyDeviceToDevice, ls), "mm_layout copy");
            src = tmpx;
        } else if (pi < po + xbytes && po < pi + xbytes) {
            set_err("%s: x_init partially overlaps x_out", who);
            return MM_ERR_INVALID_ARGUMENT;
        }
        const float* res = nullptr;
        int32_t nsw = 0;
        trace("layout: sweeps enqueue");
        if ((s = run.run(S, dim, q, nullptr, src, A, B, dstats, sb, ls, 0, false, &res, &nsw)) != MM_OK) return s;
        trace("layout: sweeps enqueued");
        if (res != x_out) MM_CU(cudaMemcpyAsync(x_out, res, xbytes, cudaMemcpyDeviceToDevice, ls), "mm_layout copy");
        mm_sweep_stats hs;
        MM_CU(cudaMemcpyAsync(&hs, dstats, sizeof(hs), cudaMemcpyDeviceToHost, ls), "mm_layout d2h");
        MM_CU(cudaStreamSynchronize(ls), "mm_layout sync");
        trace("layout: sweeps done (synced)");
        R.levels = 1;
        R.n_level[0] = n0;
        R.sweeps_level[0] = nsw;
        R.rel_change = hs.x2 > 0 ? sqrt(hs.dx2 / hs.x2) : INFINITY;
        R.vertex_updates = (int64_t)n0 * nsw;
        R.pair_interactions = (int64_t)n0 * (n0 - 1) * nsw;
        if (hs.flags & 1) { set_err("%s: non-finite coordinate produced", who); return MM_ERR_NONFINITE; }
    } else {
        mm_hierarchy* H = nullptr;
        // dynamic update: "stop the coarsening process after the computation of h levels"
        const int32_t max_levels = dynamic ? std::min(h + 1, (int)MM_MAX_LEVELS) : MM_MAX_LEVELS;
        HierMode hm;
        hm.sclap = (flags & MM_LAYOUT_SCLAP) != 0;
        if ((s = build_hierarchy_impl(g, nullptr, dim, seed, dynamic ? 1 : n_stop, max_levels, 64, &H, ls, hm)) !=
            MM_OK)
            return s;
        struct HGuard {
            mm_hierarchy* h;
            ~HGuard() { mm_hierarchy_free(h); }
        } hg{H};
        const int32_t nl = (int32_t)H->lv.size(), L = nl - 1;
        R.levels = nl;
        auto S_of = [&](int32_t l) {
            mm_sset t;
            if (l == 0) return *S;
            t.n = H->lv[l].n;
            t.nnz = H->lv[l].nnz;
            t.row_ptr = H->lv[l].rp;
            t.col = H->lv[l].col;
            t.d = H->lv[l].d;
            t.w = H->lv[l].w;
            return t;
        };
        const int32_t lo_level = 0, hi_level = dynamic ? 0 : L;  // levels optimized
        // workspace = max over the optimized levels
        size_t wsb = 0;
        for (int32_t l = lo_level; l <= hi_level; ++l) {
            const int32_t hp = std::min(h, L - l);
            const int32_t k = hp > 0 ? H->lv[l + hp].n : 0;
            wsb = std::max(wsb, sweep_bytes(H->lv[l].n, dim, k, hp > 0, 1.0));
        }
        const size_t need = wsb + 2 * al(xbytes) + 2 * al((size_t)n0 * 4) + al(sizeof(mm_sweep_stats)) + al(64);
        // locality renumbering of the Eq.(3) levels that run on the tiled path
        size_t rnb = 0;
        if (renumber_enabled()) {
            for (int32_t l = lo_level; l <= hi_level; ++l) {
                const int32_t hp = std::min(h, L - l);
                if (hp <= 0) continue;
                const int32_t k = H->lv[l + hp].n;
                if (small_level_ok(dim, H->lv[l].n, k, true)) continue;
                const int64_t nnz_l = l == 0 ? S->nnz : H->lv[l].nnz;
                rnb = std::max(rnb, renumber_bytes(H->lv[l].n, nnz_l, k));
            }
        }
        DevBuf rbuf(rnb, ls);
        if (rnb && !rbuf.p) { set_err("%s: out of device memory (%zu B)", who, rnb); return MM_ERR_OUT_OF_MEMORY; }
        DevBuf buf(need, ls);
        if (!buf.p) { set_err("%s: out of device memory (%zu B)", who, need); return MM_ERR_OUT_OF_MEMORY; }
        Carver cv(buf.p, need);
        float* xa = cv.take<float>((size_t)n0 * st_w);
        float* xb = cv.take<float>((size_t)n0 * st_w);
        int32_t* anc = cv.take<int32_t>(n0);
        int32_t* anc2 = cv.take<int32_t>(n0);
        mm_sweep_stats* dstats = cv.take<mm_sweep_stats>(1);
        double* dsum = cv.take<double>(8);
        const size_t ws_off = cv.off;
        MM_CU(cudaMemsetAsync(dstats, 0, sizeof(mm_sweep_stats), ls), "mm_layout memset");
        const float* cur = nullptr;
        if (dynamic) {
            MM_CU(cudaMemcpyAsync(xa, x_init, xbytes, cudaMemcpyDeviceToDevice, ls), "mm_layout copy");
            cur = xa;
        } else {
            // coarsest level: box init (Q14), then the level's sweeps (exact, Q13)
            mm_sset SL = S_of(L);
            MM_CU(launch_init_box(dim, SL.n, SL.d, SL.nnz, dsum, seed, L, xa, ls), "mm_layout init");
            cur = xa;
        }
        for (int32_t l = hi_level; l >= lo_level; --l) {
            const int32_t nf = H->lv[l].n;
            if (!dynamic && l < L) {
                float* dst = (cur == xa) ? xb : xa;
                if (flags & MM_LAYOUT_DISC_PROLONG)
                    MM_CU(launch_prolong_disc(dim, nf, H->lv[l].parent, cur, H->lv[l + 1].c, seed, l, dst, ls),
                          "mm_layout prolong");
                else
                    MM_CU(launch_prolong(dim, nf, H->lv[l].parent, cur, seed, l, dst, ls), "mm_layout prolong");
                cur = dst;
            }
            const int32_t hp = std::min(h, L - l);
            mm_approx ap;
            mm_approx* app = nullptr;
            if (hp > 0) {
                // H = parent_{l+hp-1} o ... o parent_l
                MM_CU(cudaMemcpyAsync(anc, H->lv[l].parent, 4 * (size_t)nf, cudaMemcpyDeviceToDevice, ls), "mm_layout anc");
                for (int32_t t = 1; t < hp; ++t) {
                    MM_CU(launch_compose(nf, anc, H->lv[l + t].parent, anc2, ls), "mm_layout compose");
                    std::swap(anc, anc2);
                }
                ap.k = H->lv[l + hp].n;
                ap.parent = H->lv[l].parent;
                ap.ancestor = anc;
                app = &ap;
            }
            mm_sset Sl = S_of(l);
            Carver wl((char*)buf.p + ws_off, need - ws_off);
            SweepBufs sbl;
            if (!carve_sweep(wl, nf, dim, app ? ap.k : 0, app != nullptr, 1.0, sbl)) {
                set_err("%s: carving failed", who);
                return MM_ERR_INVALID_ARGUMENT;
            }
            MM_CU(cudaMemsetAsync(sbl.flags, 0, 4 * sizeof(int32_t), ls), "mm_layout memset");
            if (app) MM_CU(prepare_approx(nf, dim, app, cur, sbl, ls), "mm_layout prepare_approx");
            float* other = (cur == xa) ? xb : xa;
            const float* res = nullptr;
            int32_t nsw = 0;
            const bool renum = app && rnb > 0 && !small_level_ok(dim, nf, ap.k, true);
            if (renum) {
                // vertices in representative-slot order (k_perm.cuh): permute S^l, the
                // maps and x, redo the maps / orders there, sweep, scatter x back
                Carver rc(rbuf.p, rnb);
                int32_t* perm = rc.take<int32_t>(nf);
                int32_t* inv = rc.take<int32_t>(nf);
                int32_t* anc_r = rc.take<int32_t>(nf);
                int32_t* par_r = rc.take<int32_t>(nf);
                int32_t* sib = rc.take<int32_t>(nf);
                int32_t* len = rc.take<int32_t>(nf);
                int32_t* cnt = rc.take<int32_t>(ap.k + 1);
                int32_t* sptr = rc.take<int32_t>(ap.k + 1);
                int64_t* rp_r = rc.take<int64_t>((size_t)nf + 1);
                int32_t* col_r = rc.take<int32_t>((size_t)Sl.nnz);
                float* d_r = rc.take<float>((size_t)Sl.nnz);
                float* w_r = rc.take<float>((size_t)Sl.nnz);
                void* stmp = rc.take<char>(perm_scan_tmp_bytes((int64_t)std::max(nf, ap.k) + 1));
                if (!rc.ok) { set_err("%s: renumber carving failed", who); return MM_ERR_INVALID_ARGUMENT; }
                if (renumber_mode() == 2) {
                    MM_CU(cudaMemcpyAsync(perm, sbl.tperm, 4 * (size_t)nf, cudaMemcpyDeviceToDevice, ls), "renumber");
                    MM_CU(cudaMemcpyAsync(inv, sbl.tpos, 4 * (size_t)nf, cudaMemcpyDeviceToDevice, ls), "renumber");
                    MM_CU(gather_i32(nf, perm, ap.ancestor, anc_r, ls), "mm_layout renumber");
                } else {
                    MM_CU(level_perm(ap.k, sbl.rord, sbl.mptr, sbl.mem, cnt, sptr, perm, inv, anc_r, stmp, ls),
                          "mm_layout renumber");
                }
                MM_CU(permute_sset(nf, Sl.row_ptr, Sl.col, Sl.d, Sl.w, perm, inv, rp_r, col_r, d_r, w_r, len, stmp, ls),
                      "mm_layout renumber");
                MM_CU(gather_i32(nf, perm, ap.parent, par_r, ls), "mm_layout renumber");
                MM_CU(permute_x(dim, nf, perm, cur, other, false, ls), "mm_layout renumber");
                mm_sset Sr = Sl;
                Sr.row_ptr = rp_r;
                Sr.col = col_r;
                Sr.d = d_r;
                Sr.w = w_r;
                mm_approx apr;
                apr.k = ap.k;
                apr.parent = par_r;
                apr.ancestor = anc_r;
                // members of every representative are now one contiguous range (mem = identity)
                sbl.contig = renumber_mode() != 2;
                MM_CU(prepare_approx(nf, dim, &apr, other, sbl, ls), "mm_layout prepare_approx");
                MM_CU(sibling_of(nf, sbl.cptr, sbl.child, sib, ls), "mm_layout renumber");
                sbl.sib = sib;
                if ((s = run.run(&Sr, dim, q, &apr, other, (float*)cur, other, dstats, sbl, ls, l, dynamic, &res,
                                 &nsw)) != MM_OK)
                    return s;
                float* back = (res == cur) ? other : (float*)cur;
                MM_CU(permute_x(dim, nf, perm, res, back, true, ls), "mm_layout renumber");
                res = back;
            } else if ((s = run.run(&Sl, dim, q, app, cur, other, (float*)cur, dstats, sbl, ls, l, dynamic, &res,
                                    &nsw)) != MM_OK) {
                return s;
            }
            if (trace_on()) {
                char msg[160];
                snprintf(msg, sizeof(msg), "layout: level %d done (n %d, k %d, %d sweeps enqueued)", l, nf,
                         app ? ap.k : 0, nsw);
                trace(msg);
            }
            cur = res;
            R.n_level[l] = nf;
            R.k_level[l] = app ? ap.k : 0;
            R.sweeps_level[l] = nsw;
            R.vertex_updates += (int64_t)nf * nsw;
            if (app)
                R.pair_interactions += ((int64_t)nf * (ap.k - 1) + 2 * (int64_t)(nf - H->lv[l + 1].n)) * nsw;
            else
                R.pair_interactions += (int64_t)nf * (nf - 1) * nsw;
        }
        MM_CU(cudaMemcpyAsync(x_out, cur, xbytes, cudaMemcpyDeviceToDevice, ls), "mm_layout copy");
        mm_sweep_stats hs;
        MM_CU(cudaMemcpyAsync(&hs, dstats, sizeof(hs), cudaMemcpyDeviceToHost, ls), "mm_layout d2h");
        MM_CU(cudaStreamSynchronize(ls), "mm_layout sync");
        R.rel_change = hs.x2 > 0 ? sqrt(hs.dx2 / hs.x2) : INFINITY;
        if (hs.flags & 1) { set_err("%s: non-finite coordinate produced", who); return MM_ERR_NONFINITE; }
    }
    double en[3] = {0, 0, 0};
    int64_t coinc = 0;
    trace("layout: energy begin");
    s = energy_core(S, dim, alpha_energy, q, x_out, en, ls, false, &coinc);
    trace("layout: energy done");
    R.coincident_pairs = coinc;
    R.stress = en[0];
    R.entropy = en[1];
    R.energy = en[2];
    if (rep) *rep = R;
    // the caller's stream observes x_out only after our private stream finished
    MM_CU(cudaEventRecord(ev, ls), "mm_layout event");
    MM_CU(cudaStreamWaitEvent(us, ev, 0), "mm_layout wait");
    return s;
}

}  // namespace

extern "C" mm_status mm_layout(const mm_graph* g, const mm_sset* S, int dim, float alpha, float q, int h,
                               const int32_t* sweeps, int32_t nsweeps, uint64_t seed, int32_t n_stop,
                               const float* x_init, float* x_out, mm_layout_report* rep, mm_stream_t stream) {
    mm_status s;
    if ((s = check_sset(S, "mm_layout")) != MM_OK) return s;
    if ((s = check_dim_q(dim, q, "mm_layout")) != MM_OK) return s;
    if ((s = check_x(x_out, dim, "x_out", "mm_layout")) != MM_OK) return s;
    if (!sweeps || nsweeps < 1 || h < 0 || !isfinite(alpha)) {
        set_err("mm_layout: bad arguments (sweeps host array with nsweeps >= 1, h >= 0, finite alpha)");
        return MM_ERR_INVALID_ARGUMENT;
    }
    for (int32_t t = 0; t < nsweeps; ++t)
        if (sweeps[t] < 0) { set_err("mm_layout: negative sweep count"); return MM_ERR_INVALID_ARGUMENT; }
    if (h == 0 && (s = check_x(x_init, dim, "x_init", "mm_layout")) != MM_OK) return s;
    if (h > 0) {
        if ((s = check_graph(g, "mm_layout")) != MM_OK) return s;
        if (g->n != S->n) { set_err("mm_layout: graph and S sizes differ"); return MM_ERR_INVALID_ARGUMENT; }
        if (n_stop < 1) { set_err("mm_layout: n_stop must be >= 1"); return MM_ERR_INVALID_ARGUMENT; }
    }
    FixedRunner fr;
    fr.alpha = alpha;
    fr.sweeps = sweeps;
    fr.nsweeps = nsweeps;
    return layout_impl(g, S, dim, q, h, fr, alpha, seed, n_stop, h > 0 ? MM_LAYOUT_MULTILEVEL : 0, x_init, x_out, rep,
                       (cudaStream_t)stream, "mm_layout");
}

extern "C" mm_status mm_sweeps(const mm_sset* S, int dim, float alpha, float q, const mm_approx* ap,
                               const float* x_in, float* x_out, int32_t K, mm_sweep_stats* stats,
                               mm_stream_t stream) {
    mm_status s;
    const char* who = "mm_sweeps";
    if ((s = check_sset(S, who)) != MM_OK) return s;
    if ((s = check_dim_q(dim, q, who)) != MM_OK) return s;
    if ((s = check_x(x_in, dim, "x_in", who)) != MM_OK) return s;
    if ((s = check_x(x_out, dim, "x_out", who)) != MM_OK) return s;
    const int32_t n = S->n;
    const size_t xbytes = (size_t)n * stride_of(dim) * sizeof(float);
    const char *a0 = (const char*)x_in, *b0 = (const char*)x_out;
    if (a0 < b0 + xbytes && b0 < a0 + xbytes) { set_err("%s: x_out must not alias x_in", who); return MM_ERR_INVALID_ARGUMENT; }
    if (K < 0 || !isfinite(alpha)) { set_err("%s: K >= 0 and a finite alpha required", who); return MM_ERR_INVALID_ARGUMENT; }
    if (ap && (ap->k <= 0 || ap->k > n || !ap->parent || !ap->ancestor)) {
        set_err("%s: bad mm_approx (k=%d must be in [1, n], maps non-NULL)", who, ap->k);
        return MM_ERR_INVALID_ARGUMENT;
    }
    cudaStream_t st = (cudaStream_t)stream;
    // the persistent small-level kernel keeps its grid-barrier state in device symbols
    std::lock_guard<std::recursive_mutex> state_lock(g_state_mu);
    const double mean_row = (double)S->nnz / (double)n;
    const size_t need = sweep_bytes(n, dim, ap ? ap->k : 0, ap != nullptr, mean_row) + al(xbytes) +
                        al(sizeof(mm_sweep_stats));
    DevBuf buf(need, st);
    if (!buf.p) { set_err("%s: out of device memory (%zu B)", who, need); return MM_ERR_OUT_OF_MEMORY; }
    Carver cv(buf.p, need);
    float* tmpx = cv.take<float>(xbytes / sizeof(float));
    mm_sweep_stats* dstats = cv.take<mm_sweep_stats>(1);
    SweepBufs sb;
    if (!carve_sweep(cv, n, dim, ap ? ap->k : 0, ap != nullptr, mean_row, sb)) {
        set_err("%s: carving failed", who);
        return MM_ERR_INVALID_ARGUMENT;
    }
    MM_CU(cudaMemsetAsync(sb.flags, 0, 4 * sizeof(int32_t), st), "mm_sweeps memset");
    MM_CU(cudaMemsetAsync(dstats, 0, sizeof(mm_sweep_stats), st), "mm_sweeps memset");
    const float* res = x_in;
    if (K > 0) {
        if (ap) MM_CU(prepare_approx(n, dim, ap, x_in, sb, st), "mm_sweeps prepare_approx");
        int32_t nsw = 0;
        s = MM_ERR_UNSUPPORTED;
        if (small_level_ok(dim, n, ap ? ap->k : 0, ap != nullptr))
            s = run_small(S, dim, q, ap, x_in, x_out, tmpx, dstats, sb, st, 0, K, alpha, nullptr, &res, &nsw);
        if (s == MM_ERR_UNSUPPORTED)
            MM_CU(run_sweeps(S, dim, alpha, q, ap, x_in, x_out, tmpx, K, dstats, sb, st, &res), "mm_sweeps");
        else if (s != MM_OK)
            return s;
    }
    if (res != x_out) MM_CU(cudaMemcpyAsync(x_out, res, xbytes, cudaMemcpyDeviceToDevice, st), "mm_sweeps copy");
    if (stats) MM_CU(cudaMemcpyAsync(stats, dstats, sizeof(mm_sweep_stats), cudaMemcpyDeviceToDevice, st), "mm_sweeps stats");
    mm_sweep_stats hs;
    MM_CU(cudaMemcpyAsync(&hs, dstats, sizeof(hs), cudaMemcpyDeviceToHost, st), "mm_sweeps d2h");
    MM_CU(cudaStreamSynchronize(st), "mm_sweeps sync");
    if (hs.flags & 1) { set_err("%s: non-finite coordinate produced", who); return MM_ERR_NONFINITE; }
    return MM_OK;
}

extern "C" mm_status mm_layout_schedule(const mm_graph* g, const mm_sset* S, int dim, float q, int h,
                                        const mm_schedule* sch, uint64_t seed, int32_t n_stop, int32_t flags,
                                        const float* x_init, float* x_out, mm_layout_report* rep, mm_stream_t stream) {
    mm_status s;
    const char* who = "mm_layout_schedule";
    if ((s = check_sset(S, who)) != MM_OK) return s;
    if ((s = check_dim_q(dim, q, who)) != MM_OK) return s;
    if ((s = check_x(x_out, dim, "x_out", who)) != MM_OK) return s;
    if (!sch || h < 0 || sch->a < 1 || sch->max_final_iters < 1 || !(sch->alpha_min > 0.0) ||
        !(sch->alpha0 >= sch->alpha_min) || !(sch->factor > 0.0 && sch->factor < 1.0) || !(sch->eps >= 0.0) ||
        (flags & ~(MM_LAYOUT_MULTILEVEL | MM_LAYOUT_DYNAMIC | MM_LAYOUT_SCLAP | MM_LAYOUT_DISC_PROLONG)) != 0) {
        set_err("%s: bad arguments (schedule: a >= 1, max_final_iters >= 1, 0 < alpha_min <= alpha0, "
                "0 < factor < 1, eps >= 0; h >= 0; flags)", who);
        return MM_ERR_INVALID_ARGUMENT;
    }
    const bool multilevel = (flags & MM_LAYOUT_MULTILEVEL) != 0, dynamic = (flags & MM_LAYOUT_DYNAMIC) != 0;
    if ((!multilevel || dynamic) && (s = check_x(x_init, dim, "x_init", who)) != MM_OK) return s;
    if (multilevel || dynamic) {
        if ((s = check_graph(g, who)) != MM_OK) return s;
        if (g->n != S->n) { set_err("%s: graph and S sizes differ", who); return MM_ERR_INVALID_ARGUMENT; }
        if (n_stop < 1) { set_err("%s: n_stop must be >= 1", who); return MM_ERR_INVALID_ARGUMENT; }
    }
    ScheduleRunner sr;
    sr.sch = *sch;
    return layout_impl(g, S, dim, q, h, sr, sch->alpha_min, seed, n_stop, flags, x_init, x_out, rep,
                       (cudaStream_t)stream, who);
}

// ================================================================== full stress (f4)
extern "C" mm_status mm_full_stress(const mm_graph* g, int dim, const float* x, double* out, mm_stream_t stream) {
    mm_status s;
    if ((s = check_graph(g, "mm_full_stress")) != MM_OK) return s;
    if (dim != 2 && dim != 3) { set_err("mm_full_stress: dim must be 2 or 3"); return MM_ERR_UNSUPPORTED; }
    if ((s = check_x(x, dim, "x", "mm_full_stress")) != MM_OK) return s;
    if (!out) { set_err("mm_full_stress: out is NULL"); return MM_ERR_INVALID_ARGUMENT; }
    const int32_t n = g->n;
    if (full_stress_smem(n) > 200 * 1024) {
        set_err("mm_full_stress: n = %d exceeds the shared-memory visited set (n <= 1,638,400)", n);
        return MM_ERR_UNSUPPORTED;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const int grid = full_stress_grid(n);
    const size_t bytes = al((size_t)grid * 2 * n * sizeof(int32_t)) + al((size_t)grid * 5 * sizeof(double));
    DevBuf buf(bytes, st);
    if (!buf.p) { set_err("mm_full_stress: out of device memory (%zu B)", bytes); return MM_ERR_OUT_OF_MEMORY; }
    Carver cv(buf.p, bytes);
    int32_t* qbuf = cv.take<int32_t>((size_t)grid * 2 * n);
    double* partial = cv.take<double>((size_t)grid * 5);
    MM_CU(launch_full_stress(dim, n, g->row_ptr, g->col, x, grid, qbuf, partial, st), "mm_full_stress");
    std::vector<double> h((size_t)grid * 5);
    MM_CU(cudaMemcpyAsync(h.data(), partial, h.size() * sizeof(double), cudaMemcpyDeviceToHost, st), "mm_full_stress d2h");
    MM_CU(cudaStreamSynchronize(st), "mm_full_stress sync");
    double A = 0, B = 0, C = 0, F = 0, P = 0;
    for (int b = 0; b < grid; ++b) {
        A += h[(size_t)b * 5];
        B += h[(size_t)b * 5 + 1];
        C += h[(size_t)b * 5 + 2];
        F += h[(size_t)b * 5 + 3];
        P += h[(size_t)b * 5 + 4];
    }
    const double sc = B > 0.0 ? A / B : 1.0;
    out[0] = F;
    out[1] = sc;
    out[2] = sc * sc * B - 2.0 * sc * A + C;
    out[3] = P;
    return MM_OK;
}

// ================================================================== prolongation
extern "C" mm_status mm_prolong(int32_t n_fine, int dim, const int32_t* parent, const float* xc,
                                const int32_t* c_coarse, uint64_t seed, int32_t level, float* x, mm_stream_t stream) {
    mm_status s;
    if (n_fine < 0) { set_err("mm_prolong: n_fine < 0"); return MM_ERR_INVALID_ARGUMENT; }
    if (dim != 2 && dim != 3) { set_err("mm_prolong: dim must be 2 or 3 (got %d)", dim); return MM_ERR_UNSUPPORTED; }
    if (n_fine == 0) return MM_OK;
    if (!parent) { set_err("mm_prolong: parent is NULL"); return MM_ERR_INVALID_ARGUMENT; }
    if ((s = check_x(xc, dim, "xc", "mm_prolong")) != MM_OK) return s;
    if ((s = check_x(x, dim, "x", "mm_prolong")) != MM_OK) return s;
    if (x == xc) { set_err("mm_prolong: x must not alias xc"); return MM_ERR_INVALID_ARGUMENT; }
    cudaStream_t st = (cudaStream_t)stream;
    if (c_coarse) MM_CU(launch_prolong_disc(dim, n_fine, parent, xc, c_coarse, seed, level, x, st), "mm_prolong");
    else MM_CU(launch_prolong(dim, n_fine, parent, xc, seed, level, x, st), "mm_prolong");
    return MM_OK;
}

// ================================================================== validation
extern "C" mm_status mm_validate_sset(const mm_sset* S, mm_stream_t stream) {
    mm_status s;
    if ((s = check_sset(S, "mm_validate_sset")) != MM_OK) return s;
    cudaStream_t st = (cudaStream_t)stream;
    DevBuf buf(64, st);
    if (!buf.p) { set_err("mm_validate_sset: out of device memory"); return MM_ERR_OUT_OF_MEMORY; }
    int32_t init[2] = {INT32_MAX, 0}, h[2] = {0, 0};
    MM_CU(cudaMemcpyAsync(buf.p, init, 8, cudaMemcpyHostToDevice, st), "mm_validate_sset h2d");
    MM_CU(launch_validate_sset(S->n, S->row_ptr, S->col, S->d, S->w, S->nnz, (int32_t*)buf.p, st), "mm_validate_sset");
    MM_CU(cudaMemcpyAsync(h, buf.p, 8, cudaMemcpyDeviceToHost, st), "mm_validate_sset d2h");
    MM_CU(cudaStreamSynchronize(st), "mm_validate_sset sync");
    if (h[1] == 0) return MM_OK;
    set_err("mm_validate_sset: row %d is invalid (%s%s%s%s%s%s)", h[0] - 1, (h[1] & 1) ? "row_ptr not monotone; " : "",
            (h[1] & 2) ? "col out of range; " : "", (h[1] & 4) ? "self entry; " : "",
            (h[1] & 8) ? "d <= 0 or non-finite; " : "", (h[1] & 16) ? "w < 0 or non-finite; " : "",
            (h[1] & 32) ? "rho_i <= 0" : "");
    return MM_ERR_INVALID_INPUT;
}
