// mra_api.cpp -- C ABI (include/mra.h): host plan builder + level-synchronous scheduler.
//
// Plan, built once on the host and uploaded as flat level-major SoA:
//   root = data bounding box with top/right pushed out 1%; J=4 halves both axes,
//   J=2 the longer one (ties -> x); r_hat = ceil(sqrt r) * floor(r/ceil(sqrt r))
//   knots on an offset grid; observations equal to a pre-finest knot are
//   eliminated; the rest are counting-sorted by leaf (CSR leaf_off, perm).
// Evaluation: gather y -> prior levels 1..M-1 -> for each chunk of subtrees
//   rooted at the chunk level c: bottom (leaves + level M-1 merge) and merges M-2..c ->
//   merges c-1..1 -> log L. Every arithmetic step runs in mra_kernels.cu; this file only
//   sizes buffers, launches and checks errors.
#include "../../include/mra.h"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>   // types and prototypes only: the library is dlopen'ed (nccl_api below)

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <mutex>
#include <new>
#include <string>
#include <type_traits>
#include <vector>

#include "mra_internal.h"

using namespace mra;

static thread_local std::string g_err;
static mra_status fail(mra_status s, const std::string& msg) {
    g_err = msg;
    return s;
}

// every extern "C" entry runs its body through this: no C++ exception (host std::bad_alloc from a huge
// plan, std::length_error, ...) ever crosses the C ABI (include/mra.h: "No call aborts")
template <class F>
static mra_status guarded(F&& f) {
    try {
        return f();
    } catch (const std::bad_alloc&) {
        return fail(MRA_E_OOM, "host allocation failed (std::bad_alloc)");
    } catch (const std::exception& e) {
        return fail(MRA_E_OOM, std::string("host exception: ") + e.what());
    } catch (...) {
        return fail(MRA_E_OOM, "unknown host exception");
    }
}

// ---------------------------------------------------------------- NCCL (dlopen'ed)
// The in-library exchange step of subtree sharding. NCCL is
// loaded at run time: the copy torch already mapped (libnccl.so.2 by soname), else the system one, or
// $MRA_NCCL_LIB; a missing library is MRA_E_NCCL at plan creation, not a link-time dependency.
struct NcclApi {
    decltype(&ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&ncclCommInitRank) commInitRank = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclReduce) reduce = nullptr;
    decltype(&ncclBroadcast) broadcast = nullptr;
    decltype(&ncclAllReduce) allReduce = nullptr;
    decltype(&ncclGetErrorString) errStr = nullptr;
    bool ok = false;
};
static const NcclApi* nccl_api() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* cands[3] = {getenv("MRA_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
        void* h = nullptr;
        for (const char* c : cands)
            if (c && *c && (h = dlopen(c, RTLD_NOW | RTLD_GLOBAL))) break;
        if (!h) return;
#define NSYM(f, n) api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, n))
        NSYM(getUniqueId, "ncclGetUniqueId");
        NSYM(commInitRank, "ncclCommInitRank");
        NSYM(commDestroy, "ncclCommDestroy");
        NSYM(reduce, "ncclReduce");
        NSYM(broadcast, "ncclBroadcast");
        NSYM(allReduce, "ncclAllReduce");
        NSYM(errStr, "ncclGetErrorString");
#undef NSYM
        api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.reduce && api.broadcast &&
                 api.allReduce && api.errStr;
    });
    return api.ok ? &api : nullptr;
}

struct mra_plan {
    int M = 0, J = 0, lj = 0, r = 0, rh = 0, nx = 0, ny = 0;
    double offset = 0, xs = 1, ys = 1;
    uint64_t n_in = 0;
    long long N = 0, nreg = 0, nint = 0, nleaf = 0, n_empty = 0, max_leaf = 0, max_group = 0;
    std::vector<long long> perm, leaf_off;
    std::vector<double> kx, ky;
    std::vector<double> box;         // interior region boxes (level-major, x0 x1 y0 y1)
    double root[4] = {0, 0, 0, 0};   // root domain (data bounding box, top/right + 1%)
    int device = 0, nsm = 148;
    cudaStream_t st = nullptr;
    // device state
    double *pxy = nullptr, *zs = nullptr, *zin = nullptr;
    long long *perm_d = nullptr, *leaf_off_d = nullptr;
    double* kxy_d = nullptr;
    double* prior = nullptr;
    long long prior_base[MAXM + 1] = {0};
    bool stream = false;             // prior rows of levels >= c live per chunk (NEXT-4)
    // host-y entry points: the H2D copy of y runs on its own stream while the prior levels (which do
    // not read y) run on st; st waits for it just before the gather into leaf order
    const double* host_y_pending = nullptr;
    cudaStream_t cst = nullptr;
    cudaEvent_t cev = nullptr;
    size_t dev_bytes = 0;            // device memory held by the plan
    double *dreg = nullptr, *ureg = nullptr, *loglik_d = nullptr;
    int* err = nullptr;
    unsigned long long* counters = nullptr;
    int n_counters = 0, next_counter = 0;
    // posterior-pass buffers: level m output has q_m = (m-1) rh + 1 rows
    int c = 1;                       // chunk level
    long long Kc = 1;                // level-c regions per chunk
    double* out_full[MAXM + 1] = {nullptr};   // levels 1..c: every region
    double* out_chunk[MAXM + 1] = {nullptr};  // levels c+1..M-1: one chunk
    double* ws = nullptr;
    long long ws_stride = 0;
    WsLayout L{};
    int grid = 0;
    // sharding
    int rank = 0, world = 1;
    std::vector<long long> my_c;     // level-c regions owned by this rank (sorted)
    // in-library exchange (opts.nccl_id): own communicator and exchange buffers
    bool nccl = false;
    ncclComm_t comm = nullptr;
    double* xbuf = nullptr;          // packed exchange buffer (mra_shard_size doubles)
    double* bcast = nullptr;         // [4] log L, error flag, d, u broadcast from rank 0
    double* mutop = nullptr;         // above-shard posterior means (mra_mutop_size doubles)
    double* sm_sorted = nullptr;     // smoothed values in leaf order (all-reduced across ranks)
    // device allocator hooks (opts.dalloc / dfree; NULL = cudaMalloc / cudaFree)
    void* (*ualloc)(size_t, int, void*) = nullptr;
    void (*ufree)(void*, int, void*) = nullptr;
    // posterior state
    double* post = nullptr;
    long long post_base[MAXM + 1] = {0};
    double* muhat = nullptr;
    double* mu_d = nullptr;
    double* smooth_d = nullptr;
    double* ws_smooth = nullptr;     // wide plans: per-CTA smoothing workspace sized for the largest leaf
    // prediction: posterior state of the last evaluation (valid only if it requested posterior state)
    bool post_valid = false;
    mra_theta post_theta{};
    double* ws_pred = nullptr;
    WsLayout Lp{};
    int pred_grid = 0;
    WsLayout Ls{};
    int smooth_grid = 0;
    uint64_t launches = 0;
    std::vector<void*> allocs;
    std::vector<size_t> alloc_bytes;   // parallel to allocs
    // theta lanes (NEXT-3): evaluation contexts sharing this plan's read-only device data, each with its
    // own stream and mutable buffers; mra_loglik_batch* runs one theta per lane concurrently
    std::vector<mra_plan*> lanes;
    bool is_lane = false;
    int n_lanes = 1;                   // requested evaluation contexts (opts.theta_lanes)
    cudaEvent_t lane_ev = nullptr;
    // wide (big-leaf) path
    bool wide = false;
    struct WideSub {
        long long g0 = 0, gcount = 0;
        long long chain_off = 0, chain_n = 0, sigma_off = 0, sigma_n = 0;
        long long cs_off = 0, cs_n = 0;   // fused chain + Sigma list (k_wide_chsig), cs_n = 0: separate kernels
        std::vector<long long> upd_off, upd_n, diag_off, diag_n, pf_off, pf_n, tr_off, tr_n;
        long long trsm_off = 0, trsm_n = 0, mt_off = 0, mt_n = 0;
    };
    std::vector<WideSub> wsubs;
    size_t wsub_next = 0;
    int4* wtasks = nullptr;
    double *wG = nullptr, *wS = nullptr, *wD = nullptr, *wlblk = nullptr;
    long long wG_rows = 0;
    // CUDA-graph replay of log-L evaluations (opts.graph)
    bool use_graph = false;
    double* theta_d = nullptr;        // {sigma2, rho, tau2} read by the kernels of a replayed evaluation
    double* theta_h = nullptr;        // pinned staging of theta_d
    cudaGraphExec_t gexec = nullptr;
    cudaStream_t gst = nullptr;       // the plan's own stream for capture / replay (the caller's stream may be the
    cudaEvent_t gev = nullptr;        // legacy default stream, which cannot be captured); ordered after the caller's
    const double* g_y = nullptr;      // key of the captured graph: y pointer and covariance family
    int g_cov = -1;
    uint64_t g_launches = 0;
    // TMA tensor maps of this context's long-lived buffers (G, prior rows per level, merge ring): handed to the GEMM
    // unit's kernels by value (build_registry)
    TmaReg treg{};
    long long *wS_off = nullptr, *wD_off = nullptr;
    int* wS_ld = nullptr;
    int wldG = 0;
    MergeRing mring{};
    // live per-kernel timing (CUDA events on the plan stream around every launch)
    bool prof = false;
    std::vector<cudaEvent_t> evpool;
    size_t ev_used = 0;
    std::vector<std::pair<int, size_t>> recs;   // (kind, index of start event; end = +1)
    double prof_ms[MRA_NKCLASS] = {0};
    uint64_t prof_cnt[MRA_NKCLASS] = {0};
};

// kernel classes of the live timing (include/mra.h MRA_NKCLASS)
enum { KIND_PRIOR = 0, KIND_BOTTOM = 1, KIND_MERGE = 2, KIND_OTHER = 3, KIND_CHAIN = 4, KIND_SIGMA = 5,
       KIND_FACTOR = 6, KIND_SOLVE = 7, KIND_SYRKMERGE = 8, KIND_COVGEN = 9 };

static cudaEvent_t take_event(mra_plan* P) {
    if (P->ev_used == P->evpool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        P->evpool.push_back(e);
    }
    return P->evpool[P->ev_used++];
}
static void prof_collect(mra_plan* P) {
    for (auto& r : P->recs) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, P->evpool[r.second], P->evpool[r.second + 1]) == cudaSuccess) {
            P->prof_ms[r.first] += ms;
            P->prof_cnt[r.first]++;
        }
    }
    P->recs.clear();
    P->ev_used = 0;
}

static long long ipow(long long b, int e) {
    long long v = 1;
    while (e-- > 0) v *= b;
    return v;
}
static long long lvl_first(int J, int m) { return (ipow(J, m - 1) - 1) / (J - 1); }
static long long q_of(int m, int rh) { return (long long)(m - 1) * rh + 1; }

#define CU(call)                                                                               \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess)                                                                 \
            return fail(e_ == cudaErrorMemoryAllocation ? MRA_E_OOM : MRA_E_CUDA,              \
                        std::string(#call) + ": " + cudaGetErrorString(e_));                   \
    } while (0)

// raw device allocation through the plan's hooks (torch's caching allocator when given)
static cudaError_t talloc(const mra_plan* p, void** ptr, size_t bytes) {
    if (bytes == 0) bytes = 8;
    if (p->ualloc) {
        *ptr = p->ualloc(bytes, p->device, (void*)p->st);
        return *ptr ? cudaSuccess : cudaErrorMemoryAllocation;
    }
    return cudaMalloc(ptr, bytes);
}
static void tfree(const mra_plan* p, void* ptr) {
    if (!ptr) return;
    if (p->ufree) p->ufree(ptr, p->device, (void*)p->st);
    else cudaFree(ptr);
}

static mra_status dalloc(mra_plan* p, void** ptr, size_t bytes, const char* what) {
    if (bytes == 0) bytes = 8;
    // slack: a bulk-copied k-row of a transposed operand is rounded up to an even number of doubles, so the copy
    // may read one double past the operand's last row (never used, but it must be mapped memory)
    bytes += 256;
    cudaError_t e = talloc(p, ptr, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        char buf[256];
        snprintf(buf, sizeof buf, "cudaMalloc(%s, %.3f GB): %s", what, bytes / 1e9, cudaGetErrorString(e));
        return fail(e == cudaErrorMemoryAllocation ? MRA_E_OOM : MRA_E_CUDA, buf);
    }
    p->allocs.push_back(*ptr);
    p->alloc_bytes.push_back(bytes);
    p->dev_bytes += bytes;
    return MRA_OK;
}

// ------------------------------------------------------------------------- plan build
static double bar_pos(double lo, double hi, int nb, int i, double off) {
    if (nb == 1) return 0.5 * (lo + hi);
    const double ext = hi - lo;
    return lo + off * ext + (double)i * (ext * (1.0 - 2.0 * off) / (double)(nb - 1));
}

// partition geometry from the data bounding box: r_hat, region counts, interior boxes (level-major,
// root = bbox with top/right pushed out 1%; J=4 quadrants / J=2 longer-axis halves,
// PAPER.md:100-103) and the knot grids
static mra_status build_geometry(mra_plan* P, double x0, double x1, double y0, double y1) {
    const int M = P->M, J = P->J;
    int nx = 1;
    while (nx * nx < P->r) nx++;
    P->nx = nx;
    P->ny = P->r / nx;
    P->rh = P->nx * P->ny;
    if (P->rh > 64) return fail(MRA_E_CONFIG, "r_hat > 64 is not supported by this build");
    P->nreg = (ipow(J, M) - 1) / (J - 1);
    P->nint = (ipow(J, M - 1) - 1) / (J - 1);
    P->nleaf = ipow(J, M - 1);
    if (!(x1 > x0) || !(y1 > y0)) return fail(MRA_E_STRUCT, "degenerate bounding box (zero extent)");
    std::vector<double> box(4 * std::max<long long>(P->nint, 1));
    if (P->nint > 0) {
        box[0] = x0; box[1] = x1 + 0.01 * (x1 - x0);
        box[2] = y0; box[3] = y1 + 0.01 * (y1 - y0);
    }
    for (int m = 1; m + 1 < M; m++) {
        const long long cnt = ipow(J, m - 1), f = lvl_first(J, m), fc = lvl_first(J, m + 1);
        for (long long t = 0; t < cnt; t++) {
            const double* b = &box[4 * (f + t)];
            const double mx = 0.5 * (b[0] + b[1]), my = 0.5 * (b[2] + b[3]);
            const bool sx = (b[1] - b[0]) >= (b[3] - b[2]);
            for (int c = 0; c < J; c++) {
                double* cb = &box[4 * (fc + t * J + c)];
                std::memcpy(cb, b, 4 * sizeof(double));
                if (J == 4) {
                    if (c & 1) cb[0] = mx; else cb[1] = mx;
                    if (c & 2) cb[2] = my; else cb[3] = my;
                } else if (sx) {
                    if (c) cb[0] = mx; else cb[1] = mx;
                } else {
                    if (c) cb[2] = my; else cb[3] = my;
                }
            }
        }
    }
    P->root[0] = x0; P->root[1] = x1 + 0.01 * (x1 - x0);
    P->root[2] = y0; P->root[3] = y1 + 0.01 * (y1 - y0);
    const int rh = P->rh;
    P->kx.assign(P->nint * rh, 0.0);
    P->ky.assign(P->nint * rh, 0.0);
    for (long long id = 0; id < P->nint; id++) {
        const double* b = &box[4 * id];
        for (int iy = 0; iy < P->ny; iy++)
            for (int ix = 0; ix < P->nx; ix++) {
                P->kx[id * rh + iy * P->nx + ix] = bar_pos(b[0], b[1], P->nx, ix, P->offset);
                P->ky[id * rh + iy * P->nx + ix] = bar_pos(b[2], b[3], P->ny, iy, P->offset);
            }
    }
    P->box = box;
    return MRA_OK;
}

// leaf statistics from the CSR offsets
static mra_status finish_leaves(mra_plan* P) {
    P->n_empty = 0;
    P->max_leaf = 0;
    for (long long t = 0; t < P->nleaf; t++) {
        const long long c = P->leaf_off[t + 1] - P->leaf_off[t];
        if (c == 0) P->n_empty++;
        P->max_leaf = std::max(P->max_leaf, c);
    }
    P->N = P->leaf_off[P->nleaf];
    if (P->N == 0) return fail(MRA_E_STRUCT, "every observation was eliminated");
    const int Jc = (P->M == 1) ? 1 : P->J;
    P->max_group = 0;
    for (long long g = 0; g < P->nleaf / Jc; g++)
        P->max_group = std::max(P->max_group, P->leaf_off[(g + 1) * Jc] - P->leaf_off[g * Jc]);
    return MRA_OK;
}

// host build (OpenMP): bounding box, leaf key by descent with the elimination test, stable counting sort
static mra_status build_host(mra_plan* P, const double* x, const double* y, uint64_t n) {
    const int M = P->M, J = P->J;
    double x0 = x[0], x1 = x[0], y0 = y[0], y1 = y[0];
    for (uint64_t i = 0; i < n; i++) {
        if (!std::isfinite(x[i]) || !std::isfinite(y[i])) return fail(MRA_E_ARG, "non-finite location");
        x0 = std::min(x0, x[i]); x1 = std::max(x1, x[i]);
        y0 = std::min(y0, y[i]); y1 = std::max(y1, y[i]);
    }
    mra_status s = build_geometry(P, x0, x1, y0, y1);
    if (s) return s;
    const int rh = P->rh;
    const std::vector<double>& box = P->box;
    // leaf key by descent; elimination test against each ancestor's bar sets
    std::vector<long long> key(n);
#pragma omp parallel for schedule(static)
    for (long long i = 0; i < (long long)n; i++) {
        const double px = x[i], py = y[i];
        long long t = 0;
        bool elim = false;
        for (int m = 1; m < M; m++) {
            const long long id = lvl_first(J, m) + t;
            const double* b = &box[4 * id];
            if (!elim) {
                bool inx = false, iny = false;
                for (int ix = 0; ix < P->nx && !inx; ix++) inx = (px == P->kx[id * rh + ix]);
                if (inx)
                    for (int iy = 0; iy < P->ny && !iny; iy++) iny = (py == P->ky[id * rh + iy * P->nx]);
                elim = inx && iny;
            }
            const double mx = 0.5 * (b[0] + b[1]), my = 0.5 * (b[2] + b[3]);
            int c;
            if (J == 4) c = (px >= mx ? 1 : 0) | (py >= my ? 2 : 0);
            else if ((b[1] - b[0]) >= (b[3] - b[2])) c = px >= mx ? 1 : 0;
            else c = py >= my ? 1 : 0;
            t = t * J + c;
        }
        key[i] = elim ? -1 : t;
    }
    // stable counting sort by leaf
    P->leaf_off.assign(P->nleaf + 1, 0);
    for (uint64_t i = 0; i < n; i++)
        if (key[i] >= 0) P->leaf_off[key[i] + 1]++;
    for (long long t = 0; t < P->nleaf; t++) P->leaf_off[t + 1] += P->leaf_off[t];
    if ((s = finish_leaves(P))) return s;
    std::vector<long long> fill(P->leaf_off.begin(), P->leaf_off.end() - 1);
    P->perm.assign(P->N, 0);
    for (uint64_t i = 0; i < n; i++)
        if (key[i] >= 0) P->perm[fill[key[i]]++] = (long long)i;
    return MRA_OK;
}

// device build (NEXT-2): upload, bounding box, leaf keys, stable radix sort by leaf, CSR offsets and
// the leaf-ordered coordinates on the GPU (mra_plan.cu). Produces the host build's plan exactly; the host
// keeps copies of leaf_off and perm (layout queries, task lists). P->pxy / P->perm_d are allocated here.
static mra_status build_device(mra_plan* P, const double* x, const double* y, uint64_t n) {
    cudaStream_t st = P->st;
    const long long nn = (long long)n;
    double *dx = nullptr, *dy = nullptr, *part = nullptr, *dbox = nullptr, *dxb = nullptr, *dyb = nullptr;
    int *bad = nullptr, *k1 = nullptr, *i1 = nullptr, *k2 = nullptr, *i2 = nullptr;
    unsigned int *cnt = nullptr, *bcnt = nullptr;
    auto release = [&]() {
        cudaStreamSynchronize(st);
        for (void* v : {(void*)dx, (void*)dy, (void*)part, (void*)dbox, (void*)dxb, (void*)dyb, (void*)bad, (void*)k1,
                        (void*)i1, (void*)k2, (void*)i2, (void*)cnt, (void*)bcnt})
            tfree(P, v);
    };
#define BD(call)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess) {                                                              \
            release();                                                                        \
            return fail(e_ == cudaErrorMemoryAllocation ? MRA_E_OOM : MRA_E_CUDA,             \
                        std::string("device plan build: " #call ": ") + cudaGetErrorString(e_)); \
        }                                                                                     \
    } while (0)
    BD(talloc(P, (void**)&dx, 8 * nn));
    BD(talloc(P, (void**)&dy, 8 * nn));
    BD(cudaMemcpyAsync(dx, x, 8 * nn, cudaMemcpyHostToDevice, st));
    BD(cudaMemcpyAsync(dy, y, 8 * nn, cudaMemcpyHostToDevice, st));
    // bounding box + finiteness
    const int nb = (int)std::min<long long>(1024, (nn + 255) / 256);
    BD(talloc(P, (void**)&part, 8 * 4 * nb));
    BD(talloc(P, (void**)&bad, 4));
    BD(cudaMemsetAsync(bad, 0, 4, st));
    BD(plan_bbox(dx, dy, nn, part, nb, bad, st));
    std::vector<double> hp(4 * nb);
    int hbad = 0;
    BD(cudaMemcpyAsync(hp.data(), part, 8 * 4 * nb, cudaMemcpyDeviceToHost, st));
    BD(cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, st));
    BD(cudaStreamSynchronize(st));
    if (hbad) { release(); return fail(MRA_E_ARG, "non-finite location"); }
    double x0 = hp[0], x1 = hp[1], y0 = hp[2], y1 = hp[3];
    for (int b = 1; b < nb; b++) {
        x0 = std::min(x0, hp[4 * b]); x1 = std::max(x1, hp[4 * b + 1]);
        y0 = std::min(y0, hp[4 * b + 2]); y1 = std::max(y1, hp[4 * b + 3]);
    }
    mra_status s = build_geometry(P, x0, x1, y0, y1);
    if (s) { release(); return s; }
    const int M = P->M, lj = P->lj;
    // boxes and knot bars on the device
    const long long ni = std::max<long long>(P->nint, 1);
    std::vector<double> hxb(ni * P->nx, 0.0), hyb(ni * P->ny, 0.0);
    for (long long id = 0; id < P->nint; id++) {
        for (int ix = 0; ix < P->nx; ix++) hxb[id * P->nx + ix] = P->kx[id * P->rh + ix];
        for (int iy = 0; iy < P->ny; iy++) hyb[id * P->ny + iy] = P->ky[id * P->rh + iy * P->nx];
    }
    BD(talloc(P, (void**)&dbox, 8 * 4 * ni));
    BD(talloc(P, (void**)&dxb, 8 * hxb.size()));
    BD(talloc(P, (void**)&dyb, 8 * hyb.size()));
    BD(cudaMemcpyAsync(dbox, P->box.data(), 8 * 4 * ni, cudaMemcpyHostToDevice, st));
    BD(cudaMemcpyAsync(dxb, hxb.data(), 8 * hxb.size(), cudaMemcpyHostToDevice, st));
    BD(cudaMemcpyAsync(dyb, hyb.data(), 8 * hyb.size(), cudaMemcpyHostToDevice, st));
    // keys (eliminated -> n_leaves), per-leaf counts
    BD(talloc(P, (void**)&k1, 4 * nn)); BD(talloc(P, (void**)&i1, 4 * nn));
    BD(talloc(P, (void**)&k2, 4 * nn)); BD(talloc(P, (void**)&i2, 4 * nn));
    BD(talloc(P, (void**)&cnt, 4 * (P->nleaf + 1)));
    BD(cudaMemsetAsync(cnt, 0, 4 * (P->nleaf + 1), st));
    PlanGeom pg{};
    pg.M = M; pg.J = P->J; pg.nx = P->nx; pg.ny = P->ny; pg.nleaf = P->nleaf;
    pg.box = dbox; pg.xbar = dxb; pg.ybar = dyb;
    BD(plan_keys(dx, dy, nn, pg, k1, i1, cnt, st));
    // stable LSD radix sort over the M base-J digits of the key (digit M-1 flags eliminated observations)
    const int nblk = plan_radix_blocks(nn), R = 1 << lj;
    BD(talloc(P, (void**)&bcnt, 4 * (size_t)R * nblk));
    std::vector<unsigned int> hb((size_t)R * nblk);
    for (int d = 0; d < M; d++) {
        BD(plan_radix_count(k1, nn, lj, d, bcnt, st));
        BD(cudaMemcpyAsync(hb.data(), bcnt, 4 * hb.size(), cudaMemcpyDeviceToHost, st));
        BD(cudaStreamSynchronize(st));
        unsigned int run = 0;   // exclusive scan, digit-major then block
        for (size_t e = 0; e < hb.size(); e++) { const unsigned int c = hb[e]; hb[e] = run; run += c; }
        BD(cudaMemcpyAsync(bcnt, hb.data(), 4 * hb.size(), cudaMemcpyHostToDevice, st));
        BD(plan_radix_scatter(k1, i1, nn, lj, d, bcnt, k2, i2, st));
        std::swap(k1, k2);
        std::swap(i1, i2);
    }
    std::vector<unsigned int> hc(P->nleaf + 1);
    BD(cudaMemcpyAsync(hc.data(), cnt, 4 * hc.size(), cudaMemcpyDeviceToHost, st));
    BD(cudaStreamSynchronize(st));
    P->leaf_off.assign(P->nleaf + 1, 0);
    for (long long t = 0; t < P->nleaf; t++) P->leaf_off[t + 1] = P->leaf_off[t] + hc[t];
    if ((s = finish_leaves(P))) { release(); return s; }
    const long long N = P->N;
    if ((s = dalloc(P, (void**)&P->pxy, 16 * N, "pxy"))) { release(); return s; }
    if ((s = dalloc(P, (void**)&P->perm_d, 8 * N, "perm"))) { release(); return s; }
    BD(plan_gather(dx, dy, i1, N, P->pxy, P->perm_d, st));
    P->perm.assign(N, 0);
    BD(cudaMemcpyAsync(P->perm.data(), P->perm_d, 8 * N, cudaMemcpyDeviceToHost, st));
    BD(cudaStreamSynchronize(st));
#undef BD
    release();
    return MRA_OK;
}

// ------------------------------------------------------------------- device sizing
static long long round_up(long long v, long long a) { return (v + a - 1) / a * a; }
static mra_status size_wide(mra_plan* P, double budget, bool explicit_budget);
static std::vector<std::pair<long long, long long>> my_runs(const mra_plan* P);

static mra_status size_device(mra_plan* P, double budget_gb, int stream_opt) {
    const int M = P->M, J = P->J, rh = P->rh;
    // prior chain rows: rh x m rh per level-m region
    auto prior_level = [&](int m) { return ipow(J, m - 1) * (long long)m * rh * rh; };
    long long tot = 0;
    for (int m = 1; m < M; m++) tot += prior_level(m);
    mra_status s;
    // workspace layout (bottom kernel; also covers merge / prior / smooth)
    const int mg = M - 1, Pg = mg * rh, ncol = Pg + 1;
    WsLayout L{};
    L.ldG = (int)round_up(ncol, 2);
    L.ldS = (int)round_up(std::max<long long>(P->max_leaf, 1), 2);
    L.ldA = (int)round_up(ncol, 2);
    // the wide path keeps G / Sigma in global per-sub-chunk buffers: its CTA slots only need A, F, L~^{-1}
    const long long mleaf = P->wide ? 1 : std::max<long long>(P->max_leaf, 1);
    const long long mgroup = P->wide ? 1 : std::max<long long>(P->max_group, 1);
    if (P->wide) L.ldS = 2;
    const long long nb = (mleaf + 63) / 64;
    long long o = 0;
    L.oG = o; o += round_up(mgroup * L.ldG, 32);
    L.oS = o; o += round_up(mleaf * (long long)L.ldS, 32);
    L.oD = o; o += nb * 4096;
    L.oA = o; o += round_up((long long)ncol * L.ldA, 32);
    L.oF = o; o += round_up((long long)ncol * rh, 32);
    L.oL = o; o += round_up((long long)rh * rh, 32);
    L.oV = o; o += round_up(mleaf, 32);
    // merge at level m <= M-2 needs qc^2 + q rh + rh^2 with qc = m rh + 1
    long long merge_need = 0;
    for (int m = 1; m + 2 <= M; m++) {
        const long long qc = (long long)m * rh + 1, q = q_of(m, rh);
        merge_need = std::max(merge_need, qc * (qc + 1) + q * rh + (long long)rh * rh + 64);
    }
    L.stride = round_up(std::max<long long>({o, merge_need, (long long)rh * rh}), 64);
    P->L = L;
    P->ws_stride = L.stride;
    size_t freeb = 0, totalb = 0;
    cudaMemGetInfo(&freeb, &totalb);
    double budget = budget_gb > 0 ? budget_gb * 1e9 : 0.85 * (double)freeb;
    budget /= std::max(1, P->n_lanes);   // every theta lane (NEXT-3) holds the same buffers
    // resident prior rows, unless they would crowd out the posterior pass (or the caller asks to
    // stream them): then only the levels above the chunk level stay resident (NEXT-4)
    P->stream = M >= 2 && (stream_opt > 0 || (stream_opt == 0 && (double)tot * 8.0 > 0.5 * budget));
    if (!P->stream) {
        long long o2 = 0;
        for (int m = 1; m < M; m++) { P->prior_base[m] = o2; o2 += prior_level(m); }
        if ((s = dalloc(P, (void**)&P->prior, sizeof(double) * tot, "prior chain rows"))) return s;
        budget -= (double)tot * 8.0;
    }
    // slots: the resident CTAs of the persistent grid, fewer if the per-slot workspace is huge
    // (wide plans: as many as the GEMM unit's prior / merge kernels keep resident; the bottom path's
    // one-CTA-per-group kernel needs far larger slots and runs on the default engine)
    long long slots = (long long)(P->wide ? std::max(resident_ctas_per_sm(), unit_ctas_per_sm())
                                          : resident_ctas_per_sm()) * P->nsm;
    const double ws_cap = std::max(0.25 * budget, (double)L.stride * 8.0);
    slots = std::min<long long>(slots, std::max<long long>(1, (long long)(ws_cap / (L.stride * 8.0))));
    P->grid = (int)slots;
    if ((s = dalloc(P, (void**)&P->ws, sizeof(double) * L.stride * slots, "workspace"))) return s;
    budget -= (double)L.stride * slots * 8.0;
    // choose chunk level c and chunk size Kc so the posterior outputs fit
    // (an explicit budget is honoured down to tiny chunks: the tests use it to force many chunks)
    const double out_budget = std::max(0.5 * budget, budget_gb > 0 ? 1e5 : 1e8);
    auto full_bytes = [&](int c) {
        double b = 0;
        for (int m = 1; m <= c && m < M; m++) b += (double)ipow(J, m - 1) * q_of(m, rh) * q_of(m, rh) * 8.0;
        return b;
    };
    auto chunk_bytes = [&](int c, long long Kc) {
        double b = 0;
        for (int m = c + 1; m < M; m++) b += (double)Kc * ipow(J, m - c) * q_of(m, rh) * q_of(m, rh) * 8.0;
        if (P->stream) {   // prior rows: levels < c for every region, levels >= c for one chunk
            for (int m = 1; m < c; m++) b += (double)prior_level(m) * 8.0;
            for (int m = c; m < M; m++) b += (double)Kc * ipow(J, m - c) * m * rh * rh * 8.0;
        }
        return b;
    };
    int c = 1;
    const int cmax = std::max(1, M - 1);
    if (P->world > 1 || P->nccl) {
        c = P->c;   // shard level fixed by the caller / auto rule
    } else {
        while (c < cmax && full_bytes(c) + chunk_bytes(c, 1) > out_budget) c++;
    }
    long long nc = ipow(J, c - 1);
    long long Kc = nc;
    while (Kc > 1 && full_bytes(c) + chunk_bytes(c, Kc) > out_budget) Kc = (Kc + 1) / 2;
    P->c = c;
    P->Kc = Kc;
    if (P->stream) {
        long long o2 = 0;
        for (int m = 1; m < M; m++) {
            P->prior_base[m] = o2;
            o2 += m < c ? prior_level(m) : Kc * ipow(J, m - c) * (long long)m * rh * rh;
        }
        if ((s = dalloc(P, (void**)&P->prior, sizeof(double) * o2, "prior chain rows (resident levels + one chunk)")))
            return s;
    }
    for (int m = 1; m <= c && m < M; m++)
        if ((s = dalloc(P, (void**)&P->out_full[m], sizeof(double) * ipow(J, m - 1) * q_of(m, rh) * q_of(m, rh),
                        "level output")))
            return s;
    for (int m = c + 1; m < M; m++)
        if ((s = dalloc(P, (void**)&P->out_chunk[m], sizeof(double) * Kc * ipow(J, m - c) * q_of(m, rh) * q_of(m, rh),
                        "chunk output")))
            return s;
    if (P->wide) return size_wide(P, budget - full_bytes(c) - chunk_bytes(c, Kc), budget_gb > 0);
    return MRA_OK;
}

// chain + Sigma as one dataflow kernel (MRA_CHSIG=1) and the lag, in leaves, of a leaf's Sigma tiles behind its
// chain tasks (MRA_CS_LAG)
static bool chsig_on() {
    static const bool on = [] { const char* e = getenv("MRA_CHSIG"); return e && atoi(e) != 0; }();
    return on;
}
static long long chsig_lag() {
    static const long long lag = [] { const char* e = getenv("MRA_CS_LAG"); return e ? std::max(1LL, atoll(e)) : 40LL; }();
    return lag;
}

// Wide path: split every posterior chunk's level-(M-1) groups into sub-chunks whose Sigma_j fit the
// budget, and precompute each sub-chunk's task lists (int4 {leaf, i, k, 0}).
static mra_status size_wide(mra_plan* P, double budget, bool explicit_budget) {
    const int M = P->M, J = P->J, rh = P->rh, mg = M - 1;
    const int Pg = mg * rh, ncol = Pg + 1, nct = (ncol + 63) / 64;
    const int qm = Pg - rh + 1, nrm = (qm + 63) / 64;   // merge tiles: q = |r| rows/cols of the merge output
    long long mt_D2 = 0;
    P->wldG = (int)round_up(ncol, 2);
    mra_status s;
    const double cap = std::max(budget * 0.8, explicit_budget ? 1e6 : 2e9);
    long long maxG = 1;
    auto leaf_n = [&](long long l) { return P->leaf_off[l + 1] - P->leaf_off[l]; };
    auto leaf_S = [&](long long l) { long long n = leaf_n(l); return n * round_up(std::max<long long>(n, 1), 2); };
    auto leaf_D = [&](long long l) { return ((leaf_n(l) + 63) / 64) * 4096LL; };
    // G = L^{-1}[V | y] through the explicit inverse X (one launch, no per-step solves) when forming X
    // (~n^3/3) costs at most about the solve itself (n^2 ncol / 2); blocked substitution otherwise
    auto xmode = [&](long long l) { return leaf_n(l) <= ncol; };
    constexpr int NBS = 8;   // super-block of the leaf Cholesky, in 64-blocks
    std::vector<int4> tasks;
    std::vector<long long> S_off(P->nleaf, 0), D_off(P->nleaf, 0);
    std::vector<int> S_ld(P->nleaf, 2);
    long long maxS = 1, maxD = 4096;
    auto runs = my_runs(P);
    for (auto& rg : runs) {
        for (long long a = rg.first; a < rg.second; a += P->Kc) {
            const long long b = std::min(rg.second, a + P->Kc);
            const long long sc = ipow(J, mg - P->c);
            const long long gA = a * sc, gB = b * sc;
            long long g = gA;
            while (g < gB) {
                mra_plan::WideSub ws;
                ws.g0 = g;
                long long sS = 0, sD = 0;
                while (g < gB) {
                    long long addS = 0, addD = 0;
                    for (int c = 0; c < J; c++) { addS += leaf_S(g * J + c); addD += leaf_D(g * J + c); }
                    const long long gRows = P->leaf_off[(g + 1) * J] - P->leaf_off[ws.g0 * J];
                    if (ws.gcount > 0 && 8.0 * (sS + addS + sD + addD + gRows * (long long)P->wldG) > cap) break;
                    for (int c = 0; c < J; c++) {
                        const long long l = g * J + c;
                        S_off[l] = sS; S_ld[l] = (int)round_up(std::max<long long>(leaf_n(l), 1), 2);
                        D_off[l] = sD;
                        sS += leaf_S(l); sD += leaf_D(l);
                    }
                    ws.gcount++;
                    g++;
                }
                maxS = std::max(maxS, sS);
                maxD = std::max(maxD, sD);
                maxG = std::max(maxG, P->leaf_off[(ws.g0 + ws.gcount) * J] - P->leaf_off[ws.g0 * J]);
                // task lists
                int Tmax = 0;
                ws.chain_off = (long long)tasks.size();
                for (long long l = ws.g0 * J; l < (ws.g0 + ws.gcount) * J; l++) {
                    const int T = (int)((leaf_n(l) + 63) / 64);
                    Tmax = std::max(Tmax, T);
                    for (int i = 0; i < T; i++) tasks.push_back(make_int4((int)l, i, 0, 0));
                }
                ws.chain_n = (long long)tasks.size() - ws.chain_off;
                ws.sigma_off = (long long)tasks.size();
                for (long long l = ws.g0 * J; l < (ws.g0 + ws.gcount) * J; l++) {
                    const int T = (int)((leaf_n(l) + 63) / 64);
                    for (int i = 0; i < T; i++)
                        for (int k = 0; k <= i; k++) tasks.push_back(make_int4((int)l, i, k, 0));
                }
                ws.sigma_n = (long long)tasks.size() - ws.sigma_off;
                // the same chain and Sigma tasks as one dataflow (k_wide_chsig): leaf l's Sigma tiles follow the
                // chain tasks of leaf l + lag (type in .w)
                if (chsig_on()) {
                    const long long L0 = ws.g0 * J, L1 = (ws.g0 + ws.gcount) * J, lag = chsig_lag();
                    auto push_sig = [&](long long l) {
                        const int T = (int)((leaf_n(l) + 63) / 64);
                        for (int i = 0; i < T; i++)
                            for (int k = 0; k <= i; k++) tasks.push_back(make_int4((int)l, i, k, 1));
                    };
                    ws.cs_off = (long long)tasks.size();
                    for (long long l = L0; l < L1; l++) {
                        const int T = (int)((leaf_n(l) + 63) / 64);
                        for (int i = 0; i < T; i++) tasks.push_back(make_int4((int)l, i, 0, 0));
                        if (l - lag >= L0) push_sig(l - lag);
                    }
                    for (long long l = std::max(L0, L1 - lag); l < L1; l++) push_sig(l);
                    ws.cs_n = (long long)tasks.size() - ws.cs_off;
                }
                // super-blocked Cholesky of the leaves' Sigma_j (blocks of 64, super-blocks of NBS blocks):
                // left-looking inside a super-block, one right-looking trailing update after it, so the
                // late steps of large leaves (C4: up to 139 blocks) keep every CTA busy with K = 64 NBS
                for (int st = 0; st < Tmax; st++) {
                    const int kb0 = st / NBS * NBS;
                    ws.upd_off.push_back((long long)tasks.size());
                    if (st > kb0)
                        for (long long l = ws.g0 * J; l < (ws.g0 + ws.gcount) * J; l++) {
                            const int T = (int)((leaf_n(l) + 63) / 64);
                            for (int i = st; i < T; i++) tasks.push_back(make_int4((int)l, i, st, 0));
                        }
                    ws.upd_n.push_back((long long)tasks.size() - ws.upd_off.back());
                    ws.diag_off.push_back((long long)tasks.size());
                    for (long long l = ws.g0 * J; l < (ws.g0 + ws.gcount) * J; l++)
                        if ((leaf_n(l) + 63) / 64 > st) tasks.push_back(make_int4((int)l, 0, 0, 0));
                    ws.diag_n.push_back((long long)tasks.size() - ws.diag_off.back());
                    // after the diagonal of step st: panel tasks L_is (i > st) and the tasks of row block
                    // st of X = L^{-1} (X_{st,k}, k < st)
                    ws.pf_off.push_back((long long)tasks.size());
                    for (long long l = ws.g0 * J; l < (ws.g0 + ws.gcount) * J; l++) {
                        const int T = (int)((leaf_n(l) + 63) / 64);
                        if (T <= st) continue;
                        for (int i = st + 1; i < T; i++) tasks.push_back(make_int4((int)l, i, 0, 0));
                        if (xmode(l))
                            for (int k = 0; k < st; k++) tasks.push_back(make_int4((int)l, k, 2, 0));
                        else
                            for (int c2 = 0; c2 < nct; c2++) tasks.push_back(make_int4((int)l, c2, 1, 0));
                    }
                    ws.pf_n.push_back((long long)tasks.size() - ws.pf_off.back());
                    ws.tr_off.push_back((long long)tasks.size());
                    if (st == kb0 + NBS - 1)
                        for (long long l = ws.g0 * J; l < (ws.g0 + ws.gcount) * J; l++) {
                            const int T = (int)((leaf_n(l) + 63) / 64);
                            for (int i = st + 1; i < T; i++) {
                                for (int j = st + 1; j <= i; j++) tasks.push_back(make_int4((int)l, i, j, 0));
                                if (!xmode(l))
                                    for (int c2 = 0; c2 < nct; c2++) tasks.push_back(make_int4((int)l, i, c2, 1));
                            }
                        }
                    ws.tr_n.push_back((long long)tasks.size() - ws.tr_off.back());
                }
                // G = X [V | y], one task per (leaf, column tile) after the factorization
                ws.trsm_off = (long long)tasks.size();
                // a lone y column (ncol = 64 k + 1) is one row-parallel GEMV task per leaf (type 2)
                const bool ycol = (ncol % 64) == 1;
                for (long long l = ws.g0 * J; l < (ws.g0 + ws.gcount) * J; l++)
                    if (leaf_n(l) > 0 && xmode(l)) {
                        for (int c2 = 0; c2 < (ycol ? nct - 1 : nct); c2++) tasks.push_back(make_int4((int)l, c2, 1, 0));
                        if (ycol) tasks.push_back(make_int4((int)l, 0, 2, 0));
                    }
                ws.trsm_n = (long long)tasks.size() - ws.trsm_off;
                // merge tile dataflow: step s holds T00 of group s, the F tasks of group s - D1 and the
                // O tasks of group s - D2; D1 covers ~1.2 ms of steps at the estimated step
                // time, D2 = D1 + 96 (measured on C3 / C4 / C2 with MRA_MT_D1US / MRA_MT_D2ADD: the merge tile
                // kernel takes 710 / 25.4 / 13.8 ms at 150 us + 12, 668 / 11.6 / 12.3 ms at 1.2 ms + 96, flat
                // beyond; with 4 CTAs per SM a consumer claimed too soon stalls its whole CTA)
                {
                    const long long gc = ws.gcount;
                    const double kavg = (double)(P->leaf_off[(ws.g0 + gc) * J] - P->leaf_off[ws.g0 * J]) / gc;
                    const double step_us = (1.0 + nrm + nrm * (nrm + 1) / 2.0) * std::max(kavg, 64.0) * 0.066 /
                                           std::max(1, wide_mtile_resident());
                    static const double D1_US = [] { const char* e = getenv("MRA_MT_D1US"); return e ? atof(e) : 1200.0; }();
                    static const long long D2_ADD = [] { const char* e = getenv("MRA_MT_D2ADD"); return e ? atoll(e) : 96LL; }();
                    const long long D1 = std::min<long long>(512, std::max<long long>(2, (long long)std::ceil(D1_US / step_us)));
                    const long long D2 = D1 + D2_ADD;   // an O task waits for all F of its group before its GEMM
                    mt_D2 = std::max(mt_D2, D2);
                    // a lone y row (q = 64 k + 1) is formed by one GEMV task per group (type 3), not by
                    // 1-row tiles (which cost nearly a full tile each)
                    const bool ysep = (qm % 64 == 1) && qm > 1;
                    const int nrF = ysep ? nrm - 1 : nrm;
                    ws.mt_off = (long long)tasks.size();
                    for (long long st = 0; st < gc + D2; st++) {
                        if (st < gc) tasks.push_back(make_int4((int)st, 0, 0, 0));
                        const long long gf = st - D1;
                        if (gf >= 0 && gf < gc)
                            for (int a = 0; a < nrF; a++) tasks.push_back(make_int4((int)gf, 1, a, 0));
                        const long long go = st - D2;
                        if (go >= 0 && go < gc) {
                            for (int a = 0; a < nrF; a++)
                                for (int b = 0; b <= a; b++) tasks.push_back(make_int4((int)go, 2, a, b));
                            // after the group's O tiles, which have just brought its G panels into L2
                            if (ysep) tasks.push_back(make_int4((int)go, 3, 0, 0));
                        }
                    }
                    ws.mt_n = (long long)tasks.size() - ws.mt_off;
                }
                P->wsubs.push_back(std::move(ws));
            }
        }
    }
    if ((s = dalloc(P, (void**)&P->wG, 8 * maxG * P->wldG, "wide G"))) return s;
    P->wG_rows = maxG;
    if ((s = dalloc(P, (void**)&P->wS, 8 * maxS, "wide Sigma"))) return s;
    if ((s = dalloc(P, (void**)&P->wD, 8 * maxD, "wide Dinv"))) return s;
    if ((s = dalloc(P, (void**)&P->wlblk, 8 * (maxD / 4096 + 1), "wide logdets"))) return s;
    if ((s = dalloc(P, (void**)&P->wS_off, 8 * P->nleaf, "wide S_off"))) return s;
    if ((s = dalloc(P, (void**)&P->wD_off, 8 * P->nleaf, "wide D_off"))) return s;
    if ((s = dalloc(P, (void**)&P->wS_ld, 4 * P->nleaf, "wide S_ld"))) return s;
    if ((s = dalloc(P, (void**)&P->wtasks, sizeof(int4) * std::max<size_t>(1, tasks.size()), "wide tasks"))) return s;
    // small-slot ring + counters of the merge tile dataflow
    {
        long long maxgc = 1;
        for (auto& w : P->wsubs) maxgc = std::max(maxgc, w.gcount);
        long long ns = std::min<long long>(maxgc, mt_D2 + 8);
        P->mring.ns = (int)ns;
        P->mring.maxg = maxgc;
        P->mring.stride = round_up(4096 + (long long)rh * rh + 2LL * qm * rh, 32);   // A_oo | Li | F | -F
        if ((s = dalloc(P, (void**)&P->mring.slot, 8 * P->mring.stride * ns, "merge slots"))) return s;
        if ((s = dalloc(P, (void**)&P->mring.flags, 4 * (3 + J) * maxgc, "merge flags"))) return s;
        P->mring.chol_done = P->mring.flags;
        P->mring.f_done = P->mring.flags + maxgc;
        P->mring.o_done = P->mring.flags + 2 * maxgc;
        if ((s = dalloc(P, (void**)&P->mring.slot_done, 8 * ns, "merge slot_done"))) return s;
    }
    CU(cudaMemcpy(P->wS_off, S_off.data(), 8 * P->nleaf, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(P->wD_off, D_off.data(), 8 * P->nleaf, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(P->wS_ld, S_ld.data(), 4 * P->nleaf, cudaMemcpyHostToDevice));
    if (!tasks.empty()) CU(cudaMemcpy(P->wtasks, tasks.data(), sizeof(int4) * tasks.size(), cudaMemcpyHostToDevice));
    return MRA_OK;
}

// --------------------------------------------------------------------- C ABI entry
extern "C" const char* mra_last_error(void) { return g_err.c_str(); }

// the context's TMA registry: G (leaf rows, row-major and transposed views), the prior chain rows of every level
// (both views), the merge ring (row-major, when its slots are laid out in whole rows of r_hat). MRA_NO_TMA=1
// leaves it empty (every GEMM then stages by cp.async / bulk copies).
static void build_registry(mra_plan* P) {
    P->treg = TmaReg{};
    if (getenv("MRA_NO_TMA")) return;
    const int rh = P->rh, M = P->M, J = P->J;
    if (P->wG && P->wG_rows > 0) {
        tma_register(P->treg, 0, P->wG, P->wldG, P->wG_rows);
        tma_register(P->treg, 1, P->wG, P->wldG, P->wG_rows);
    }
    if (P->prior)
        for (int m = 1; m < M; m++) {
            long long regions = ipow(J, m - 1);
            if (P->stream && m >= P->c) regions = P->Kc * ipow(J, m - P->c);
            const long long ld = (long long)m * rh, rows = regions * rh;
            tma_register(P->treg, 0, P->prior + P->prior_base[m], ld, rows);
            tma_register(P->treg, 1, P->prior + P->prior_base[m], ld, rows);
        }
    if (P->mring.slot && P->mring.stride % rh == 0 && 4096 % rh == 0)
        tma_register(P->treg, 0, P->mring.slot, rh, P->mring.stride * P->mring.ns / rh);
}

// an evaluation context for theta-batched sweeps: a copy of the plan's host metadata that shares its
// read-only device data (observations, knots, CSR, task lists) and owns the buffers an evaluation
// writes (sorted y, prior rows, per-region terms, merge outputs, workspaces, counters, wide buffers)
static mra_status make_lane(mra_plan* P, mra_plan** out) {
    mra_plan* Q = new mra_plan(*P);
    Q->allocs.clear();
    Q->alloc_bytes.clear();
    Q->dev_bytes = 0;
    Q->evpool.clear();
    Q->ev_used = 0;
    Q->recs.clear();
    Q->lanes.clear();
    Q->is_lane = true;
    Q->lane_ev = nullptr;
    Q->cst = nullptr;
    Q->cev = nullptr;
    Q->host_y_pending = nullptr;
    Q->post = Q->muhat = Q->mu_d = Q->smooth_d = Q->ws_smooth = Q->ws_pred = nullptr;
    Q->use_graph = false;
    Q->gexec = nullptr;
    Q->gst = nullptr;
    Q->gev = nullptr;
    Q->theta_h = nullptr;
    Q->theta_d = nullptr;
    Q->post_valid = false;
    Q->st = nullptr;
    *out = nullptr;
    if (cudaStreamCreateWithFlags(&Q->st, cudaStreamNonBlocking) != cudaSuccess) {
        delete Q;
        return fail(MRA_E_CUDA, "theta lane: cudaStreamCreate failed");
    }
    auto bytes_of = [&](const void* ptr) -> size_t {
        for (size_t i = 0; i < P->allocs.size(); i++)
            if (P->allocs[i] == ptr) return P->alloc_bytes[i];
        return 0;
    };
    mra_status s = MRA_OK;
    auto dup = [&](auto*& f, const char* what) {
        if (s || !f) return;
        const size_t b = bytes_of(f);
        if (!b) { s = fail(MRA_E_CUDA, std::string("theta lane: unknown buffer ") + what); return; }
        void* p = nullptr;
        s = dalloc(Q, &p, b, what);
        f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(p);
    };
    dup(Q->zs, "lane zs");
    dup(Q->prior, "lane prior");
    dup(Q->dreg, "lane dreg");
    dup(Q->ureg, "lane ureg");
    dup(Q->loglik_d, "lane loglik");
    dup(Q->err, "lane err");
    dup(Q->counters, "lane counters");
    dup(Q->ws, "lane workspace");
    for (int m = 0; m <= MAXM; m++) {
        dup(Q->out_full[m], "lane level output");
        dup(Q->out_chunk[m], "lane chunk output");
    }
    dup(Q->wG, "lane wide G");
    dup(Q->wS, "lane wide Sigma");
    dup(Q->wD, "lane wide Dinv");
    dup(Q->wlblk, "lane wide logdets");
    dup(Q->mring.slot, "lane merge slots");
    dup(Q->mring.flags, "lane merge flags");
    dup(Q->mring.slot_done, "lane merge slot_done");
    if (Q->mring.flags) {
        Q->mring.chol_done = Q->mring.flags;
        Q->mring.f_done = Q->mring.flags + Q->mring.maxg;
        Q->mring.o_done = Q->mring.flags + 2 * Q->mring.maxg;
    }
    if (s) {
        mra_plan_destroy(Q);
        return s;
    }
    build_registry(Q);   // the lane's own buffers
    *out = Q;
    return MRA_OK;
}

extern "C" mra_status mra_plan_create(const double* x, const double* y, uint64_t n, int M, int J, int r,
                                      const mra_opts* opts, mra_plan** out) {
    return guarded([&]() -> mra_status {
        g_err.clear();
        if (!out) return fail(MRA_E_ARG, "out is NULL");
        *out = nullptr;
        if (!x || !y || n == 0) return fail(MRA_E_ARG, "x/y NULL or n == 0");
        if (M < 1 || M > MAXM - 1) return fail(MRA_E_CONFIG, "M out of range [1, 23]");
        if (J != 2 && J != 4) return fail(MRA_E_CONFIG, "J must be 2 or 4 (PAPER.md:100)");
        if (r < 1) return fail(MRA_E_CONFIG, "r must be >= 1");
        // the task lists index leaves with 32-bit fields and the host keeps O(regions) metadata: bound the tree
        if (ipow(J, M - 1) > (1LL << 30)) return fail(MRA_E_CONFIG, "tree too large: J^(M-1) leaves must be <= 2^30");
        mra_opts o{};
        if (opts) o = *opts;
        if ((o.dalloc == nullptr) != (o.dfree == nullptr)) return fail(MRA_E_ARG, "dalloc and dfree must be given together");
        mra_plan* P = new mra_plan();
        P->ualloc = o.dalloc;
        P->ufree = o.dfree;
        P->M = M; P->J = J; P->lj = (J == 4) ? 2 : 1; P->r = r;
        P->offset = o.offset > 0 ? o.offset : std::exp(1.0) / 100.0;
        if (!(P->offset > 0 && P->offset < 0.5)) { delete P; return fail(MRA_E_ARG, "offset must be in (0, 0.5)"); }
        P->xs = o.xscale > 0 ? o.xscale : 1.0;
        P->ys = o.yscale > 0 ? o.yscale : 1.0;
        P->n_in = n;
        P->rank = o.world > 1 ? o.rank : 0;
        P->world = o.world > 1 ? o.world : 1;
        P->nccl = o.nccl_id != nullptr;
        if (P->nccl && o.device == -2) { delete P; return fail(MRA_E_ARG, "a host-only plan has no communicator"); }
        if (o.world > 1 && (o.rank < 0 || o.rank >= o.world)) { delete P; return fail(MRA_E_ARG, "rank out of [0, world)"); }
        // S0 on the device (NEXT-2) unless this is a host-only plan, the caller asks for the host build,
        // or the keys / indices would not fit the device build's 32-bit fields
        const bool dev_build = o.device != -2 && !o.host_plan && n < (1ULL << 31) &&
                               ipow(J, M - 1) < (1LL << 30);
        mra_status s = MRA_OK;
        if (dev_build) {
            int dev = o.device;
            if (dev < 0 && cudaGetDevice(&dev) != cudaSuccess) { delete P; return fail(MRA_E_CUDA, "no CUDA device"); }
            if (cudaSetDevice(dev) != cudaSuccess) { delete P; return fail(MRA_E_CUDA, "cudaSetDevice failed (no GPU?)"); }
            P->device = dev;
            P->st = (cudaStream_t)o.stream;
            s = build_device(P, x, y, n);
            if (s) { mra_plan_destroy(P); return s; }
        } else {
            s = build_host(P, x, y, n);
            if (s) { delete P; return s; }
        }
        // the grid-wide task path is at least as fast as one-CTA-per-group on every configuration measured
        // (C0 4.3x, C1 1.2x, C2/C3 ~1.02x, C4 > 100x: DESIGN.md §5), so it is the default for M >= 2
        P->wide = M >= 2 && o.wide >= 0;
        // sharding: shard level = first level with >= 8*world regions (or the caller's choice); an in-library
        // communicator runs the sharded schedule at any world size (world 1: the path on one rank)
        if (P->world > 1 || P->nccl) {
            int sl = o.shard_level;
            if (sl <= 0) { sl = 1; while (sl < M - 1 && ipow(J, sl - 1) < 8LL * P->world) sl++; }
            if (sl >= M) sl = M - 1;
            if (sl < 1) { delete P; return fail(MRA_E_CONFIG, "tree too shallow to shard (need M >= 2)"); }
            P->c = sl;
            // LPT over the per-shard leaf work (sum n_j^3 + n_j^2 ((M-1) r_hat))
            const long long ns = ipow(J, sl - 1), per = ipow(J, M - sl);
            std::vector<std::pair<double, long long>> cost(ns);
            for (long long s2 = 0; s2 < ns; s2++) {
                double cst = 0;
                for (long long l = s2 * per; l < (s2 + 1) * per; l++) {
                    const double nj = (double)(P->leaf_off[l + 1] - P->leaf_off[l]);
                    cst += nj * nj * nj / 3.0 + nj * nj * (M - 1) * P->rh * 2.0 + nj * std::pow((M - 1) * P->rh, 2);
                }
                cost[s2] = {cst + 1.0, s2};
            }
            std::vector<double> in_order(ns);
            for (auto& cs : cost) in_order[cs.second] = cs.first;
            std::sort(cost.begin(), cost.end(), [](auto& a, auto& b) { return a.first > b.first || (a.first == b.first && a.second < b.second); });
            std::vector<double> load(P->world, 0.0);
            std::vector<int> lpt_owner(ns, 0);
            for (auto& cs : cost) {
                int best = 0;
                for (int w = 1; w < P->world; w++) if (load[w] < load[best]) best = w;
                load[best] += cs.first;
                lpt_owner[cs.second] = best;
            }
            const double lpt_max = *std::max_element(load.begin(), load.end());
            // contiguous alternative: the smallest-max-load split of the shards, in order, into `world` runs
            // (bisection on the capacity, greedy fill). Taken when within 3 % of LPT's max load: a rank's
            // subtrees then form ONE run -- one chunk sequence of launches instead of one per scattered subtree
            // (projected C3 at 8 GPUs: LPT's scattered runs cost the per-rank pass 16 % over an even share)
            auto split = [&](double cap, std::vector<long long>& starts) {
                starts.assign(1, 0);
                double acc = 0;
                for (long long s2 = 0; s2 < ns; s2++) {
                    if (in_order[s2] > cap) return false;
                    if (acc + in_order[s2] > cap) { starts.push_back(s2); acc = 0; }
                    acc += in_order[s2];
                }
                return (long long)starts.size() <= P->world;
            };
            double lo = *std::max_element(in_order.begin(), in_order.end()), hi = 0;
            for (double v : in_order) hi += v;
            std::vector<long long> starts;
            for (int it = 0; it < 64; it++) {
                const double mid = 0.5 * (lo + hi);
                if (split(mid, starts)) hi = mid; else lo = mid;
            }
            split(hi, starts);
            static const bool force_lpt = getenv("MRA_SHARD_LPT") != nullptr;
            const bool contiguous = !force_lpt && (long long)starts.size() == P->world && hi <= 1.03 * lpt_max;
            for (long long s2 = 0; s2 < ns; s2++) {
                int owner = lpt_owner[s2];
                if (contiguous) owner = (int)(std::upper_bound(starts.begin(), starts.end(), s2) - starts.begin()) - 1;
                if (owner == P->rank) P->my_c.push_back(s2);
            }
        }
        if (o.device == -2) {   // host-only plan: structure only (PAPER.md:228 build_structure_only)
            P->device = -2;
            *out = P;
            return MRA_OK;
        }
    
        int dev = o.device;
        if (dev < 0) {
            if (cudaGetDevice(&dev) != cudaSuccess) { delete P; return fail(MRA_E_CUDA, "no CUDA device"); }
        }
        P->device = dev;
        if (cudaSetDevice(dev) != cudaSuccess) { delete P; return fail(MRA_E_CUDA, "cudaSetDevice failed (no GPU?)"); }
        cudaDeviceGetAttribute(&P->nsm, cudaDevAttrMultiProcessorCount, dev);
        P->st = (cudaStream_t)o.stream;
        mra_status st;
    #define TRY(x) do { if ((st = (x))) { mra_plan_destroy(P); return st; } } while (0)
        const long long N = P->N;
        if (!dev_build) {
            TRY(dalloc(P, (void**)&P->pxy, 16 * N, "pxy"));
            TRY(dalloc(P, (void**)&P->perm_d, 8 * N, "perm"));
        }
        TRY(dalloc(P, (void**)&P->zs, 8 * N, "zs"));
        TRY(dalloc(P, (void**)&P->zin, 8 * (long long)n, "zin"));
        TRY(dalloc(P, (void**)&P->leaf_off_d, 8 * (P->nleaf + 1), "leaf_off"));
        TRY(dalloc(P, (void**)&P->kxy_d, 16 * std::max<long long>(1, P->nint * P->rh), "kxy"));
        TRY(dalloc(P, (void**)&P->dreg, 8 * P->nreg, "dreg"));
        TRY(dalloc(P, (void**)&P->ureg, 8 * P->nreg, "ureg"));
        TRY(dalloc(P, (void**)&P->loglik_d, 8, "loglik"));
        TRY(dalloc(P, (void**)&P->err, 16, "err"));
        P->n_counters = 1 << 16;
        TRY(dalloc(P, (void**)&P->counters, 8 * (size_t)P->n_counters, "counters"));
        {
            std::vector<double> kxy(2 * std::max<long long>(1, P->nint * P->rh));
            for (long long i = 0; i < P->nint * P->rh; i++) { kxy[2 * i] = P->kx[i]; kxy[2 * i + 1] = P->ky[i]; }
            auto cp = [&](void* d, const void* h, size_t b) -> mra_status {
                cudaError_t e = cudaMemcpy(d, h, b, cudaMemcpyHostToDevice);
                if (e != cudaSuccess) return fail(MRA_E_CUDA, std::string("upload: ") + cudaGetErrorString(e));
                return MRA_OK;
            };
            if (!dev_build) {
                std::vector<double> sxy(2 * N);
                for (long long i = 0; i < N; i++) { sxy[2 * i] = x[P->perm[i]]; sxy[2 * i + 1] = y[P->perm[i]]; }
                TRY(cp(P->pxy, sxy.data(), 16 * N));
                TRY(cp(P->perm_d, P->perm.data(), 8 * N));
            }
            TRY(cp(P->leaf_off_d, P->leaf_off.data(), 8 * (P->nleaf + 1)));
            if (P->nint) TRY(cp(P->kxy_d, kxy.data(), 16 * P->nint * P->rh));
        }
        // the copy stream / event of the host-y entry points (created here, not inside the first timed call)
        if (cudaStreamCreateWithFlags(&P->cst, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&P->cev, cudaEventDisableTiming) != cudaSuccess) {
            mra_plan_destroy(P);
            return fail(MRA_E_CUDA, "copy stream / event creation failed");
        }
        P->n_lanes = std::max(1, std::min(o.theta_lanes, 16));
        if (P->world > 1 || P->nccl) P->n_lanes = 1;
        TRY(size_device(P, o.mem_budget_gb, o.stream_prior));
    init_kernel_attrs();   // smem attributes / occupancy now: nothing of the kind may run inside a graph capture
    if (o.graph) {
        P->use_graph = true;
        TRY(dalloc(P, (void**)&P->theta_d, 8 * 4, "theta"));
        if (cudaMallocHost((void**)&P->theta_h, 32) != cudaSuccess ||
            cudaStreamCreateWithFlags(&P->gst, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&P->gev, cudaEventDisableTiming) != cudaSuccess) {
            mra_plan_destroy(P);
            return fail(MRA_E_CUDA, "graph staging (pinned theta, stream, event)");
        }
    }
    build_registry(P);
        if (P->nccl) {
            const NcclApi* nc = nccl_api();
            if (!nc) {
                mra_plan_destroy(P);
                return fail(MRA_E_NCCL, "opts.nccl_id given but no NCCL library could be loaded (libnccl.so.2 / $MRA_NCCL_LIB)");
            }
            ncclUniqueId id;
            std::memcpy(&id, o.nccl_id, sizeof id);
            const ncclResult_t r0 = nc->commInitRank(&P->comm, P->world, id, P->rank);
            if (r0 != ncclSuccess) {
                P->comm = nullptr;
                mra_plan_destroy(P);
                return fail(MRA_E_NCCL, std::string("ncclCommInitRank: ") + nc->errStr(r0));
            }
            TRY(dalloc(P, (void**)&P->xbuf, 8 * mra_shard_size(P), "exchange buffer"));
            TRY(dalloc(P, (void**)&P->bcast, 8 * 4, "broadcast scalars"));
        }
        for (int k = 1; k < P->n_lanes; k++) {
            mra_plan* Q = nullptr;
            TRY(make_lane(P, &Q));
            P->lanes.push_back(Q);
        }
    #undef TRY
        *out = P;
        return MRA_OK;
    });
}

extern "C" void mra_plan_destroy(mra_plan* P) {
    if (!P) return;
    for (mra_plan* Q : P->lanes) mra_plan_destroy(Q);
    P->lanes.clear();
    if (P->device >= 0 && cudaSetDevice(P->device) == cudaSuccess) {
        cudaDeviceSynchronize();
        if (P->is_lane && P->st) cudaStreamDestroy(P->st);
        if (P->gexec) cudaGraphExecDestroy(P->gexec);
        if (P->gev) cudaEventDestroy(P->gev);
        if (P->gst) cudaStreamDestroy(P->gst);
        if (P->theta_h && !P->is_lane) cudaFreeHost(P->theta_h);
        if (P->lane_ev) cudaEventDestroy(P->lane_ev);
        for (cudaEvent_t e : P->evpool) cudaEventDestroy(e);
        if (P->cev) cudaEventDestroy(P->cev);
        if (P->cst) cudaStreamDestroy(P->cst);
        for (void* a : P->allocs) tfree(P, a);
        if (P->comm && !P->is_lane) {
            if (const NcclApi* nc = nccl_api()) nc->commDestroy(P->comm);
        }
    }
    delete P;
}

extern "C" mra_status mra_plan_info(const mra_plan* P, uint64_t* n_retained, int* r_hat, uint64_t* n_regions,
                                    uint64_t* n_leaves, uint64_t* n_empty, uint64_t* max_leaf) {
    return guarded([&]() -> mra_status {
        if (!P) return fail(MRA_E_ARG, "plan is NULL");
        if (n_retained) *n_retained = (uint64_t)P->N;
        if (r_hat) *r_hat = P->rh;
        if (n_regions) *n_regions = (uint64_t)P->nreg;
        if (n_leaves) *n_leaves = (uint64_t)P->nleaf;
        if (n_empty) *n_empty = (uint64_t)P->n_empty;
        if (max_leaf) *max_leaf = (uint64_t)P->max_leaf;
        return MRA_OK;
    });
}

extern "C" mra_status mra_plan_layout(const mra_plan* P, int64_t* perm, int64_t* leaf_off, double* kx, double* ky) {
    return guarded([&]() -> mra_status {
        if (!P) return fail(MRA_E_ARG, "plan is NULL");
        if (perm) std::memcpy(perm, P->perm.data(), 8 * P->N);
        if (leaf_off) std::memcpy(leaf_off, P->leaf_off.data(), 8 * (P->nleaf + 1));
        if (kx && P->nint) std::memcpy(kx, P->kx.data(), 8 * P->nint * P->rh);
        if (ky && P->nint) std::memcpy(ky, P->ky.data(), 8 * P->nint * P->rh);
        return MRA_OK;
    });
}

extern "C" uint64_t mra_last_launches(const mra_plan* P) { return P ? P->launches : 0; }

extern "C" mra_status mra_profile(mra_plan* P, int enable) {
    return guarded([&]() -> mra_status {
        if (!P) return fail(MRA_E_ARG, "plan is NULL");
        for (mra_plan* Q : P->lanes) mra_profile(Q, enable);
        P->prof = enable != 0;
        P->recs.clear();
        P->ev_used = 0;
        for (int k = 0; k < MRA_NKCLASS; k++) { P->prof_ms[k] = 0; P->prof_cnt[k] = 0; }
        return MRA_OK;
    });
}

extern "C" mra_status mra_kernel_times(const mra_plan* P, double* ms, uint64_t* launches) {
    return guarded([&]() -> mra_status {
        if (!P) return fail(MRA_E_ARG, "plan is NULL");
        for (int k = 0; k < MRA_NKCLASS; k++) {   // summed over the theta lanes
            double t = P->prof_ms[k];
            uint64_t c = P->prof_cnt[k];
            for (const mra_plan* Q : P->lanes) { t += Q->prof_ms[k]; c += Q->prof_cnt[k]; }
            if (ms) ms[k] = t;
            if (launches) launches[k] = c;
        }
        return MRA_OK;
    });
}

// diagnostics of -DMRA_PHASE_TIMING builds (zeros otherwise): CTA-cycles per bottom-kernel phase
extern "C" void mra_debug_phase_cycles(uint64_t* out32, int reset) {
    unsigned long long v[32], w[32];
    phase_cycles(v, reset != 0);
    phase_cycles_unit(w, reset != 0);   // the GEMM unit's kernels count into their own copy
    for (int i = 0; i < 32; i++) out32[i] = v[i] + w[i];
}

extern "C" mra_status mra_plan_memory(const mra_plan* P, int* streams_prior, int* chunk_level,
                                      uint64_t* chunk_regions, uint64_t* device_bytes) {
    return guarded([&]() -> mra_status {
        if (!P) return fail(MRA_E_ARG, "plan is NULL");
        if (streams_prior) *streams_prior = P->stream ? 1 : 0;
        if (chunk_level) *chunk_level = P->c;
        if (chunk_regions) *chunk_regions = (uint64_t)P->Kc;
        if (device_bytes) {
            uint64_t b = P->dev_bytes;
            for (const mra_plan* Q : P->lanes) b += Q->dev_bytes;   // theta lanes (NEXT-3)
            *device_bytes = b;
        }
        return MRA_OK;
    });
}

extern "C" mra_status mra_plan_shards(const mra_plan* P, int* shard_level, int64_t* own, uint64_t* n_own) {
    return guarded([&]() -> mra_status {
        if (!P) return fail(MRA_E_ARG, "plan is NULL");
        if (shard_level) *shard_level = (P->world > 1 || P->nccl) ? P->c : 0;
        if (n_own) *n_own = (uint64_t)P->my_c.size();
        if (own) for (size_t i = 0; i < P->my_c.size(); i++) own[i] = P->my_c[i];
        return MRA_OK;
    });
}

// ------------------------------------------------------------------------ evaluation
static TreeParams tree_params(mra_plan* P, const mra_theta* th) {
    TreeParams tp{};
    tp.M = P->M; tp.J = P->J; tp.lj = P->lj; tp.rh = P->rh;
    tp.cp.kind = th->cov; tp.cp.s2 = th->sigma2; tp.cp.rho = th->rho; tp.cp.xs = P->xs; tp.cp.ys = P->ys;
    tp.tau2 = th->tau2;
    tp.pxy = P->pxy; tp.zs = P->zs; tp.leaf_off = P->leaf_off_d;
    tp.kxy = P->kxy_d; tp.prior = P->prior;
    for (int m = 0; m <= MAXM; m++) { tp.prior_base[m] = P->prior_base[m]; tp.post_base[m] = P->post_base[m]; }
    tp.dreg = P->dreg; tp.ureg = P->ureg; tp.err = P->err; tp.post = nullptr;
    tp.theta_dev = nullptr;
    return tp;
}

static mra_status check_theta(const mra_theta* th) {
    if (!th) return fail(MRA_E_ARG, "theta is NULL");
    if (th->cov != MRA_COV_EXP && th->cov != MRA_COV_MATERN32) return fail(MRA_E_ARG, "unknown covariance kind");
    if (!(th->sigma2 > 0) || !(th->rho > 0) || !(th->tau2 > 0) || !std::isfinite(th->sigma2) ||
        !std::isfinite(th->rho) || !std::isfinite(th->tau2))
        return fail(MRA_E_ARG, "theta must be finite and > 0");
    return MRA_OK;
}

#define LCHK_K(kind, expr)                                                                   \
    do {                                                                                     \
        size_t ev0_ = 0;                                                                     \
        const unsigned long long k0_ = g_kernel_launches;                                    \
        if (P->prof) {                                                                       \
            ev0_ = P->ev_used;                                                               \
            cudaEventRecord(take_event(P), P->st);                                           \
        }                                                                                    \
        cudaError_t e_ = (expr);                                                             \
        if (P->prof) {                                                                       \
            cudaEventRecord(take_event(P), P->st);                                           \
            P->recs.push_back({(kind), ev0_});                                               \
        }                                                                                    \
        P->launches += g_kernel_launches - k0_;   /* kernels this wrapper actually launched */ \
        if (e_ != cudaSuccess) return fail(MRA_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)
#define LCHK(expr) LCHK_K(KIND_OTHER, expr)

// one zeroed work-queue counter per persistent launch. The array is zeroed per evaluation; an evaluation that
// uses them all (very many chunks / sub-chunks) re-zeroes the array on the plan stream before reusing it --
// stream order puts that memset after every earlier launch that counted with them
static unsigned long long* take_counter(mra_plan* P) {
    if (P->next_counter >= P->n_counters) {
        cudaMemsetAsync(P->counters, 0, 8 * (size_t)P->n_counters, P->st);
        P->next_counter = 0;
    }
    return P->counters + P->next_counter++;
}

// ranges of level-m regions under the level-c regions [a, b)
static void range_at(const mra_plan* P, int m, long long a, long long b, long long* f, long long* cnt) {
    const long long s = ipow(P->J, m - P->c);
    *f = a * s;
    *cnt = (b - a) * s;
}

// contiguous runs of this rank's level-c regions
static std::vector<std::pair<long long, long long>> my_runs(const mra_plan* P) {
    std::vector<std::pair<long long, long long>> runs;
    if (P->world <= 1) {
        runs.push_back({0, ipow(P->J, P->c - 1)});
        return runs;
    }
    for (long long s : P->my_c) {
        if (!runs.empty() && runs.back().second == s) runs.back().second = s + 1;
        else runs.push_back({s, s + 1});
    }
    return runs;
}

// wide path for the level-(M-1) groups [gf, gf + gc): consumes the precomputed sub-chunks in order
static mra_status eval_wide(mra_plan* P, const TreeParams& tp, long long gf, long long gc, double* gout,
                            long long gout_first) {
    WideParams wp;
    wp.G = P->wG; wp.ldG = P->wldG; wp.S = P->wS; wp.S_off = P->wS_off; wp.S_ld = P->wS_ld;
    wp.D = P->wD; wp.D_off = P->wD_off; wp.lblk = P->wlblk;
    wp.kb0 = wp.kb1 = 0;
    const int q = (int)q_of(P->M - 1, P->rh);
    cudaStream_t st = P->st;
    long long done = 0;
    while (done < gc) {
        if (P->wsub_next >= P->wsubs.size()) return fail(MRA_E_CUDA, "internal: wide sub-chunk schedule exhausted");
        const auto& w = P->wsubs[P->wsub_next++];
        if (w.g0 != gf + done) return fail(MRA_E_CUDA, "internal: wide sub-chunk schedule out of order");
        wp.G_base = P->leaf_off[w.g0 * P->J];
        LCHK_K(KIND_COVGEN, launch_wide(6, tp, P->treg, wp, 0, P->wtasks + w.chain_off, w.chain_n, P->grid, take_counter(P), st));
        if (w.cs_n > 0) {
            LCHK_K(KIND_CHAIN, launch_wide_chsig(tp, P->treg, wp, P->wtasks + w.cs_off, w.cs_n, take_counter(P),
                                                 P->mring.flags + 3 * P->mring.maxg, w.g0 * P->J, w.gcount * P->J, st));
        } else {
            LCHK_K(KIND_CHAIN, launch_wide(0, tp, P->treg, wp, 0, P->wtasks + w.chain_off, w.chain_n, P->grid, take_counter(P), st));
            LCHK_K(KIND_SIGMA, launch_wide(1, tp, P->treg, wp, 0, P->wtasks + w.sigma_off, w.sigma_n, P->grid, take_counter(P), st));
        }
        constexpr int NBS = 8;   // as in size_wide
        for (size_t s2 = 0; s2 < w.diag_n.size(); s2++) {
            const int kb0 = (int)s2 / NBS * NBS;
            wp.kb0 = kb0;
            wp.kb1 = (int)s2;
            if (w.upd_n[s2] > 0)
                LCHK_K(KIND_FACTOR, launch_wide(2, tp, P->treg, wp, (int)s2, P->wtasks + w.upd_off[s2], w.upd_n[s2], P->grid,
                                                take_counter(P), st));
            LCHK_K(KIND_FACTOR, launch_wide(3, tp, P->treg, wp, (int)s2, P->wtasks + w.diag_off[s2], w.diag_n[s2], P->grid,
                                            take_counter(P), st));
            LCHK_K(KIND_FACTOR, launch_wide(4, tp, P->treg, wp, (int)s2, P->wtasks + w.pf_off[s2], w.pf_n[s2], P->grid,
                                            take_counter(P), st));
            if (w.tr_n[s2] > 0) {
                wp.kb1 = kb0 + NBS;
                LCHK_K(KIND_FACTOR, launch_wide(2, tp, P->treg, wp, (int)s2, P->wtasks + w.tr_off[s2], w.tr_n[s2], P->grid,
                                                take_counter(P), st));
            }
        }
        if (w.trsm_n > 0)
            LCHK_K(KIND_SOLVE, launch_wide(5, tp, P->treg, wp, 0, P->wtasks + w.trsm_off, w.trsm_n, P->grid, take_counter(P), st));
        LCHK_K(KIND_SYRKMERGE, launch_wide_mtile(tp, P->treg, wp, w.g0, w.gcount, gout, gout_first, q, P->wtasks + w.mt_off,
                                                  w.mt_n, P->grid, take_counter(P), P->mring, st));
        done += w.gcount;
    }
    return MRA_OK;
}

// prior + posterior below (and at) level c for this rank's subtrees
static mra_status flush_host_y(mra_plan* P);

static mra_status eval_lower(mra_plan* P, const TreeParams& tp0) {
    const int M = P->M, J = P->J, rh = P->rh, c = P->c;
    const TreeParams& tp = tp0;
    cudaStream_t st = P->st;
    auto runs = my_runs(P);
    // prior: levels < c for every region, levels >= c for own subtrees (streaming plans: per chunk, below).
    // With the in-library exchange, rank 0 computes the above-shard levels and broadcasts their chain rows
    // (north_star: "ancestor W and K blocks are broadcast down with NCCL"); without it every rank
    // replicates that small computation (21 regions for C3 at 8 GPUs)
    for (int m = 1; m < M; m++) {
        if (m == c && P->nccl && c > 1) {
            const NcclApi* nc = nccl_api();
            const size_t cnt_top = (size_t)(P->prior_base[c] - P->prior_base[1]);   // levels 1..c-1, contiguous
            if (cnt_top) {
                const ncclResult_t r0 = nc->broadcast(P->prior + P->prior_base[1], P->prior + P->prior_base[1], cnt_top,
                                                      ncclFloat64, 0, P->comm, st);
                if (r0 != ncclSuccess) return fail(MRA_E_NCCL, std::string("ncclBroadcast(prior rows): ") + nc->errStr(r0));
            }
        }
        if (m >= c && P->stream) break;
        if (m < c) {
            if (P->nccl && P->rank != 0) continue;   // received from rank 0 (above)
            TreeParams t2 = tp;
            LCHK_K(KIND_PRIOR, launch_prior(t2, P->treg, m, 0, ipow(J, m - 1), P->grid, P->ws, P->ws_stride, take_counter(P), st));
        } else {
            for (auto& rg : runs) {
                long long f, cnt;
                range_at(P, m, rg.first, rg.second, &f, &cnt);
                LCHK_K(KIND_PRIOR, launch_prior(tp, P->treg, m, f, cnt, P->grid, P->ws, P->ws_stride, take_counter(P), st));
            }
        }
    }
    mra_status hs = flush_host_y(P);
    if (hs) return hs;
    // posterior: chunks of Kc level-c regions
    for (auto& rg : runs) {
        for (long long a = rg.first; a < rg.second; a += P->Kc) {
            const long long b = std::min(rg.second, a + P->Kc);
            const int mg = M - 1;
            if (M == 1) {
                LCHK_K(KIND_BOTTOM, launch_bottom(tp, 0, 1, nullptr, 0, 0, P->grid, P->ws, P->L, take_counter(P), st));
                continue;
            }
            TreeParams tp = tp0;
            if (P->stream) {
                // this chunk's prior rows, levels c..M-1, top-down (their ancestors above c are resident)
                for (int m = c; m < M; m++) {
                    long long f, cnt;
                    range_at(P, m, a, b, &f, &cnt);
                    tp.prior_first[m] = f;
                    LCHK_K(KIND_PRIOR, launch_prior(tp, P->treg, m, f, cnt, P->grid, P->ws, P->ws_stride, take_counter(P), st));
                }
            }
            long long gf, gc;
            range_at(P, mg, a, b, &gf, &gc);
            double* gout = (mg <= c) ? P->out_full[mg] : P->out_chunk[mg];
            const long long gout_first = (mg <= c) ? 0 : gf;
            if (P->wide) {
                mra_status ws_ = eval_wide(P, tp, gf, gc, gout, gout_first);
                if (ws_) return ws_;
            } else {
                LCHK_K(KIND_BOTTOM, launch_bottom(tp, gf, gc, gout, gout_first, (int)q_of(mg, rh), P->grid, P->ws,
                                                  P->L, take_counter(P), st));
            }
            for (int m = mg - 1; m >= c; m--) {
                long long f, cnt, cf, ccnt;
                range_at(P, m, a, b, &f, &cnt);
                range_at(P, m + 1, a, b, &cf, &ccnt);
                const double* cout_ = (m + 1 <= c) ? P->out_full[m + 1] : P->out_chunk[m + 1];
                const long long cfirst = (m + 1 <= c) ? 0 : cf;
                double* o = (m <= c) ? P->out_full[m] : P->out_chunk[m];
                const long long ofirst = (m <= c) ? 0 : f;
                LCHK_K(KIND_MERGE, launch_merge(tp, P->treg, m, f, cnt, cout_, cfirst, o, ofirst, (int)q_of(m, rh), P->grid, P->ws,
                                  P->ws_stride, take_counter(P), st));
            }
        }
    }
    return MRA_OK;
}

// merges above the chunk level and log L
static mra_status eval_upper(mra_plan* P, const TreeParams& tp) {
    const int M = P->M, J = P->J, rh = P->rh, c = P->c;
    for (int m = std::min(c - 1, M - 2); m >= 1; m--)
        LCHK_K(KIND_MERGE, launch_merge(tp, P->treg, m, 0, ipow(J, m - 1), P->out_full[m + 1], 0, P->out_full[m], 0, (int)q_of(m, rh),
                          P->grid, P->ws, P->ws_stride, take_counter(P), P->st));
    LCHK(launch_final(tp, (double)P->N, P->loglik_d, P->st));
    return MRA_OK;
}

static mra_status check_err(mra_plan* P) {
    int h[4];
    cudaError_t e = cudaMemcpyAsync(h, P->err, 16, cudaMemcpyDeviceToHost, P->st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(P->st);
    if (e != cudaSuccess) return fail(MRA_E_CUDA, std::string("evaluation: ") + cudaGetErrorString(e));
    if (P->prof) prof_collect(P);
    if (h[0]) {
        long long idx;
        std::memcpy(&idx, h + 2, 8);
        char buf[160];
        snprintf(buf, sizeof buf, "Cholesky failed (matrix not positive definite) at region level %d index %lld",
                 h[1], idx);
        return fail(MRA_E_NUMERIC, buf);
    }
    return MRA_OK;
}

static mra_status begin_eval(mra_plan* P, const double* d_y, const mra_theta* th) {
    g_err.clear();
    if (P->device < 0) return fail(MRA_E_CUDA, "host-only plan (device -2) cannot evaluate");
    P->launches = 0;
    P->next_counter = 0;
    P->post_valid = false;   // zs (and, when requested, the posterior state) are overwritten below
    mra_status s = check_theta(th);
    if (s) return s;
    if (cudaSetDevice(P->device) != cudaSuccess) return fail(MRA_E_CUDA, "cudaSetDevice failed");
    CU(cudaMemsetAsync(P->counters, 0, 8 * (size_t)P->n_counters, P->st));
    P->wsub_next = 0;
    CU(cudaMemsetAsync(P->err, 0, 16, P->st));
    if (!P->host_y_pending) LCHK(launch_gather(d_y, P->perm_d, P->zs, P->N, P->st));
    return MRA_OK;
}

// the deferred host-y copy (mra_loglik / mra_loglik_batch): issued after the prior launches, on the copy
// stream, so it overlaps them; the gather into leaf order then waits for it on the plan stream
static mra_status flush_host_y(mra_plan* P) {
    if (!P->host_y_pending) return MRA_OK;
    if (!P->cst) {
        CU(cudaStreamCreateWithFlags(&P->cst, cudaStreamNonBlocking));
        CU(cudaEventCreateWithFlags(&P->cev, cudaEventDisableTiming));
    }
    CU(cudaMemcpyAsync(P->zin, P->host_y_pending, 8 * P->n_in, cudaMemcpyHostToDevice, P->cst));
    CU(cudaEventRecord(P->cev, P->cst));
    CU(cudaStreamWaitEvent(P->st, P->cev, 0));
    P->host_y_pending = nullptr;
    LCHK(launch_gather(P->zin, P->perm_d, P->zs, P->N, P->st));
    return MRA_OK;
}

static mra_status ensure_post(mra_plan* P) {
    if (P->post) return MRA_OK;
    if (P->stream)
        return fail(MRA_E_CONFIG, "this plan streams its prior rows per chunk (stream_prior, NEXT-4) and keeps no "
                                  "posterior state; build it with stream_prior = -1 for posterior means, smoothing "
                                  "or prediction");
    const int M = P->M, J = P->J, rh = P->rh;
    long long tot = 0;
    for (int m = 1; m < M; m++) {
        P->post_base[m] = tot;
        tot += ipow(J, m - 1) * ((long long)rh * rh + q_of(m, rh) * rh);
    }
    mra_status s;
    if ((s = dalloc(P, (void**)&P->post, 8 * std::max<long long>(tot, 1), "posterior state"))) return s;
    if ((s = dalloc(P, (void**)&P->muhat, 8 * std::max<long long>(P->nint * rh, 1), "muhat"))) return s;
    if ((s = dalloc(P, (void**)&P->mu_d, 8 * std::max<long long>(P->nint * rh, 1), "mu"))) return s;
    if ((s = dalloc(P, (void**)&P->smooth_d, 8 * (long long)P->n_in, "smooth"))) return s;
    if (P->wide) {
        // the wide path keeps no per-CTA leaf workspace; smoothing recomputes each leaf on one CTA
        WsLayout L = P->L;
        const long long mleaf = std::max<long long>(P->max_leaf, 1);
        L.ldS = (int)round_up(mleaf, 2);
        long long o = 0;
        L.oG = o; o += round_up(mleaf * L.ldG, 32);
        L.oS = o; o += round_up(mleaf * (long long)L.ldS, 32);
        L.oD = o; o += ((mleaf + 63) / 64) * 4096;
        L.oA = L.oF = L.oL = o;
        L.oV = o; o += round_up(mleaf, 32);
        L.stride = round_up(o, 64);
        size_t freeb = 0, totalb = 0;
        cudaMemGetInfo(&freeb, &totalb);
        long long slots = std::min<long long>(P->grid, std::max<long long>(1, (long long)(0.5 * freeb / (8.0 * L.stride))));
        P->Ls = L;
        P->smooth_grid = (int)slots;
        if ((s = dalloc(P, (void**)&P->ws_smooth, 8 * L.stride * slots, "smoothing workspace"))) return s;
    }
    return MRA_OK;
}

// NaN / Inf scan of a host array (OpenMP above 4M values: 47M in a few ms; below, waking the thread
// team costs more than the scan)
static bool all_finite(const double* y, uint64_t n) {
    long long bad = 0;
#pragma omp parallel for schedule(static) reduction(+ : bad) if (n > (4u << 20))
    for (long long i = 0; i < (long long)n; i++) bad += !std::isfinite(y[i]);
    return bad == 0;
}

static mra_status run_eval_nccl(mra_plan* P, const double* d_y, const mra_theta* th, double* loglik, mra_post* post,
                                bool host_post);

// opts.graph: the whole log-L evaluation (memsets, gather, prior, the wide phases, merges, final) captured once on the
// plan stream as a CUDA graph and replayed; the kernels read theta from P->theta_d (refreshed before each replay),
// so the graph depends only on the plan, the y pointer and the covariance family (re-captured when those change)
static mra_status run_eval_graph_on(mra_plan* P, const double* d_y, const mra_theta* th, double* loglik,
                                   mra_post* post);
static mra_status run_eval_graph(mra_plan* P, const double* d_y, const mra_theta* th, double* loglik, mra_post* post) {
    mra_status s = check_theta(th);
    if (s) return s;
    if (cudaSetDevice(P->device) != cudaSuccess) return fail(MRA_E_CUDA, "cudaSetDevice failed");
    g_err.clear();
    // capture / replay on the plan's own stream, after everything the caller queued (e.g. the write of y)
    CU(cudaEventRecord(P->gev, P->st));
    CU(cudaStreamWaitEvent(P->gst, P->gev, 0));
    cudaStream_t user = P->st;
    P->st = P->gst;
    s = run_eval_graph_on(P, d_y, th, loglik, post);
    P->st = user;
    return s;
}
static mra_status run_eval_graph_on(mra_plan* P, const double* d_y, const mra_theta* th, double* loglik,
                                   mra_post* post) {
    mra_status s;
    if (!P->gexec || P->g_y != d_y || P->g_cov != th->cov) {
        if (P->gexec) { cudaGraphExecDestroy(P->gexec); P->gexec = nullptr; }
        CU(cudaStreamBeginCapture(P->st, cudaStreamCaptureModeThreadLocal));
        mra_status cs = begin_eval(P, d_y, th);
        TreeParams tp = tree_params(P, th);
        tp.theta_dev = P->theta_d;
        if (!cs) cs = eval_lower(P, tp);
        if (!cs) cs = eval_upper(P, tp);
        cudaGraph_t g = nullptr;
        const cudaError_t ec = cudaStreamEndCapture(P->st, &g);
        if (cs) { if (g) cudaGraphDestroy(g); return cs; }
        if (ec != cudaSuccess) return fail(MRA_E_CUDA, std::string("graph capture: ") + cudaGetErrorString(ec));
        const cudaError_t ei = cudaGraphInstantiate(&P->gexec, g, 0);
        cudaGraphDestroy(g);
        if (ei != cudaSuccess) { P->gexec = nullptr; return fail(MRA_E_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ei)); }
        P->g_y = d_y;
        P->g_cov = th->cov;
        P->g_launches = P->launches;
    }
    P->post_valid = false;
    P->theta_h[0] = th->sigma2; P->theta_h[1] = th->rho; P->theta_h[2] = th->tau2; P->theta_h[3] = 0.0;
    CU(cudaMemcpyAsync(P->theta_d, P->theta_h, 32, cudaMemcpyHostToDevice, P->st));
    CU(cudaGraphLaunch(P->gexec, P->st));
    P->launches = P->g_launches;
    double ll = NAN;
    CU(cudaMemcpyAsync(&ll, P->loglik_d, 8, cudaMemcpyDeviceToHost, P->st));
    if ((s = check_err(P))) return s;
    if (loglik) *loglik = ll;
    if (post) {
        CU(cudaMemcpy(&post->d, P->dreg, 8, cudaMemcpyDeviceToHost));
        CU(cudaMemcpy(&post->u, P->ureg, 8, cudaMemcpyDeviceToHost));
        if (post->region_d) CU(cudaMemcpy(post->region_d, P->dreg, 8 * P->nreg, cudaMemcpyDeviceToHost));
        if (post->region_u) CU(cudaMemcpy(post->region_u, P->ureg, 8 * P->nreg, cudaMemcpyDeviceToHost));
    }
    return MRA_OK;
}

static mra_status run_eval(mra_plan* P, const double* d_y, const mra_theta* th, double* loglik, mra_post* post,
                           bool host_post) {
    if (P->nccl) return run_eval_nccl(P, d_y, th, loglik, post, host_post);
    if (P->world > 1)
        return fail(MRA_E_CONFIG, "sharded plan without a communicator (opts.nccl_id): use mra_loglik_shard / "
                                  "mra_loglik_finish");
    mra_status s;
    const bool want_state = post && (post->mu || post->smooth);
    if (want_state && (s = ensure_post(P))) return s;
    if (P->use_graph && !want_state && !P->prof && !P->host_y_pending) return run_eval_graph(P, d_y, th, loglik, post);
    if ((s = begin_eval(P, d_y, th))) return s;
    TreeParams tp = tree_params(P, th);
    if (want_state) tp.post = P->post;
    if ((s = eval_lower(P, tp))) return s;
    if ((s = eval_upper(P, tp))) return s;
    double ll = NAN;
    CU(cudaMemcpyAsync(&ll, P->loglik_d, 8, cudaMemcpyDeviceToHost, P->st));
    if ((s = check_err(P))) return s;
    if (loglik) *loglik = ll;
    if (post) {
        CU(cudaMemcpy(&post->d, P->dreg, 8, cudaMemcpyDeviceToHost));
        CU(cudaMemcpy(&post->u, P->ureg, 8, cudaMemcpyDeviceToHost));
        if (post->region_d) CU(cudaMemcpy(post->region_d, P->dreg, 8 * P->nreg, cudaMemcpyDeviceToHost));
        if (post->region_u) CU(cudaMemcpy(post->region_u, P->ureg, 8 * P->nreg, cudaMemcpyDeviceToHost));
    }
    if (want_state) {
        for (int m = 1; m < P->M; m++) LCHK(launch_mu(tp, m, P->muhat, P->mu_d, 0, ipow(P->J, m - 1), P->st));
        if (post->smooth) {
            LCHK(launch_fill(P->smooth_d, (long long)P->n_in, NAN, P->st));
            LCHK(launch_smooth(tp, P->muhat, P->perm_d, P->smooth_d, P->wide ? P->smooth_grid : P->grid,
                               P->wide ? P->ws_smooth : P->ws, P->wide ? P->Ls : P->L, take_counter(P), 0, P->nleaf,
                               P->st));
        }
        if ((s = check_err(P))) return s;
        const size_t nmu = 8 * (size_t)P->nint * P->rh;
        const cudaMemcpyKind k = host_post ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
        if (post->mu && nmu) CU(cudaMemcpyAsync(post->mu, P->mu_d, nmu, k, P->st));
        if (post->smooth) CU(cudaMemcpyAsync(post->smooth, P->smooth_d, 8 * P->n_in, k, P->st));
        CU(cudaStreamSynchronize(P->st));
        P->post_valid = true;
        P->post_theta = *th;
    }
    return MRA_OK;
}

// ----------------------------------------------------------------------- prediction
extern "C" mra_status mra_predict(mra_plan* P, const double* qx, const double* qy, uint64_t nq, double* mean,
                                  double* var) {
    return guarded([&]() -> mra_status {
        g_err.clear();
        if (!P || !qx || !qy || !mean || !var) return fail(MRA_E_ARG, "NULL argument");
        if (P->device < 0) return fail(MRA_E_CUDA, "host-only plan (device -2) cannot evaluate");
        if (P->world > 1 && !P->nccl)
            return fail(MRA_E_CONFIG, "prediction on a sharded plan needs the in-library exchange (opts.nccl_id)");
        if (!P->post_valid)
            return fail(MRA_E_ARG, "no posterior state: evaluate with posterior state (post->mu or post->smooth) first");
        if (nq == 0) return MRA_OK;
        if (cudaSetDevice(P->device) != cudaSuccess) return fail(MRA_E_CUDA, "cudaSetDevice failed");
        const int M = P->M, J = P->J;
        // leaf of each query by the plan's descent (half-open boxes); outside the root -> NaN
        std::vector<long long> qleaf(nq);
        for (uint64_t i = 0; i < nq; i++) {
            const double px = qx[i], py = qy[i];
            if (!std::isfinite(px) || !std::isfinite(py)) return fail(MRA_E_ARG, "non-finite query location");
            if (!(px >= P->root[0] && px < P->root[1] && py >= P->root[2] && py < P->root[3])) { qleaf[i] = -1; continue; }
            long long t = 0;
            for (int m = 1; m < M; m++) {
                const double* b = &P->box[4 * (lvl_first(J, m) + t)];
                const double mx = 0.5 * (b[0] + b[1]), my = 0.5 * (b[2] + b[3]);
                int c;
                if (J == 4) c = (px >= mx ? 1 : 0) | (py >= my ? 2 : 0);
                else if ((b[1] - b[0]) >= (b[3] - b[2])) c = px >= mx ? 1 : 0;
                else c = py >= my ? 1 : 0;
                t = t * J + c;
            }
            qleaf[i] = t;
        }
        std::vector<long long> qoff(P->nleaf + 1, 0);
        for (uint64_t i = 0; i < nq; i++) if (qleaf[i] >= 0) qoff[qleaf[i] + 1]++;
        // sharded plans: this rank predicts the queries of its own leaves; the others come from the all-reduce
        std::vector<char> own_leaf;
        if (P->nccl) {
            own_leaf.assign(P->nleaf, 0);
            const long long per = ipow(J, M - P->c);
            for (long long t : P->my_c)
                for (long long l = t * per; l < (t + 1) * per; l++) own_leaf[l] = 1;
        }
        std::vector<long long> leaves;
        for (long long l = 0; l < P->nleaf; l++) {
            if (qoff[l + 1] && (own_leaf.empty() || own_leaf[l])) leaves.push_back(l);
            qoff[l + 1] += qoff[l];
        }
        const long long nin = qoff[P->nleaf];
        std::vector<long long> fillp(qoff.begin(), qoff.end() - 1), qperm(std::max<long long>(nin, 1));
        std::vector<double> qxy(2 * std::max<long long>(nin, 1));
        for (uint64_t i = 0; i < nq; i++)
            if (qleaf[i] >= 0) {
                const long long d = fillp[qleaf[i]]++;
                qperm[d] = (long long)i;
                qxy[2 * d] = qx[i];
                qxy[2 * d + 1] = qy[i];
            }
        mra_status s;
        // per-CTA workspace: the leaf's G, Sigma, inverted diagonal blocks, r, and the query tiles
        if (!P->ws_pred) {
            const int Pg = (M - 1) * P->rh;
            WsLayout L{};
            const long long mleaf = std::max<long long>(P->max_leaf, 1);
            L.ldG = (int)round_up(Pg + 1, 2);
            L.ldS = (int)round_up(mleaf, 2);
            long long o = 0;
            L.oG = o; o += round_up(mleaf * L.ldG, 32);
            L.oS = o; o += round_up(mleaf * (long long)L.ldS, 32);
            L.oD = o; o += ((mleaf + 63) / 64) * 4096;
            L.oV = o; o += round_up(mleaf, 32);
            L.oQ = o; o += round_up(64LL * L.ldG, 32);
            L.oE = o; o += round_up(mleaf * 64, 32);
            L.oW = o; o += round_up(64LL * L.ldG, 32);
            L.oA = L.oF = L.oL = 0;
            L.stride = round_up(o, 64);
            size_t freeb = 0, totalb = 0;
            cudaMemGetInfo(&freeb, &totalb);
            long long slots = std::min<long long>(P->grid, std::max<long long>(1, (long long)(0.4 * freeb / (8.0 * L.stride))));
            P->Lp = L;
            P->pred_grid = (int)slots;
            if ((s = dalloc(P, (void**)&P->ws_pred, 8 * L.stride * slots, "prediction workspace"))) return s;
        }
        double *d_qxy = nullptr, *d_mean = nullptr, *d_var = nullptr;
        long long *d_qoff = nullptr, *d_qperm = nullptr, *d_leaves = nullptr;
        auto release = [&]() {
            cudaStreamSynchronize(P->st);
            for (void* v : {(void*)d_qxy, (void*)d_mean, (void*)d_var, (void*)d_qoff, (void*)d_qperm, (void*)d_leaves})
                tfree(P, v);
        };
    #define PCU(call)                                                                              \
        do {                                                                                       \
            cudaError_t e_ = (call);                                                               \
            if (e_ != cudaSuccess) {                                                               \
                release();                                                                         \
                return fail(e_ == cudaErrorMemoryAllocation ? MRA_E_OOM : MRA_E_CUDA,              \
                            std::string(#call) + ": " + cudaGetErrorString(e_));                   \
            }                                                                                      \
        } while (0)
        PCU(talloc(P, (void**)&d_qxy, 16 * std::max<long long>(nin, 1)));
        PCU(talloc(P, (void**)&d_mean, 8 * nq));
        PCU(talloc(P, (void**)&d_var, 8 * nq));
        PCU(talloc(P, (void**)&d_qoff, 8 * (P->nleaf + 1)));
        PCU(talloc(P, (void**)&d_qperm, 8 * std::max<long long>(nin, 1)));
        PCU(talloc(P, (void**)&d_leaves, 8 * std::max<size_t>(leaves.size(), 1)));
        PCU(cudaMemcpyAsync(d_qxy, qxy.data(), 16 * std::max<long long>(nin, 1), cudaMemcpyHostToDevice, P->st));
        PCU(cudaMemcpyAsync(d_qoff, qoff.data(), 8 * (P->nleaf + 1), cudaMemcpyHostToDevice, P->st));
        PCU(cudaMemcpyAsync(d_qperm, qperm.data(), 8 * std::max<long long>(nin, 1), cudaMemcpyHostToDevice, P->st));
        if (!leaves.empty())
            PCU(cudaMemcpyAsync(d_leaves, leaves.data(), 8 * leaves.size(), cudaMemcpyHostToDevice, P->st));
        PCU(launch_fill(d_mean, (long long)nq, P->nccl ? 0.0 : NAN, P->st));
        PCU(launch_fill(d_var, (long long)nq, P->nccl ? 0.0 : NAN, P->st));
        PCU(cudaMemsetAsync(P->err, 0, 16, P->st));
        PCU(cudaMemsetAsync(P->counters, 0, 8, P->st));
        TreeParams tp = tree_params(P, &P->post_theta);
        tp.post = P->post;
        PredParams pp{};
        pp.qxy = d_qxy; pp.q_off = d_qoff; pp.q_perm = d_qperm; pp.leaves = d_leaves;
        pp.n_leaves = (long long)leaves.size(); pp.muhat = P->muhat; pp.mean = d_mean; pp.var = d_var;
        const unsigned long long k0 = g_kernel_launches;
        PCU(launch_predict(tp, pp, P->pred_grid, P->ws_pred, P->Lp, P->counters, P->st));
        P->launches = g_kernel_launches - k0;
        if (P->nccl) {
            const NcclApi* nc = nccl_api();
            ncclResult_t r0 = nc->allReduce(d_mean, d_mean, nq, ncclFloat64, ncclSum, P->comm, P->st);
            if (r0 == ncclSuccess) r0 = nc->allReduce(d_var, d_var, nq, ncclFloat64, ncclSum, P->comm, P->st);
            if (r0 != ncclSuccess) {
                release();
                return fail(MRA_E_NCCL, std::string("ncclAllReduce(prediction): ") + nc->errStr(r0));
            }
        }
        PCU(cudaMemcpyAsync(mean, d_mean, 8 * nq, cudaMemcpyDeviceToHost, P->st));
        PCU(cudaMemcpyAsync(var, d_var, 8 * nq, cudaMemcpyDeviceToHost, P->st));
        int h[4];
        PCU(cudaMemcpyAsync(h, P->err, 16, cudaMemcpyDeviceToHost, P->st));
        PCU(cudaStreamSynchronize(P->st));
    #undef PCU
        release();
        if (h[0]) return fail(MRA_E_NUMERIC, "Cholesky failed while recomputing a leaf for prediction");
        if (P->nccl)
            for (uint64_t i = 0; i < nq; i++)
                if (qleaf[i] < 0) mean[i] = var[i] = NAN;
        return MRA_OK;
    });
}

extern "C" mra_status mra_loglik_dev(mra_plan* P, const double* d_y, const mra_theta* th, double* loglik,
                                     mra_post* post) {
    return guarded([&]() -> mra_status {
        if (!P || !d_y) return fail(MRA_E_ARG, "plan or y is NULL");
        return run_eval(P, d_y, th, loglik, post, false);
    });
}

extern "C" mra_status mra_loglik(mra_plan* P, const double* y, const mra_theta* th, double* loglik, mra_post* post) {
    return guarded([&]() -> mra_status {
        if (!P || !y) return fail(MRA_E_ARG, "plan or y is NULL");
        if (P->device < 0) return fail(MRA_E_CUDA, "host-only plan (device -2) cannot evaluate");
        if (!all_finite(y, P->n_in)) return fail(MRA_E_ARG, "non-finite observation value");
        if (cudaSetDevice(P->device) != cudaSuccess) return fail(MRA_E_CUDA, "cudaSetDevice failed");
        P->host_y_pending = y;   // copied by flush_host_y, overlapping the prior levels
        const mra_status s = run_eval(P, P->zin, th, loglik, post, true);
        P->host_y_pending = nullptr;
        return s;
    });
}

// one log-likelihood evaluation issued on the context's stream without waiting (theta lanes)
static mra_status issue_eval(mra_plan* P, const double* d_y, const mra_theta* th) {
    mra_status s;
    if ((s = begin_eval(P, d_y, th))) return s;
    TreeParams tp = tree_params(P, th);
    if ((s = eval_lower(P, tp))) return s;
    return eval_upper(P, tp);
}
static mra_status finish_eval(mra_plan* P, double* loglik) {
    mra_status s = check_err(P);   // synchronises the context's stream
    if (s) return s;
    CU(cudaMemcpy(loglik, P->loglik_d, 8, cudaMemcpyDeviceToHost));
    return MRA_OK;
}

extern "C" mra_status mra_loglik_batch_dev(mra_plan* P, const double* d_y, const mra_theta* th, int n_theta,
                                           double* loglik) {
    return guarded([&]() -> mra_status {
        if (!P || !d_y || !th || !loglik || n_theta < 0) return fail(MRA_E_ARG, "bad arguments");
        uint64_t total = 0;
        const int L = std::min<int>(n_theta, 1 + (int)P->lanes.size());
        if (L <= 1 || P->world > 1) {
            for (int i = 0; i < n_theta; i++) {
                mra_status s = run_eval(P, d_y, th + i, loglik + i, nullptr, false);
                if (s) return s;
                total += P->launches;
            }
            P->launches = total;
            return MRA_OK;
        }
        for (int i = 0; i < n_theta; i++)
            if (mra_status s = check_theta(th + i)) return s;
        if (cudaSetDevice(P->device) != cudaSuccess) return fail(MRA_E_CUDA, "cudaSetDevice failed");
        // the lanes start after everything the caller queued on the plan stream (e.g. the write of y)
        if (!P->lane_ev) CU(cudaEventCreateWithFlags(&P->lane_ev, cudaEventDisableTiming));
        CU(cudaEventRecord(P->lane_ev, P->st));
        for (mra_plan* Q : P->lanes) CU(cudaStreamWaitEvent(Q->st, P->lane_ev, 0));
        auto lane = [&](int j) { return j == 0 ? P : P->lanes[j - 1]; };
        for (int i0 = 0; i0 < n_theta; i0 += L) {
            const int nb = std::min(L, n_theta - i0);
            mra_status first = MRA_OK;
            int issued = 0;
            for (int j = 0; j < nb && !first; j++, issued++) first = issue_eval(lane(j), d_y, th + i0 + j);
            for (int j = 0; j < issued; j++) {
                mra_status s = finish_eval(lane(j), loglik + i0 + j);
                if (!first) first = s;
                total += lane(j)->launches;
            }
            if (first) return first;
        }
        P->launches = total;   // every launch of the sweep (mra_last_launches)
        return MRA_OK;
    });
}

extern "C" mra_status mra_loglik_batch(mra_plan* P, const double* y, const mra_theta* th, int n_theta,
                                       double* loglik) {
    return guarded([&]() -> mra_status {
        if (!P || !y || !th || !loglik || n_theta < 0) return fail(MRA_E_ARG, "bad arguments");
        if (P->device < 0) return fail(MRA_E_CUDA, "host-only plan (device -2) cannot evaluate");
        if (!all_finite(y, P->n_in)) return fail(MRA_E_ARG, "non-finite observation value");
        if (cudaSetDevice(P->device) != cudaSuccess) return fail(MRA_E_CUDA, "cudaSetDevice failed");
        if (n_theta == 0) return MRA_OK;
        if (!P->lanes.empty()) {   // copied once; the lanes wait for it through the plan stream
            CU(cudaMemcpyAsync(P->zin, y, 8 * P->n_in, cudaMemcpyHostToDevice, P->st));
            return mra_loglik_batch_dev(P, P->zin, th, n_theta, loglik);
        }
        P->host_y_pending = y;   // copied once, during the first evaluation's prior levels
        mra_status s = run_eval(P, P->zin, th, loglik, nullptr, false);
        P->host_y_pending = nullptr;
        if (s) return s;
        const uint64_t first = P->launches;
        s = mra_loglik_batch_dev(P, P->zin, th + 1, n_theta - 1, loglik + 1);
        P->launches += first;
        return s;
    });
}

// ----------------------------------------------------------------------- optimization
// The paper's "optimization" calculation mode: maximise log L over (sigma2, rho, tau2)
// by derivative-free search, each step one full evaluation. Nelder-Mead on the log-parameters inside
// the box [lower, upper] (reflections clamped to the box), a deterministic stand-in for the paper's
// BOBYQA (dlib); non-PD evaluations count as -inf.
extern "C" mra_status mra_optimize(mra_plan* P, const double* d_y, mra_theta* theta, const double* lower,
                                   const double* upper, int max_evals, double tol, double* best_loglik,
                                   int* n_evals) {
    return guarded([&]() -> mra_status {
        if (!P || !d_y || !theta) return fail(MRA_E_ARG, "NULL argument");
        if (P->world > 1 && !P->nccl)
            return fail(MRA_E_CONFIG, "optimization on a sharded plan needs the in-library exchange (opts.nccl_id)");
        mra_status s = check_theta(theta);
        if (s) return s;
        if (max_evals < 1) max_evals = 200;
        if (!(tol > 0)) tol = 1e-6;
        double lo[3], hi[3];
        const double v0[3] = {theta->sigma2, theta->rho, theta->tau2};
        for (int i = 0; i < 3; i++) {
            lo[i] = lower ? std::log(lower[i]) : -INFINITY;
            hi[i] = upper ? std::log(upper[i]) : INFINITY;
            if (lower && upper && !(lower[i] > 0 && upper[i] >= lower[i])) return fail(MRA_E_ARG, "bad bounds");
            if (std::log(v0[i]) < lo[i] || std::log(v0[i]) > hi[i]) return fail(MRA_E_ARG, "initial theta outside the bounds");
        }
        int evals = 0;
        auto clampv = [&](double* v) { for (int i = 0; i < 3; i++) v[i] = std::min(hi[i], std::max(lo[i], v[i])); };
        // objective: -log L (minimised); failures -> +inf
        auto f = [&](const double* v, double* out) -> mra_status {
            mra_theta th = *theta;
            th.sigma2 = std::exp(v[0]); th.rho = std::exp(v[1]); th.tau2 = std::exp(v[2]);
            double ll = NAN;
            mra_status e = run_eval(P, d_y, &th, &ll, nullptr, false);
            evals++;
            if (e == MRA_E_NUMERIC || !std::isfinite(ll)) { *out = INFINITY; g_err.clear(); return MRA_OK; }
            if (e) return e;
            *out = -ll;
            return MRA_OK;
        };
        // several independent points (initial simplex, shrink): one theta sweep, concurrent on a laned plan
        auto f_many = [&](double (*Xs)[3], double* out, int n) -> mra_status {
            if (!P->lanes.empty()) {
                std::vector<mra_theta> ths(n, *theta);
                for (int j = 0; j < n; j++) {
                    ths[j].sigma2 = std::exp(Xs[j][0]); ths[j].rho = std::exp(Xs[j][1]); ths[j].tau2 = std::exp(Xs[j][2]);
                }
                std::vector<double> ll(n, NAN);
                if (mra_loglik_batch_dev(P, d_y, ths.data(), n, ll.data()) == MRA_OK) {
                    bool ok = true;
                    for (int j = 0; j < n; j++) ok = ok && std::isfinite(ll[j]);
                    if (ok) {
                        for (int j = 0; j < n; j++) out[j] = -ll[j];
                        evals += n;
                        return MRA_OK;
                    }
                }
                g_err.clear();   // a failing point: evaluate one by one below (non-PD counts as +inf)
            }
            for (int j = 0; j < n; j++)
                if (mra_status e = f(Xs[j], out + j)) return e;
            return MRA_OK;
        };
        double X[4][3], F[4];
        for (int j = 0; j < 4; j++) {
            for (int i = 0; i < 3; i++) X[j][i] = std::log(v0[i]) + ((j == i + 1) ? 0.5 : 0.0);
            clampv(X[j]);
        }
        if ((s = f_many(X, F, 4))) return s;
        while (evals < max_evals) {
            int ord[4] = {0, 1, 2, 3};
            std::sort(ord, ord + 4, [&](int a, int b) { return F[a] < F[b]; });
            double Xs[4][3], Fs[4];
            for (int j = 0; j < 4; j++) { std::memcpy(Xs[j], X[ord[j]], sizeof Xs[j]); Fs[j] = F[ord[j]]; }
            std::memcpy(X, Xs, sizeof X); std::memcpy(F, Fs, sizeof F);
            double size = 0;
            for (int j = 1; j < 4; j++)
                for (int i = 0; i < 3; i++) size = std::max(size, std::fabs(X[j][i] - X[0][i]));
            if (size < tol || (std::isfinite(F[3]) && std::fabs(F[3] - F[0]) <= tol * (1.0 + std::fabs(F[0])) && size < 1e3 * tol))
                break;
            double c[3] = {0, 0, 0};
            for (int j = 0; j < 3; j++) for (int i = 0; i < 3; i++) c[i] += X[j][i] / 3.0;
            double xr[3], fr;
            for (int i = 0; i < 3; i++) xr[i] = c[i] + (c[i] - X[3][i]);
            clampv(xr);
            if ((s = f(xr, &fr))) return s;
            if (fr < F[0]) {
                double xe[3], fe;
                for (int i = 0; i < 3; i++) xe[i] = c[i] + 2.0 * (c[i] - X[3][i]);
                clampv(xe);
                if ((s = f(xe, &fe))) return s;
                if (fe < fr) { std::memcpy(X[3], xe, sizeof xe); F[3] = fe; }
                else { std::memcpy(X[3], xr, sizeof xr); F[3] = fr; }
            } else if (fr < F[2]) {
                std::memcpy(X[3], xr, sizeof xr); F[3] = fr;
            } else {
                double xc[3], fc;
                const bool outside = fr < F[3];
                for (int i = 0; i < 3; i++) xc[i] = outside ? c[i] + 0.5 * (xr[i] - c[i]) : c[i] + 0.5 * (X[3][i] - c[i]);
                clampv(xc);
                if ((s = f(xc, &fc))) return s;
                if (fc < (outside ? fr : F[3])) { std::memcpy(X[3], xc, sizeof xc); F[3] = fc; }
                else {   // shrink towards the best vertex
                    for (int j = 1; j < 4; j++)
                        for (int i = 0; i < 3; i++) X[j][i] = X[0][i] + 0.5 * (X[j][i] - X[0][i]);
                    if ((s = f_many(X + 1, F + 1, 3))) return s;
                }
            }
        }
        int b = 0;
        for (int j = 1; j < 4; j++) if (F[j] < F[b]) b = j;
        if (!std::isfinite(F[b])) return fail(MRA_E_NUMERIC, "no feasible parameter point found");
        theta->sigma2 = std::exp(X[b][0]); theta->rho = std::exp(X[b][1]); theta->tau2 = std::exp(X[b][2]);
        if (best_loglik) *best_loglik = -F[b];
        if (n_evals) *n_evals = evals;
        return MRA_OK;
    });
}

// ------------------------------------------------------------------------ sharding
// Exchange buffer (include/mra.h mra_shard_size): per level-c region the lower triangle of its q x q augmented
// output packed row by row, then the regions' d, u, then one error flag -- zero outside this rank's slots, so
// a sum-reduce over ranks assembles every region once (the paper's supervisor gather).
static long long xbuf_len(const mra_plan* P) {
    const long long ns = ipow(P->J, P->c - 1), q = q_of(P->c, P->rh);
    return ns * q * (q + 1) / 2 + 2 * ns + 1;
}

extern "C" uint64_t mra_shard_size(const mra_plan* P) {
    if (!P) return 0;
    return (uint64_t)xbuf_len(P);
}

// this rank's subtrees, packed into d_xbuf. check = false (in-library exchange): a Cholesky failure is not
// returned here but travels to rank 0 as the buffer's error flag, so no rank leaves the collectives early
static mra_status shard_impl(mra_plan* P, const double* d_y, const mra_theta* th, double* d_xbuf, bool post,
                             bool check) {
    if (!P || !d_y || !d_xbuf) return fail(MRA_E_ARG, "NULL argument");
    if (P->M < 2) return fail(MRA_E_CONFIG, "sharding needs M >= 2");
    if (P->world <= 1 && !P->nccl) return fail(MRA_E_CONFIG, "not a sharded plan");
    mra_status s;
    if (post && (s = ensure_post(P))) return s;
    if ((s = begin_eval(P, d_y, th))) return s;
    TreeParams tp = tree_params(P, th);
    if (post) tp.post = P->post;
    CU(cudaMemsetAsync(P->dreg, 0, 8 * P->nreg, P->st));
    CU(cudaMemsetAsync(P->ureg, 0, 8 * P->nreg, P->st));
    const long long ns = ipow(P->J, P->c - 1), q = q_of(P->c, P->rh);
    CU(cudaMemsetAsync(P->out_full[P->c], 0, 8 * ns * q * q, P->st));
    if ((s = eval_lower(P, tp))) return s;
    const long long f = lvl_first(P->J, P->c);
    LCHK(launch_pack_exchange(P->out_full[P->c], ns, (int)q, P->dreg + f, P->ureg + f, P->err, d_xbuf, P->st));
    if (check && (s = check_err(P))) return s;
    if (post) {
        P->post_valid = true;   // the own subtrees' merge factors (Li, F) of this theta are kept
        P->post_theta = *th;
    }
    return MRA_OK;
}

extern "C" mra_status mra_loglik_shard(mra_plan* P, const double* d_y, const mra_theta* th, double* d_xbuf) {
    return guarded([&]() -> mra_status { return shard_impl(P, d_y, th, d_xbuf, false, true); });
}

extern "C" mra_status mra_loglik_shard_post(mra_plan* P, const double* d_y, const mra_theta* th, double* d_xbuf) {
    return guarded([&]() -> mra_status { return shard_impl(P, d_y, th, d_xbuf, true, true); });
}

// rank 0: the reduced buffer -> merges of the levels above the shard level -> log L (and the above-shard
// posterior means into d_mutop). The caller's stream order makes the buffer complete before this runs.
static mra_status finish_impl(mra_plan* P, const mra_theta* th, const double* d_xbuf, double* loglik,
                              double* d_mutop) {
    if (!P || !d_xbuf) return fail(MRA_E_ARG, "NULL argument");
    if (P->device < 0) return fail(MRA_E_CUDA, "host-only plan (device -2) cannot evaluate");
    mra_status s = check_theta(th);
    if (s) return s;
    if (cudaSetDevice(P->device) != cudaSuccess) return fail(MRA_E_CUDA, "cudaSetDevice failed");
    const long long ns = ipow(P->J, P->c - 1), q = q_of(P->c, P->rh);
    double flag = 0.0;
    CU(cudaMemcpyAsync(&flag, d_xbuf + xbuf_len(P) - 1, 8, cudaMemcpyDeviceToHost, P->st));
    CU(cudaStreamSynchronize(P->st));
    if (flag != 0.0)
        return fail(MRA_E_NUMERIC, "Cholesky failed (matrix not positive definite) in the subtrees of "
                                   + std::to_string((long long)flag) + " shard(s)");
    if (d_mutop && (s = ensure_post(P))) return s;
    TreeParams tp = tree_params(P, th);
    if (d_mutop) tp.post = P->post;
    const long long f = lvl_first(P->J, P->c);
    LCHK(launch_unpack_exchange(d_xbuf, ns, (int)q, P->out_full[P->c], P->dreg + f, P->ureg + f, P->st));
    if ((s = eval_upper(P, tp))) return s;
    double ll = NAN;
    CU(cudaMemcpyAsync(&ll, P->loglik_d, 8, cudaMemcpyDeviceToHost, P->st));
    if (d_mutop) {
        // posterior means of the levels above the shard level (merged here), to be broadcast
        for (int m = 1; m < P->c; m++) LCHK(launch_mu(tp, m, P->muhat, P->mu_d, 0, ipow(P->J, m - 1), P->st));
        const long long top = f * P->rh;
        if (top > 0) {
            CU(cudaMemcpyAsync(d_mutop, P->muhat, 8 * top, cudaMemcpyDeviceToDevice, P->st));
            CU(cudaMemcpyAsync(d_mutop + top, P->mu_d, 8 * top, cudaMemcpyDeviceToDevice, P->st));
        }
    }
    if ((s = check_err(P))) return s;
    if (loglik) *loglik = ll;
    return MRA_OK;
}

extern "C" mra_status mra_loglik_finish(mra_plan* P, const mra_theta* th, const double* d_xbuf, double* loglik) {
    return guarded([&]() -> mra_status { return finish_impl(P, th, d_xbuf, loglik, nullptr); });
}

extern "C" uint64_t mra_mutop_size(const mra_plan* P) {
    if (!P || (P->world <= 1 && !P->nccl)) return 0;
    return (uint64_t)(2 * lvl_first(P->J, P->c) * P->rh);
}

extern "C" mra_status mra_loglik_finish_post(mra_plan* P, const mra_theta* th, const double* d_xbuf, double* loglik,
                                             double* d_mutop) {
    return guarded([&]() -> mra_status {
        if (!d_mutop && P && P->c > 1) return fail(MRA_E_ARG, "d_mutop is NULL");
        return finish_impl(P, th, d_xbuf, loglik, d_mutop);
    });
}

// every rank, after receiving the levels above the shard level: posterior means of its own subtrees' regions
// and the smoothed values of its own observations (S6 for G > 1). fill = value of the entries
// this rank does not own (NaN for the caller-driven API; 0 when the in-library exchange all-reduces them)
static mra_status posterior_local(mra_plan* P, const double* d_mutop, double fill) {
    if (!P->post_valid) return fail(MRA_E_ARG, "no posterior state: run mra_loglik_shard_post first");
    P->next_counter = 0;
    CU(cudaMemsetAsync(P->counters, 0, 8 * (size_t)P->n_counters, P->st));
    CU(cudaMemsetAsync(P->err, 0, 16, P->st));
    TreeParams tp = tree_params(P, &P->post_theta);
    tp.post = P->post;
    const long long top = lvl_first(P->J, P->c) * P->rh, nmu = P->nint * P->rh;
    LCHK(launch_fill(P->mu_d, std::max<long long>(nmu, 1), fill, P->st));
    if (top > 0) {
        CU(cudaMemcpyAsync(P->muhat, d_mutop, 8 * top, cudaMemcpyDeviceToDevice, P->st));
        CU(cudaMemcpyAsync(P->mu_d, d_mutop + top, 8 * top, cudaMemcpyDeviceToDevice, P->st));
    }
    auto runs = my_runs(P);
    for (int m = P->c; m < P->M; m++)
        for (auto& rg : runs) {
            long long f, cnt;
            range_at(P, m, rg.first, rg.second, &f, &cnt);
            LCHK(launch_mu(tp, m, P->muhat, P->mu_d, f, cnt, P->st));
        }
    LCHK(launch_fill(P->smooth_d, (long long)P->n_in, fill, P->st));
    const long long per = ipow(P->J, P->M - P->c);
    for (auto& rg : runs)
        LCHK(launch_smooth(tp, P->muhat, P->perm_d, P->smooth_d, P->wide ? P->smooth_grid : P->grid,
                           P->wide ? P->ws_smooth : P->ws, P->wide ? P->Ls : P->L, take_counter(P), rg.first * per,
                           (rg.second - rg.first) * per, P->st));
    return check_err(P);
}

extern "C" mra_status mra_posterior_shard(mra_plan* P, const double* d_mutop, double* d_mu, double* d_smooth) {
    return guarded([&]() -> mra_status {
        g_err.clear();
        if (!P || (!d_mutop && P->c > 1)) return fail(MRA_E_ARG, "NULL argument");
        if (P->world <= 1 && !P->nccl) return fail(MRA_E_CONFIG, "not a sharded plan");
        if (cudaSetDevice(P->device) != cudaSuccess) return fail(MRA_E_CUDA, "cudaSetDevice failed");
        P->launches = 0;
        mra_status s = posterior_local(P, d_mutop, NAN);
        if (s) return s;
        const long long nmu = P->nint * P->rh;
        if (d_mu && nmu) CU(cudaMemcpyAsync(d_mu, P->mu_d, 8 * nmu, cudaMemcpyDeviceToDevice, P->st));
        if (d_smooth) CU(cudaMemcpyAsync(d_smooth, P->smooth_d, 8 * P->n_in, cudaMemcpyDeviceToDevice, P->st));
        CU(cudaStreamSynchronize(P->st));
        return MRA_OK;
    });
}

// ------------------------------------------------------- in-library exchange (opts.nccl_id)
#define NC(call, what)                                                                          \
    do {                                                                                        \
        const ncclResult_t r_ = (call);                                                         \
        if (r_ != ncclSuccess) return fail(MRA_E_NCCL, std::string(what) + ": " + nc->errStr(r_)); \
    } while (0)

// One sharded evaluation with the exchange step inside the library: every rank runs its
// subtrees (the above-shard prior rows arrive by broadcast inside eval_lower), the packed shard outputs are
// sum-reduced to rank 0, rank 0 merges the levels above the shard level, log L / d / u / the error flag are
// broadcast, and -- when posterior state is requested -- the above-shard means (and merge factors, for
// prediction) are broadcast and each rank's own means / smoothed values are all-reduced into full arrays.
static mra_status run_eval_nccl(mra_plan* P, const double* d_y, const mra_theta* th, double* loglik, mra_post* post,
                                bool host_post) {
    const NcclApi* nc = nccl_api();
    if (!nc || !P->comm) return fail(MRA_E_NCCL, "plan has no communicator");
    const bool want_state = post && (post->mu || post->smooth);
    mra_status s;
    if (want_state && (s = ensure_post(P))) return s;
    if (want_state && !P->mutop) {
        if ((s = dalloc(P, (void**)&P->mutop, 8 * std::max<uint64_t>(1, mra_mutop_size(P)), "mutop"))) return s;
        if ((s = dalloc(P, (void**)&P->sm_sorted, 8 * std::max<long long>(1, P->N), "sorted smoothing"))) return s;
    }
    if ((s = shard_impl(P, d_y, th, P->xbuf, want_state, false))) return s;
    cudaStream_t st = P->st;
    const size_t xl = (size_t)xbuf_len(P);
    NC(nc->reduce(P->xbuf, P->xbuf, xl, ncclFloat64, ncclSum, 0, P->comm, st), "ncclReduce(shard outputs)");
    double hv[4] = {NAN, 0.0, NAN, NAN};
    if (P->rank == 0) {
        const mra_status fs = finish_impl(P, th, P->xbuf, &hv[0], want_state ? P->mutop : nullptr);
        if (fs == MRA_E_NUMERIC) {
            hv[1] = 1.0;
        } else if (fs) {
            hv[1] = 2.0;   // other ranks report a generic failure; rank 0 returns its own status below
        } else {
            CU(cudaMemcpy(&hv[2], P->dreg, 8, cudaMemcpyDeviceToHost));
            CU(cudaMemcpy(&hv[3], P->ureg, 8, cudaMemcpyDeviceToHost));
        }
        CU(cudaMemcpyAsync(P->bcast, hv, 32, cudaMemcpyHostToDevice, st));
        NC(nc->broadcast(P->bcast, P->bcast, 4, ncclFloat64, 0, P->comm, st), "ncclBroadcast(log L)");
        CU(cudaStreamSynchronize(st));
        if (fs) return fs;
    } else {
        NC(nc->broadcast(P->bcast, P->bcast, 4, ncclFloat64, 0, P->comm, st), "ncclBroadcast(log L)");
        CU(cudaMemcpyAsync(hv, P->bcast, 32, cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        if (P->prof) prof_collect(P);
        if (hv[1] == 1.0) return fail(MRA_E_NUMERIC, "Cholesky failed (matrix not positive definite) on some rank");
        if (hv[1] != 0.0) return fail(MRA_E_CUDA, "rank 0 failed to merge the levels above the shard level");
    }
    if (loglik) *loglik = hv[0];
    if (post) {
        post->d = hv[2];
        post->u = hv[3];
        if (post->region_d || post->region_u) {
            // every region once: own subtrees on their rank, the shard level and above on rank 0
            const long long f = lvl_first(P->J, P->c), ns = ipow(P->J, P->c - 1);
            if (P->rank != 0) {
                CU(cudaMemsetAsync(P->dreg, 0, 8 * (f + ns), st));
                CU(cudaMemsetAsync(P->ureg, 0, 8 * (f + ns), st));
            }
            NC(nc->allReduce(P->dreg, P->dreg, (size_t)P->nreg, ncclFloat64, ncclSum, P->comm, st), "ncclAllReduce(d_R)");
            NC(nc->allReduce(P->ureg, P->ureg, (size_t)P->nreg, ncclFloat64, ncclSum, P->comm, st), "ncclAllReduce(u_R)");
            if (post->region_d) CU(cudaMemcpyAsync(post->region_d, P->dreg, 8 * P->nreg, cudaMemcpyDeviceToHost, st));
            if (post->region_u) CU(cudaMemcpyAsync(post->region_u, P->ureg, 8 * P->nreg, cudaMemcpyDeviceToHost, st));
            CU(cudaStreamSynchronize(st));
        }
    }
    if (!want_state) return MRA_OK;
    // above-shard means, and the above-shard merge factors (Ltilde^{-1}, F) that prediction walks through
    const uint64_t nmt = mra_mutop_size(P);
    if (nmt) NC(nc->broadcast(P->mutop, P->mutop, nmt, ncclFloat64, 0, P->comm, st), "ncclBroadcast(mu top)");
    const long long ptop = P->post_base[P->c] - P->post_base[1];
    if (ptop > 0)
        NC(nc->broadcast(P->post + P->post_base[1], P->post + P->post_base[1], (size_t)ptop, ncclFloat64, 0, P->comm, st),
           "ncclBroadcast(top merge factors)");
    if ((s = posterior_local(P, P->mutop, 0.0))) return s;
    // full arrays on every rank: mu by a sum over ranks (rank 0 alone contributes the above-shard levels), the
    // smoothed values through the leaf order (so observations eliminated at knots come back as NaN)
    const long long top = lvl_first(P->J, P->c) * P->rh, nmu = P->nint * P->rh;
    if (P->rank != 0 && top > 0) CU(cudaMemsetAsync(P->mu_d, 0, 8 * top, st));
    if (nmu) NC(nc->allReduce(P->mu_d, P->mu_d, (size_t)nmu, ncclFloat64, ncclSum, P->comm, st), "ncclAllReduce(mu)");
    CU(cudaMemsetAsync(P->sm_sorted, 0, 8 * P->N, st));
    const long long per = ipow(P->J, P->M - P->c);
    for (auto& rg : my_runs(P)) {
        const long long o0 = P->leaf_off[rg.first * per], o1 = P->leaf_off[rg.second * per];
        if (o1 > o0) LCHK(launch_gather(P->smooth_d, P->perm_d + o0, P->sm_sorted + o0, o1 - o0, st));
    }
    NC(nc->allReduce(P->sm_sorted, P->sm_sorted, (size_t)P->N, ncclFloat64, ncclSum, P->comm, st),
       "ncclAllReduce(smoothing)");
    LCHK(launch_fill(P->smooth_d, (long long)P->n_in, NAN, st));
    LCHK(launch_scatter(P->sm_sorted, P->perm_d, P->smooth_d, P->N, st));
    const cudaMemcpyKind k = host_post ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    if (post->mu && nmu) CU(cudaMemcpyAsync(post->mu, P->mu_d, 8 * nmu, k, st));
    if (post->smooth) CU(cudaMemcpyAsync(post->smooth, P->smooth_d, 8 * P->n_in, k, st));
    CU(cudaStreamSynchronize(st));
    P->post_valid = true;
    P->post_theta = *th;
    return MRA_OK;
}

extern "C" mra_status mra_nccl_unique_id(void* id_out) {
    return guarded([&]() -> mra_status {
        g_err.clear();
        if (!id_out) return fail(MRA_E_ARG, "id_out is NULL");
        const NcclApi* nc = nccl_api();
        if (!nc) return fail(MRA_E_NCCL, "no NCCL library could be loaded (libnccl.so.2 / $MRA_NCCL_LIB)");
        ncclUniqueId id;
        NC(nc->getUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(id_out, &id, sizeof id);
        return MRA_OK;
    });
}
