// mra_internal.h -- host-side launch interface between the C-ABI (mra_api.cpp) and the
// sm_100a kernels (mra_kernels.cu). Not part of the public ABI.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace mra {

constexpr int MAXM = 24;

struct CovParams {
    int kind;
    double s2, rho, xs, ys;
};

// Everything a kernel needs to know about the tree and the current theta (passed by value).
struct TreeParams {
    int M, J, lj, rh;           // levels, children, log2 J, r_hat
    CovParams cp;
    double tau2;
    const double* pxy;          // [2N] sorted (by leaf) retained observations, interleaved (x, y)
    const double* zs;           // [N] observed values in sorted order
    const long long* leaf_off;  // [n_leaves + 1]
    const double* kxy;          // [2 * n_interior * rh] knots, level-major regions, interleaved (x, y)
    double* prior;              // chain rows R_R = [Linv_R | -U^{m-1}_R .. -U^1_R], rh x m*rh each
    long long prior_base[MAXM + 1];  // offset (doubles) of level m's first stored region
    long long prior_first[MAXM + 1]; // index (within level m) of that region: 0 when the level is resident,
                                     // the chunk's first region when the plan streams the prior (NEXT-4)
    double* dreg;               // [n_regions] per-region log-det term
    double* ureg;               // [n_regions] per-region quadratic term
    int* err;                   // [4]: flag, level, index lo, index hi
    // posterior-state storage (nullptr unless requested)
    double* post;               // per interior region: Ltilde^{-1} (rh x rh) then F = H^T (q x rh)
    long long post_base[MAXM + 1];
    const double* theta_dev;    // nullptr, or {sigma2, rho, tau2} in device memory (evaluations replayed as graphs)
};

// per-CTA workspace layout of the bottom / smoothing kernels (offsets in doubles)
struct WsLayout {
    long long stride;           // doubles per CTA slot
    long long oG, oS, oD, oA, oF, oL, oV;
    long long oQ, oE, oW;       // prediction: query basis tile, L^{-1} C_M(S, P) tile, chain solve tile
    int ldG, ldS, ldA;
};

// prediction (mra_predict): queries sorted by leaf
struct PredParams {
    const double* qxy;          // [2 nq] interleaved (x, y), leaf-sorted
    const long long* q_off;     // [n_leaves + 1] CSR offsets of each leaf's queries
    const long long* q_perm;    // [nq] sorted position -> caller's query index
    const long long* leaves;    // leaves that hold queries
    long long n_leaves;
    const double* muhat;        // whitened posterior means per interior region (k_mu)
    double* mean;               // [nq] outputs, caller's order
    double* var;
};

// wide (big-leaf) path buffers: G rows indexed by sorted observation, Sigma / inverted diagonal
// blocks / block log-dets per leaf of the current sub-chunk (offsets valid for its leaves)
struct WideParams {
    double* G;                // row of sorted observation o at G + (o - G_base) * ldG
    long long G_base;
    int ldG;
    double* S;
    const long long* S_off;
    const int* S_ld;
    double* D;
    const long long* D_off;   // multiple of 4096; block log-det of (leaf, s) at lblk[D_off/4096 + s]
    double* lblk;
    int kb0, kb1;             // K range [64 kb0, 64 kb1) of the update / substitution tasks of this launch
                              // (super-blocked Cholesky: kb0 = first block of the current super-step)
};

// TMA tensor maps of one evaluation context's long-lived buffers (the leaf rows G, the prior chain rows of each
// level, the merge ring), encoded once on the host and handed to the GEMM unit's kernels BY VALUE as a
// __grid_constant__ parameter: never modified on the device. A GEMM operand that lies inside a registered buffer
// with the buffer's row stride is staged by cp.async.bulk.tensor at (row, column) coordinates of that buffer.
//   kind 0 (row-major operand, MEMN): 2-D (columns = ld, rows), box 16 x 64, 128-byte swizzle
//   kind 1 (transposed operand, MEMT): 3-D (8, rows, ceil(ld / 8)) with strides (ld, 8) doubles, box 8 x 16 x 8
constexpr int TMA_NREG = 32;
struct alignas(64) TmaReg {
    CUtensorMap map[TMA_NREG];
    unsigned long long base[TMA_NREG];
    unsigned long long bytes[TMA_NREG];
    long long ld[TMA_NREG];
    int kind[TMA_NREG];
    int n;
};

// per-group small slots (Li, F) and dependency counters of the level-(M-1) merge tile dataflow
struct MergeRing {
    double* slot;           // ns slots of stride doubles: [A_oo 64x64 | Li rh x rh | F q x rh | -F q x rh]
    long long stride;
    int ns;
    long long maxg;         // groups per launch (counter arrays)
    int* flags;             // [(3 + J) * maxg]: chol_done | f_done | o_done | leaf_done (k_wide_chsig, J * maxg)
    int *chol_done, *f_done, *o_done;
    long long* slot_done;   // [ns] groups that have released the slot
};

// register buffer [base, base + rows * ld) with row stride ld (doubles) under `kind`; false if full or not encodable
bool tma_register(TmaReg& reg, int kind, const double* base, long long ld, long long rows);

// launchers (all asynchronous on `st`); return cudaGetLastError()
cudaError_t launch_gather(const double* z, const long long* perm, double* zs, long long N, cudaStream_t st);
// region ranges: level-m regions [t_first, t_first + t_count); output buffers are indexed by
// (t - out_first), child buffers by (child t - child_first)
cudaError_t launch_prior(const TreeParams& tp, const TmaReg& reg, int m, long long t_first, long long t_count,
                         int grid, double* ws, long long ws_stride, unsigned long long* counter, cudaStream_t st);
cudaError_t launch_bottom(const TreeParams& tp, long long g_first, long long g_count, double* out,
                          long long out_first, int q, int grid, double* ws, const WsLayout& L,
                          unsigned long long* counter, cudaStream_t st);
cudaError_t launch_merge(const TreeParams& tp, const TmaReg& reg, int m, long long t_first, long long t_count,
                         const double* child_out, long long child_first, double* out, long long out_first,
                         int q, int grid, double* ws, long long ws_stride, unsigned long long* counter,
                         cudaStream_t st);
cudaError_t launch_final(const TreeParams& tp, double N, double* d_loglik, cudaStream_t st);
cudaError_t launch_mu(const TreeParams& tp, int m, double* muhat, double* mu, long long t_first, long long t_count,
                      cudaStream_t st);
cudaError_t launch_smooth(const TreeParams& tp, const double* muhat, const long long* perm, double* smooth,
                          int grid, double* ws, const WsLayout& L, unsigned long long* counter, long long l_first,
                          long long l_count, cudaStream_t st);
cudaError_t launch_fill(double* p, long long n, double v, cudaStream_t st);
cudaError_t launch_scatter(const double* zs, const long long* perm, double* z, long long N, cudaStream_t st);
// exchange buffer of subtree sharding (packed lower triangles, d, u, error flag; include/mra.h)
cudaError_t launch_pack_exchange(const double* out, long long ns, int q, const double* d, const double* u,
                                 const int* err, double* xbuf, cudaStream_t st);
cudaError_t launch_unpack_exchange(const double* xbuf, long long ns, int q, double* out, double* d, double* u,
                                   cudaStream_t st);
cudaError_t launch_predict(const TreeParams& tp, const PredParams& pp, int grid, double* ws, const WsLayout& L,
                           unsigned long long* counter, cudaStream_t st);
// wide path: phase 0 chain, 1 sigma, 2 column update (step), 3 diagonal (step), 4 panel + X row (step),
// 5 G = X [V | y]
cudaError_t launch_wide(int phase, const TreeParams& tp, const TmaReg& reg, const WideParams& wp, int step,
                        const int4* tasks, long long ntask, int grid, unsigned long long* counter, cudaStream_t st);
cudaError_t launch_wide_main(int phase, const TreeParams& tp, const WideParams& wp, int step, const int4* tasks,
                        long long ntask, int grid, unsigned long long* counter, cudaStream_t st);
cudaError_t launch_prior_unit(const TreeParams& tp, const TmaReg& reg, int m, long long t_first, long long t_count,
                              int grid, double* ws, long long ws_stride, unsigned long long* counter, cudaStream_t st);
int unit_ctas_per_sm();
void init_kernel_attrs();   // every kernel's smem attribute / occupancy for the current device (before any capture)
void phase_cycles_unit(unsigned long long* out32, bool reset);
int wide_mtile_resident();
cudaError_t launch_wide_chsig(const TreeParams& tp, const TmaReg& reg, const WideParams& wp, const int4* tasks,
                              long long ntask, unsigned long long* counter, int* leaf_done, long long l0,
                              long long nleaf, cudaStream_t st);
cudaError_t launch_wide_mtile(const TreeParams& tp, const TmaReg& reg, const WideParams& wp, long long g_first,
                              long long g_count,
                              double* out, long long out_first, int q, const int4* tasks, long long ntask, int grid,
                              unsigned long long* counter, const MergeRing& ring, cudaStream_t st);
// device plan build (mra_plan.cu): geometry of the partition (host-computed boxes and knot bars)
struct PlanGeom {
    int M, J, nx, ny;
    long long nleaf;
    const double* box;    // [4 n_interior]: x0 x1 y0 y1, level-major
    const double* xbar;   // [n_interior * nx]
    const double* ybar;   // [n_interior * ny]
};
cudaError_t plan_bbox(const double* x, const double* y, long long n, double* part, int nblk, int* bad,
                      cudaStream_t st);
cudaError_t plan_keys(const double* x, const double* y, long long n, const PlanGeom& pg, int* key, int* idx,
                      unsigned int* cnt, cudaStream_t st);
int plan_radix_blocks(long long n);
cudaError_t plan_radix_count(const int* key, long long n, int lj, int d, unsigned int* bcnt, cudaStream_t st);
cudaError_t plan_radix_scatter(const int* key, const int* idx, long long n, int lj, int d, const unsigned int* boff,
                               int* key2, int* idx2, cudaStream_t st);
cudaError_t plan_gather(const double* x, const double* y, const int* idx, long long N, double* pxy, long long* perm,
                        cudaStream_t st);
int smem_bytes();
int resident_ctas_per_sm();   // engine kernels (k_bottom occupancy)
extern thread_local unsigned long long g_kernel_launches;   // host-side count of every kernel this library launched
void phase_cycles(unsigned long long* out32, bool reset);   // -DMRA_PHASE_TIMING builds only

}  // namespace mra
