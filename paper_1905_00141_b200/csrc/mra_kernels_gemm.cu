// mra_kernels_gemm.cu -- the GEMM-only kernels of the wide (grid-wide task) path: leaf V chains,
// Sigma tiles, the Cholesky column updates / panels / X = L^{-1} rows, and G = X [V | y].
//
// They run nothing but 64 x 64 tile GEMMs (no in-smem factorization), so this translation unit builds
// the engine (mra_device.cuh) in its own shape: 4 warps of 32 x 32 per CTA, K stages of 16, two stages,
// four resident CTAs per SM (41 KB smem each: the stages only; 128 registers, no spills). The default
// shape (8 warps, K stages of 32, three stages, two CTAs per SM) is what the factorizing kernels need
// (their 64 x 64 Cholesky + inverse wants 8 warps and 76 KB of smem). Measured per C3 evaluation
// (tools/run_eval.py --prof): chain 667 -> 639 ms, sigma 322 -> 302, solve 322 -> 290, factor 215 -> 202,
// C3 2561 -> 2467 ms; C4 758 -> 681 ms per theta; C2 49.8 -> 48.3 ms. Three CTAs of 4 warps with K
// stages of 32 gained a third of that; five CTAs (96 registers) spill and lose 7 %.
#ifndef MRA_GEMM_NT
#define MRA_GEMM_NT 128
#endif
#ifndef MRA_GEMM_NSTAGE
#define MRA_GEMM_NSTAGE 2
#endif
#ifndef MRA_GEMM_MINB
#define MRA_GEMM_MINB 4
#endif
#ifndef MRA_GEMM_TK
#define MRA_GEMM_TK 16
#endif
#undef MRA_NT
#undef MRA_TK
#undef MRA_NSTAGE
#undef MRA_MINB
#define MRA_NT MRA_GEMM_NT
#define MRA_TK MRA_GEMM_TK
#define MRA_NSTAGE MRA_GEMM_NSTAGE
#define MRA_MINB MRA_GEMM_MINB
#define MRA_FAC_INPLACE 1
#ifndef MRA_NO_BULK
#define MRA_BULK 1   // transposed operands staged by 1-D bulk copies + mbarriers (mra_device.cuh); -DMRA_NO_BULK: cp.async
#endif

#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>

#include "mra_device.cuh"
#include "mra_internal.h"
#include "mra_kcommon.cuh"

namespace mra {

#ifdef MRA_BULK
#define ENGINE_INIT(smem) engine_init(smem, &reg)
// kernels whose GEMM operands never lie in a registered buffer (the per-leaf Sigma / X, the merge workspaces) skip
// the per-call registry lookup
#define ENGINE_INIT_NOREG(smem) ((void)reg, engine_init(smem, nullptr))
#else
#define ENGINE_INIT(smem) ((void)reg)
#define ENGINE_INIT_NOREG(smem) ((void)reg)
#endif
// every kernel of the unit that runs GEMMs takes the context's tensor-map registry by value (param space)
#define TREG const __grid_constant__ TmaReg reg

// V chain for 64 rows of one leaf (covariance blocks in place from k_wide_covfill)
__global__ void __launch_bounds__(NT, MRA_MINB)
k_wide_chain(TreeParams tp, TREG, WideParams wp, const int4* tasks, long long ntask, unsigned long long* counter) {
    double* smem = dyn_smem();
    ENGINE_INIT(smem);
    const CovP cp = covp_of(tp);
    const int m = tp.M - 1;
    for (;;) {
        const long long it = next_item(counter, smem);
        if (it >= ntask) break;
        const int4 tk = tasks[it];
        const long long l = tk.x;
        const long long o0 = tp.leaf_off[l] + 64LL * tk.y;
        const int n = min(64, leaf_n(tp, l) - 64 * tk.y);
        double* Gr = wp.G + (o0 - wp.G_base) * wp.ldG;
        PHASE_MARK(pt0);
        point_chain_pre(tp, m, l >> tp.lj, n, Gr, wp.ldG, cp, smem);
        PHASE_ADD(28, pt0);
#ifdef MRA_PHASE_TIMING
        if (threadIdx.x == 0) atomicAdd(&g_phase_cycles[29], 1ULL);
#endif
    }
}

// Sigma_l tile (i, k), k <= i: C(S_i, S_k) + tau2 delta - V_i V_k^T
__global__ void __launch_bounds__(NT, MRA_MINB)
k_wide_sigma(TreeParams tp, TREG, WideParams wp, const int4* tasks, long long ntask, unsigned long long* counter) {
    double* smem = dyn_smem();
    ENGINE_INIT(smem);
    const CovP cp = covp_of(tp);
    const int Pg = (tp.M - 1) * tp.rh;
    for (;;) {
        const long long it = next_item(counter, smem);
        if (it >= ntask) break;
        const int4 tk = tasks[it];
        const long long l = tk.x;
        const int i = tk.y, k = tk.z, n = leaf_n(tp, l);
        const long long o = tp.leaf_off[l];
        const int ld = wp.S_ld[l];
        double* C = wp.S + wp.S_off[l] + 64LL * i * ld + 64LL * k;
        const double* Gi = wp.G + (o - wp.G_base + 64LL * i) * wp.ldG;
        const double* Gk = wp.G + (o - wp.G_base + 64LL * k) * wp.ldG;
        cta_gemm<MEMN, MEMN, MEMN, MEMN, 1>(min(64, n - 64 * i), min(64, n - 64 * k), i == k, op_mem(Gi, wp.ldG),
                                         op_mem(Gk, wp.ldG), Pg, op_mem(Gi, 0), op_mem(Gi, 0), 0,
                                         ci_cov(tp.pxy + 2 * (o + 64LL * i), tp.pxy + 2 * (o + 64LL * k),
                                                i == k ? tau2_of(tp) : 0.0),
                                         -1.0, C, ld, cp, smem);
    }
}

// chain and Sigma tasks of one sub-chunk as one dataflow (host-ordered list, int4 {leaf, i, k, type}: type 0 the
// V chain of row tile i, type 1 the Sigma tile (i, k)); the host puts a leaf's Sigma tiles `lag` leaves after its
// chain tasks, so they normally run while the leaf's V rows are still in L2 (the phase-separated kernels read them
// back from DRAM: the whole sub-chunk's chain runs first). A Sigma task waits for its leaf's chain tasks, claimed
// earlier by co-resident CTAs (the grid is exactly the resident CTA count), so the waits always terminate.
__global__ void __launch_bounds__(NT, MRA_MINB)
k_wide_chsig(TreeParams tp, TREG, WideParams wp, const int4* tasks, long long ntask, unsigned long long* counter,
             int* leaf_done, long long l0) {
    double* smem = dyn_smem();
    ENGINE_INIT(smem);
    const CovP cp = covp_of(tp);
    const int m = tp.M - 1, Pg = m * tp.rh;
    for (;;) {
        const long long it = next_item(counter, smem);
        if (it >= ntask) break;
        const int4 tk = tasks[it];
        const long long l = tk.x;
        const long long o = tp.leaf_off[l];
        const int nl = leaf_n(tp, l);
        if (tk.w == 0) {
            const int n = min(64, nl - 64 * tk.y);
            double* Gr = wp.G + (o + 64LL * tk.y - wp.G_base) * wp.ldG;
            point_chain_pre(tp, m, l >> tp.lj, n, Gr, wp.ldG, cp, smem);
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                atomicAdd(leaf_done + (l - l0), 1);
            }
        } else {
            if (threadIdx.x == 0) {
                const int T = (nl + 63) / 64;
                while (*(volatile int*)(leaf_done + (l - l0)) < T) __nanosleep(100);
                __threadfence();
            }
            __syncthreads();
            const int i = tk.y, k = tk.z;
            const int ld = wp.S_ld[l];
            double* C = wp.S + wp.S_off[l] + 64LL * i * ld + 64LL * k;
            const double* Gi = wp.G + (o - wp.G_base + 64LL * i) * wp.ldG;
            const double* Gk = wp.G + (o - wp.G_base + 64LL * k) * wp.ldG;
            cta_gemm<MEMN, MEMN, MEMN, MEMN, 1>(min(64, nl - 64 * i), min(64, nl - 64 * k), i == k,
                                                 op_mem(Gi, wp.ldG), op_mem(Gk, wp.ldG), Pg, op_mem(Gi, 0),
                                                 op_mem(Gi, 0), 0,
                                                 ci_cov(tp.pxy + 2 * (o + 64LL * i), tp.pxy + 2 * (o + 64LL * k),
                                                        i == k ? tau2_of(tp) : 0.0),
                                                 -1.0, C, ld, cp, smem);
        }
    }
}

// ---- factorization task bodies of the per-step kernels
// update tile (i, j) of leaf l: A_ij -= A_{i,K} A_{j,K}^T over block columns [k0, k0 + K)
__device__ __forceinline__ void wide_upd_tile(const TreeParams& tp, const WideParams& wp, long long l, int i, int j,
                                              int k0, int K, const CovP& cp, double* smem) {
    const int n = leaf_n(tp, l), ld = wp.S_ld[l];
    double* Sl = wp.S + wp.S_off[l];
    const double* Ai = Sl + 64LL * i * ld + k0;
    double* C = Sl + 64LL * i * ld + 64LL * j;
    const double* Aj = Sl + 64LL * j * ld + k0;
    cta_gemm<MEMN, MEMN, MEMN, MEMN>(min(64, n - 64 * i), min(64, n - 64 * j), i == j, op_mem(Ai, ld), op_mem(Aj, ld),
                                     K, op_mem(Ai, 0), op_mem(Ai, 0), 0, ci_mem(C, ld), -1.0, C, ld, cp, smem);
}

// panel tile of step s: L_is = A_is D_s^T
__device__ __forceinline__ void wide_panel(const TreeParams& tp, const WideParams& wp, long long l, int s, int i,
                                           const CovP& cp, double* smem) {
    const int n = leaf_n(tp, l), ld = wp.S_ld[l], nb = min(64, n - 64 * s);
    double* P = wp.S + wp.S_off[l] + 64LL * i * ld + 64LL * s;
    const double* Ds = wp.D + wp.D_off[l] + 4096LL * s;
    cta_gemm<MEMN, MEMN, MEMN, MEMN>(min(64, n - 64 * i), nb, 0, op_mem(P, ld), op_mem(Ds, 64), nb, op_mem(P, 0),
                                     op_mem(P, 0), 0, ci_zero(), 1.0, P, ld, cp, smem);
}

// block (s, kb), kb < s, of X = L^{-1}: X_sk = -D_s sum_{k<=j<s} L_sj X_jk, stored transposed at S[kb][s]
__device__ __forceinline__ void wide_xrow(const TreeParams& tp, const WideParams& wp, long long l, int s, int kb,
                                          const CovP& cp, double* smem) {
    const int n = leaf_n(tp, l), ld = wp.S_ld[l], nb = min(64, n - 64 * s);
    double* Sl = wp.S + wp.S_off[l];
    const double* Ds = wp.D + wp.D_off[l] + 4096LL * s;
    const long long k0 = 64LL * kb, s0 = 64LL * s;
    const double* Dk = wp.D + wp.D_off[l] + 4096LL * kb;
    double* Yt = Sl + k0 * ld + s0;   // X_sk^T lives here (64 x nb)
    // Y^T = D_k^T L_sk^T + sum_{k<j<s} X_jk^T L_sj^T
    cta_gemm<MEMT, MEMN, MEMN, MEMN>(64, nb, 0, op_mem(Dk, 64), op_mem(Sl + s0 * ld + k0, ld), 64,
                                     op_mem(Sl + k0 * ld + k0 + 64, ld), op_mem(Sl + s0 * ld + k0 + 64, ld),
                                     (int)(s0 - k0 - 64), ci_zero(), 1.0, Yt, ld, cp, smem);
    // X_sk^T = -Y^T D_s^T (in place: one output tile, every operand element is read first)
    cta_gemm<MEMN, MEMN, MEMN, MEMN>(64, nb, 0, op_mem(Yt, ld), op_mem(Ds, 64), nb, op_mem(Yt, 0), op_mem(Yt, 0), 0,
                                     ci_zero(), -1.0, Yt, ld, cp, smem);
}

// Updates of the super-blocked Cholesky (blocks of 64, super-blocks of NB blocks), K range
// [64 kb0, 64 kb1) of the launch:
//   type 0 (leaf, i, j): A_ij -= L_{i,K} L_{j,K}^T   (i >= j; lower when i == j) -- the left-looking update
//          of step j inside a super-block (K = the super-block's columns left of j), or the right-looking
//          trailing update after a super-block (K = its NB columns)
//   type 1 (leaf, i, c): G_i[:, c] -= L_{i,K} G_K[:, c] -- trailing update of the blocked substitution
//          (leaves solved without the explicit inverse)
__global__ void __launch_bounds__(NT, MRA_MINB)
k_wide_update(TreeParams tp, TREG, WideParams wp, int s, const int4* tasks, long long ntask, unsigned long long* counter) {
    double* smem = dyn_smem();
    ENGINE_INIT_NOREG(smem);
    const CovP cp = covp_of(tp);
    const int ncol = (tp.M - 1) * tp.rh + 1;
    const int k0 = 64 * wp.kb0, K = 64 * (wp.kb1 - wp.kb0);
    (void)s;
    for (;;) {
        const long long it = next_item(counter, smem);
        if (it >= ntask) break;
        const int4 tk = tasks[it];
        const long long l = tk.x;
        const int i = tk.y, n = leaf_n(tp, l), ld = wp.S_ld[l];
        double* Sl = wp.S + wp.S_off[l];
        const double* Ai = Sl + 64LL * i * ld + k0;
        if (tk.w == 0) {
            wide_upd_tile(tp, wp, l, i, tk.z, k0, K, cp, smem);
        } else {
            const int c = tk.z;
            const long long o = tp.leaf_off[l];
            double* Gl = wp.G + (o - wp.G_base) * wp.ldG + 64LL * c;
            double* Gi = Gl + 64LL * i * wp.ldG;
            cta_gemm<MEMN, MEMT, MEMN, MEMN>(min(64, n - 64 * i), min(64, ncol - 64 * c), 0, op_mem(Ai, ld),
                                             op_mem(Gl + (long long)k0 * wp.ldG, wp.ldG), K, op_mem(Ai, 0),
                                             op_mem(Ai, 0), 0, ci_mem(Gi, wp.ldG), -1.0, Gi, wp.ldG, cp, smem);
        }
    }
}

// step s, after the diagonal: panel tasks (leaf, i > s, 0): L_is = A_is D_s^T; for small leaves
// (n <= ncol) the tasks of row block s of X = L^{-1} (leaf, k < s, 2): X_sk = -D_s sum_{k<=j<s} L_sj X_jk,
// for large leaves the forward-substitution tasks of row block s (leaf, column tile, 1). X's off-diagonal blocks are
// kept TRANSPOSED in the (otherwise unused) upper triangle of the leaf's Sigma buffer: X[a][b] (block
// a > block b) at S[b * ld + a]; its diagonal blocks are the inverted D_s.
__global__ void __launch_bounds__(NT, MRA_MINB)
k_wide_panel_x(TreeParams tp, TREG, WideParams wp, int s, const int4* tasks, long long ntask, unsigned long long* counter) {
    double* smem = dyn_smem();
    ENGINE_INIT_NOREG(smem);
    const CovP cp = covp_of(tp);
    for (;;) {
        const long long it = next_item(counter, smem);
        if (it >= ntask) break;
        const int4 tk = tasks[it];
        const long long l = tk.x;
        const int n = leaf_n(tp, l), ld = wp.S_ld[l], nb = min(64, n - 64 * s);
        double* Sl = wp.S + wp.S_off[l];
        const double* Ds = wp.D + wp.D_off[l] + 4096LL * s;
        if (tk.z == 0) {
            wide_panel(tp, wp, l, s, tk.y, cp, smem);
        } else if (tk.z == 1) {
            // large leaves (n > ncol): blocked forward substitution G_s[:, c] = D_s (G_s - L_{s,<s} G_{<s})
            // interleaved with the factorization (X = L^{-1} would cost n^3/3 > the solve itself)
            const int c = tk.y, ncol = (tp.M - 1) * tp.rh + 1;
            const long long o = tp.leaf_off[l];
            double* Gs = wp.G + (o - wp.G_base + 64LL * s) * wp.ldG + 64LL * c;
            const int nc = min(64, ncol - 64 * c);
            const int k0 = 64 * wp.kb0;   // earlier super-blocks arrived through trailing updates
            if (s > wp.kb0)
                cta_gemm<MEMN, MEMT, MEMN, MEMN>(nb, nc, 0, op_mem(Sl + 64LL * s * ld + k0, ld),
                                                 op_mem(wp.G + (o - wp.G_base + k0) * wp.ldG + 64LL * c, wp.ldG),
                                                 64 * s - k0, op_mem(Sl, 0), op_mem(Sl, 0), 0, ci_mem(Gs, wp.ldG),
                                                 -1.0, Gs, wp.ldG, cp, smem);
            cta_gemm<MEMN, MEMT, MEMN, MEMN>(nb, nc, 0, op_mem(Ds, 64), op_mem(Gs, wp.ldG), nb, op_mem(Ds, 0),
                                             op_mem(Ds, 0), 0, ci_zero(), 1.0, Gs, wp.ldG, cp, smem);
        } else {
            wide_xrow(tp, wp, l, s, tk.y, cp, smem);
        }
    }
}

// G[:, c] = X [V | y][:, c] per (leaf, 64-column tile), row blocks in DESCENDING order so the product
// can overwrite its input: G_i = [X_{i,<i} | D_i] [B_{<i} ; B_i] only reads rows <= i of B.
__global__ void __launch_bounds__(NT, MRA_MINB)
k_wide_trsm(TreeParams tp, TREG, WideParams wp, const int4* tasks, long long ntask, unsigned long long* counter) {
    double* smem = dyn_smem();
    ENGINE_INIT_NOREG(smem);
    const CovP cp = covp_of(tp);
    const int ncol = (tp.M - 1) * tp.rh + 1;
    for (;;) {
        const long long it = next_item(counter, smem);
        if (it >= ntask) break;
        const int4 tk = tasks[it];
        const long long l = tk.x;
        const int n = leaf_n(tp, l), ld = wp.S_ld[l];
        const double* Sl = wp.S + wp.S_off[l];
        if (tk.z == 2) {
            // the y column alone (ncol = 64 k + 1): g = X y by rows, X[i][K] = Sl[K ld + i] (K < block start)
            // and the inverted diagonal block. y is first staged in shared memory (g_i needs y_k for k <= i only, so
            // the snapshot gives the in-place result); each thread's loads of its X row then run back to back
            // (unrolled; the two accumulators keep their order)
            double* gcol = wp.G + (tp.leaf_off[l] - wp.G_base) * wp.ldG + (ncol - 1);
            double* ys = smem;   // n <= ncol doubles: the GEMM stage area is idle between calls
            for (int i = threadIdx.x; i < n; i += NT) ys[i] = gcol[(long long)i * wp.ldG];
            __syncthreads();
            for (int i = threadIdx.x; i < n; i += NT) {
                const int bi = i / 64, i0 = 64 * bi;
                double s0 = 0.0, s1 = 0.0;
                int k = 0;
#pragma unroll 4
                for (; k + 1 < i0; k += 2) {
                    s0 += Sl[(long long)k * ld + i] * ys[k];
                    s1 += Sl[(long long)(k + 1) * ld + i] * ys[k + 1];
                }
                if (k < i0) s0 += Sl[(long long)k * ld + i] * ys[k];
                const double* Di = wp.D + wp.D_off[l] + 4096LL * bi + (long long)(i - i0) * 64;
#pragma unroll 4
                for (int kk = 0; kk <= i - i0; kk++) s1 += Di[kk] * ys[i0 + kk];
                gcol[(long long)i * wp.ldG] = s0 + s1;
            }
            __syncthreads();   // ys is free for the next task
            continue;
        }
        const int c0 = 64 * tk.y, nc = min(64, ncol - c0);
        double* Gl = wp.G + (tp.leaf_off[l] - wp.G_base) * wp.ldG + c0;
        for (int i = (n - 1) / 64; i >= 0; i--) {
            const int i0 = 64 * i, nb = min(64, n - i0);
            const double* Di = wp.D + wp.D_off[l] + 4096LL * i;
            double* Gi = Gl + (long long)i0 * wp.ldG;
            // G_i = D_i B_i (single tile, in place: every operand element is read before the epilogue), then
            // G_i += X_{i,<i} B_{<i} (both operands transposed: the bulk-copy engine; B_{<i} is still the input,
            // the row blocks run in descending order)
#ifdef MRA_SPLIT_O
            cta_gemm<MEMN, MEMT, MEMN, MEMN>(nb, nc, 0, op_mem(Di, 64), op_mem(Gi, wp.ldG), nb, op_mem(Di, 0),
                                             op_mem(Di, 0), 0, ci_zero(), 1.0, Gi, wp.ldG, cp, smem);
            if (i0 > 0)
                cta_gemm<MEMT, MEMT, MEMN, MEMN>(nb, nc, 0, op_mem(Sl + i0, ld), op_mem(Gl, wp.ldG), i0, op_mem(Gl, 0),
                                                 op_mem(Gl, 0), 0, ci_mem(Gi, wp.ldG), 1.0, Gi, wp.ldG, cp, smem);
#else
            cta_gemm<MEMT, MEMT, MEMN, MEMT>(nb, nc, 0, op_mem(Sl + i0, ld), op_mem(Gl, wp.ldG), i0, op_mem(Di, 64),
                                             op_mem(Gi, wp.ldG), nb, ci_zero(), 1.0, Gi, wp.ldG, cp, smem);
#endif
        }
    }
}

// diagonal block s of leaf l: D_s = L_ss^{-1} (in place; L_ss itself is never read again: panels, X rows,
// substitutions and trsm use D_s), block log-det
__device__ __forceinline__ void wide_diag_blk(const TreeParams& tp, const WideParams& wp, long long l, int s,
                                              double* smem) {
    FacSmem f = fac_smem_inplace(smem);
    if (threadIdx.x == 0) *f.bad = 0;
    const int n = leaf_n(tp, l), ld = wp.S_ld[l], nb = min(64, n - 64 * s);
    double* Sss = wp.S + wp.S_off[l] + 64LL * s * ld + 64LL * s;
    double* Ds = wp.D + wp.D_off[l] + 4096LL * s;
    load_block_lower(f.blk, Sss, ld, nb, 0.0);
    const double ldet = chol_inv_small(f.blk, f.inv, nb, f.diagv, f.bad, f.red, f.tmp);
    if (*f.bad && threadIdx.x == 0) set_err(tp.err, tp.M, l);
    store_block_full(f.inv, Ds, 64, nb);
    if (threadIdx.x == 0) wp.lblk[wp.D_off[l] / 4096 + s] = ldet;
}

// diagonal block of step s for every leaf with more than s blocks: L_ss, D_s = L_ss^{-1}, log-det.
// No GEMM here: the 42 KB factor view and 96 registers let FIVE CTAs share an SM (factor class 180 -> 174 ms
// on C3), one more latency-bound factorization in flight than the GEMM kernels' four
__global__ void __launch_bounds__(NT, 5)
k_wide_diag(TreeParams tp, TREG, WideParams wp, int s, const int4* tasks, long long ntask, unsigned long long* counter) {
    double* smem = dyn_smem();
    ENGINE_INIT_NOREG(smem);
    for (;;) {
        const long long it = next_item(counter, smem);
        if (it >= ntask) break;
        wide_diag_blk(tp, wp, tasks[it].x, s, smem);
    }
}

// Level-(M-1) stacked SYRK and merge as one dataflow of tile tasks (host-ordered list, int4
// {group, type, a, b}). With G = [G_o | G_r] (o = the group region's own rh columns, r = the rest incl.
// the y column; q = |r|):
//   type 0  T00(g):   A_oo = G_o^T G_o, Lt = chol(I + A_oo), Li = Lt^{-1}, log|I + A_oo|, leaf d/u
//   type 1  F(g, a):  F_a = (G_r,a^T G_o) Li^T    (waits for T00(g), which owns the slot once it runs)
//   type 2  O(g,a,b): O_ab = G_r,a^T G_r,b - F_a F_b^T  -> output   (waits for every F(g, .), then ONE
//                     two-segment GEMM with -F kept beside F)
// i.e. Atilde = G^T G and the merge O = A_rr - A_ro (I + A_oo)^{-1} A_or without ever storing A_rr.
// The host staggers the three task kinds (T00 of group s, F of group s - D1, O of group s - D2) so a
// dependency is normally complete when its consumer is claimed; waits spin on counters of tasks
// claimed earlier by co-resident CTAs, so they always terminate. Li and F live in a ring of small
// per-group slots (reused NS groups later, after the group's last O task).
__global__ void __launch_bounds__(NT, MRA_MINB)
k_wide_mtile(TreeParams tp, TREG, WideParams wp, long long g_first, double* out, long long out_first, int q,
             const int4* tasks, long long ntask, unsigned long long* counter, MergeRing ring) {
    double* smem = dyn_smem();
    ENGINE_INIT(smem);
    const CovP cp = covp_of(tp);
    const int M = tp.M, J = tp.J, m = M - 1, rh = tp.rh, Pg = m * rh;
    const int nr = (q + 63) / 64;
    // when the y row is alone in the last 64-row tile (q = 64 k + 1: r_hat = 64), the tile tasks cover
    // rows 0..q-2 only and ONE task per group forms the y row from w = g^T G (a GEMV over the group's G)
    const bool ysep = (q % 64 == 1) && q > 1;
    const int nrF = ysep ? nr - 1 : nr;
    const int nO = nrF * (nrF + 1) / 2 + (ysep ? 1 : 0);
    FacSmem f = fac_smem_inplace(smem);
    double* red = misc_smem(smem);
    const long long leaf_id0 = lvl_first(J, M);
    for (;;) {
        const long long it = next_item(counter, smem);
        if (it >= ntask) break;
        const int4 tk = tasks[it];
        const long long gi = tk.x, g = g_first + gi;
        const int slot = (int)(gi % ring.ns);
        double* Aoo = ring.slot + (long long)slot * ring.stride;
        double* Li = Aoo + 4096;
        double* F = Li + rh * rh;
        double* Fn = F + (long long)q * rh;   // -F, so an O tile is ONE two-segment GEMM
        const long long o = tp.leaf_off[g * J];
        const int ng = (int)(tp.leaf_off[g * J + J] - o);
        const double* G = wp.G + (o - wp.G_base) * wp.ldG;
        const long long id = lvl_first(J, m) + g;
        PHASE_MARK(ph0);
        if (tk.y == 0) {
            if (gi >= ring.ns) {   // the group NS earlier must have released the slot
                if (threadIdx.x == 0) {
                    while (*(volatile long long*)(ring.slot_done + slot) < gi / ring.ns) __nanosleep(100);
                    __threadfence();
                }
                __syncthreads();
            }
            if (threadIdx.x == 0) *f.bad = 0;
            double dsum = 0.0;
            for (int c = 0; c < J; c++) {
                const long long l = g * J + c;
                const long long ol = tp.leaf_off[l];
                const int n = leaf_n(tp, l);
                double u = 0.0;
                for (int i = threadIdx.x; i < n; i += NT) {
                    const double gv = wp.G[(ol - wp.G_base + i) * wp.ldG + Pg];
                    u += gv * gv;
                }
                u = cta_sum(u, red);
                if (threadIdx.x == 0) {
                    double d = 0.0;
                    for (int bb = 0; bb < (n + 63) / 64; bb++) d += wp.lblk[wp.D_off[l] / 4096 + bb];
                    tp.dreg[leaf_id0 + l] = d;
                    tp.ureg[leaf_id0 + l] = u;
                    red[9] = d;
                }
                __syncthreads();
                dsum += red[9];
                __syncthreads();
            }
            cta_gemm<MEMT, MEMT, MEMN, MEMN>(rh, rh, 1, op_mem(G, wp.ldG), op_mem(G, wp.ldG), ng, op_mem(G, 0),
                                             op_mem(G, 0), 0, ci_zero(), 1.0, Aoo, 64, cp, smem);
            load_block_lower(f.blk, Aoo, 64, rh, 1.0);
            const double ldm = chol_inv_small(f.blk, f.inv, rh, f.diagv, f.bad, f.red, f.tmp);
            if (*f.bad && threadIdx.x == 0) set_err(tp.err, m, g);
            store_block_full(f.inv, Li, rh, rh);
            if (tp.post) {
                double* P = tp.post + tp.post_base[m] + g * ((long long)rh * rh + (long long)q * rh);
                for (int e = threadIdx.x; e < rh * rh; e += NT) P[e] = f.inv[(e / rh) * LDB + (e % rh)];
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                tp.dreg[id] = dsum + ldm;
                __threadfence();
                atomicExch(ring.chol_done + gi, 1);
            }
            PHASE_ADD(16, ph0);
#ifdef MRA_PHASE_TIMING
            if (threadIdx.x == 0) atomicAdd(&g_phase_cycles[17], 1ULL);
#endif
        } else if (tk.y == 1) {
            const int a = tk.z, r0 = 64 * a, nrow = min(64, q - r0);
            double* Fa = F + (long long)r0 * rh;
            // the slot is this group's only after T00 has waited for it (chol_done is set after that)
            if (threadIdx.x == 0) {
                while (*(volatile int*)(ring.chol_done + gi) == 0) __nanosleep(100);
                __threadfence();
            }
            __syncthreads();
            PHASE_ADD(19, ph0);
            PHASE_MARK(ph1);
            cta_gemm<MEMT, MEMT, MEMN, MEMN>(nrow, rh, 0, op_mem(G + rh + r0, wp.ldG), op_mem(G, wp.ldG), ng,
                                             op_mem(G, 0), op_mem(G, 0), 0, ci_zero(), 1.0, Fa, rh, cp, smem);
            PHASE_ADD(18, ph1);
            PHASE_MARK(ph2);
            cta_gemm<MEMN, MEMN, MEMN, MEMN>(nrow, rh, 0, op_mem(Fa, rh), op_mem(Li, rh), rh, op_mem(Fa, 0),
                                             op_mem(Fa, 0), 0, ci_zero(), 1.0, Fa, rh, cp, smem);
            {
                double* Fna = Fn + (long long)r0 * rh;
                double* P = tp.post ? tp.post + tp.post_base[m] + g * ((long long)rh * rh + (long long)q * rh) +
                                          rh * rh + (long long)r0 * rh
                                    : nullptr;
                // all loads first (Fa / Fna / P may alias as far as the compiler knows: interleaved
                // load-store pairs would serialise on the L2 latency)
                constexpr int NU = 4096 / NT;   // nrow * rh <= 64 * 64
                double v[NU];
#pragma unroll
                for (int u = 0; u < NU; u++) {
                    const int e = threadIdx.x + u * NT;
                    v[u] = (e < nrow * rh) ? __ldcg(Fa + e) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < NU; u++) {
                    const int e = threadIdx.x + u * NT;
                    if (e < nrow * rh) {
                        Fna[e] = -v[u];
                        if (P) P[e] = v[u];
                    }
                }
            }
            __syncthreads();
            PHASE_ADD(20, ph2);
#ifdef MRA_PHASE_TIMING
            if (threadIdx.x == 0) atomicAdd(&g_phase_cycles[21], 1ULL);
#endif
            if (threadIdx.x == 0) {
                __threadfence();
                atomicAdd(ring.f_done + gi, 1);
            }
        } else if (tk.y == 3) {
            // y row: w = g^T [G_o | G_r] (g = G's last column), F_y = w_o Li^T, O[y, :] = w_r - F_y F^T
            if (threadIdx.x == 0) {
                while (*(volatile int*)(ring.f_done + gi) < nrF) __nanosleep(100);
                __threadfence();
            }
            __syncthreads();
            const int ncg = Pg + 1, np2 = (ncg + 1) / 2;            // columns of G, column pairs
            const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
            constexpr int MAXP = 12, CH = 2 * 32 * MAXP;            // column pairs per lane, columns per chunk
            double* w = smem;                                        // [2 np2]
            double* fy = w + 2 * np2;                                // [rh]
            double* part = fy + 64;                                  // [NT / 32][CH] per-warp partial sums
            for (int cb = 0; cb < np2; cb += 32 * MAXP) {
                double2 acc2[MAXP];
#pragma unroll
                for (int u = 0; u < MAXP; u++) acc2[u] = make_double2(0.0, 0.0);
                for (int r = warp; r < ng; r += NT / 32) {   // warp-strided rows, coalesced 16-byte loads
                    const double* Gr = G + (long long)r * wp.ldG;
                    const double gr = Gr[Pg];
#pragma unroll
                    for (int u = 0; u < MAXP; u++) {
                        const int c2 = cb + lane + 32 * u;
                        if (c2 < np2) {
                            const double2 v = *reinterpret_cast<const double2*>(Gr + 2 * c2);
                            acc2[u].x += gr * v.x;
                            acc2[u].y += gr * v.y;
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < MAXP; u++) {
                    part[warp * CH + 2 * (lane + 32 * u)] = acc2[u].x;
                    part[warp * CH + 2 * (lane + 32 * u) + 1] = acc2[u].y;
                }
                __syncthreads();
                for (int c = threadIdx.x; c < CH && 2 * cb + c < 2 * np2; c += NT) {
                    double v = 0.0;
                    for (int ww = 0; ww < NT / 32; ww++) v += part[ww * CH + c];
                    w[2 * cb + c] = v;
                }
                __syncthreads();
            }
            for (int c = threadIdx.x; c < rh; c += NT) {
                double v = 0.0;
                for (int k = 0; k < rh; k++) v += w[k] * Li[c * rh + k];
                fy[c] = v;
            }
            __syncthreads();
            double* Fy = F + (long long)(q - 1) * rh;
            double* Fny = Fn + (long long)(q - 1) * rh;
            double* Py = tp.post ? tp.post + tp.post_base[m] + g * ((long long)rh * rh + (long long)q * rh) + rh * rh +
                                       (long long)(q - 1) * rh
                                 : nullptr;
            for (int c = threadIdx.x; c < rh; c += NT) {
                Fy[c] = fy[c];
                Fny[c] = -fy[c];
                if (Py) Py[c] = fy[c];
            }
            double* Oy = out + (g - out_first) * (long long)q * q + (long long)(q - 1) * q;
            for (int b = threadIdx.x; b < q; b += NT) {
                const double* Fb = (b == q - 1) ? fy : F + (long long)b * rh;
                double v = w[rh + b];
                for (int c = 0; c < rh; c++) v -= fy[c] * Fb[c];
                Oy[b] = v;
                if (b == q - 1) tp.ureg[id] = v;
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                if (atomicAdd(ring.o_done + gi, 1) == nO - 1) {
                    __threadfence();
                    atomicAdd((unsigned long long*)(ring.slot_done + slot), 1ULL);
                }
            }
        } else {
            const int a = tk.z, b = tk.w, r0 = 64 * a, c0 = 64 * b;
            const int nrow = min(64, q - r0), ncl = min(64, q - c0);
            double* Oab = out + (g - out_first) * (long long)q * q + (long long)r0 * q + c0;
            // every F of the group is final (the host schedules O tasks ~6 steps after the F tasks)
            if (threadIdx.x == 0) {
                while (*(volatile int*)(ring.f_done + gi) < nrF) __nanosleep(100);
                __threadfence();
            }
            __syncthreads();
            PHASE_ADD(23, ph0);
            PHASE_MARK(ph2);
            // O_ab = G_r,a^T G_r,b + (-F_a) F_b^T: the transposed-operand product (K = n_group) on the bulk-copy
            // engine, then the K = rh correction on cp.async, in place (each element re-read by the thread that
            // wrote it)
#ifdef MRA_SPLIT_O
            cta_gemm<MEMT, MEMT, MEMN, MEMN>(nrow, ncl, a == b, op_mem(G + rh + r0, wp.ldG),
                                             op_mem(G + rh + c0, wp.ldG), ng, op_mem(G, 0), op_mem(G, 0), 0,
                                             ci_zero(), 1.0, Oab, q, cp, smem);
            cta_gemm<MEMN, MEMN, MEMN, MEMN>(nrow, ncl, a == b, op_mem(Fn + (long long)r0 * rh, rh),
                                             op_mem(F + (long long)c0 * rh, rh), rh, op_mem(F, 0), op_mem(F, 0), 0,
                                             ci_mem(Oab, q), 1.0, Oab, q, cp, smem);
#else
            // diagonal tiles (a == b, lower) of long-K groups through the EPI = 2 instantiation: the balanced warp map
            // and the skipped 8 x 8 blocks above the diagonal (its own function, so the off-diagonal tiles' code is
            // unchanged). Measured: C3 (K = 720 + 64) merge tiles 579 -> 553 ms; C2 (K = 256 + 64) 10.9 -> 12.3 ms,
            // hence the K threshold
#ifndef MRA_BAL_MINK
#define MRA_BAL_MINK 512
#endif
            if (a == b && ng >= MRA_BAL_MINK)
                cta_gemm<MEMT, MEMT, MEMN, MEMN, 2>(nrow, ncl, 1, op_mem(G + rh + r0, wp.ldG),
                                                    op_mem(G + rh + c0, wp.ldG), ng, op_mem(Fn + (long long)r0 * rh, rh),
                                                    op_mem(F + (long long)c0 * rh, rh), rh, ci_zero(), 1.0, Oab, q, cp,
                                                    smem);
            else
                cta_gemm<MEMT, MEMT, MEMN, MEMN>(nrow, ncl, a == b, op_mem(G + rh + r0, wp.ldG),
                                                 op_mem(G + rh + c0, wp.ldG), ng, op_mem(Fn + (long long)r0 * rh, rh),
                                                 op_mem(F + (long long)c0 * rh, rh), rh, ci_zero(), 1.0, Oab, q, cp,
                                                 smem);
#endif
            PHASE_ADD(24, ph2);
#ifdef MRA_PHASE_TIMING
            if (threadIdx.x == 0) atomicAdd(&g_phase_cycles[25], 1ULL);
            if (a == nr - 1 && threadIdx.x == 0) {
                atomicAdd(&g_phase_cycles[30], (unsigned long long)(clock64() - ph2));
                atomicAdd(&g_phase_cycles[31], 1ULL);
            }
#endif
            if (threadIdx.x == 0) {
                if (a == nr - 1 && b == nr - 1) tp.ureg[id] = Oab[(long long)(nrow - 1) * q + ncl - 1];
                __threadfence();
                if (atomicAdd(ring.o_done + gi, 1) == nO - 1) {
                    __threadfence();
                    atomicAdd((unsigned long long*)(ring.slot_done + slot), 1ULL);
                }
            }
        }
    }
}

__global__ void __launch_bounds__(NT, MRA_MINB)
k_prior(TreeParams tp, TREG, int m, long long t_first, long long nitems, double* ws, long long ws_stride,
        unsigned long long* counter) {
    double* smem = dyn_smem();
    ENGINE_INIT(smem);
    const CovP cp = covp_of(tp);
    const int rh = tp.rh;
    double* W = ws + (long long)blockIdx.x * ws_stride;
    FacSmem f = fac_view(smem);
    const long long ldR = (long long)m * rh;
    for (;;) {
        const long long it = next_item(counter, smem);
        if (it >= nitems) break;
        if (threadIdx.x == 0) *f.bad = 0;
        const long long t = t_first + it;
        double* R = tp.prior + tp.prior_base[m] + (t - tp.prior_first[m]) * ldR * rh;
        // V^k_R for k < m over R's blocks m-k, which hold C(Q_R, Q_{a_k}) (k_prior_covfill); they become -U
        // after the inverse is known
        point_chain_pre(tp, m - 1, t >> tp.lj, rh, R + rh, ldR, cp, smem);
        // W^m_R = C(Q_R, Q_R) - sum_k V^k V^kT   (C(Q_R, Q_R) in R's block 0)
        cta_gemm<MEMN, MEMN, MEMN, MEMN>(rh, rh, 1, op_mem(R + rh, ldR), op_mem(R + rh, ldR), (m - 1) * rh,
                                         op_mem(R, ldR), op_mem(R, ldR), 0, ci_mem(R, ldR), -1.0, W, rh, cp,
                                         smem);
        load_block_lower(f.blk, W, rh, rh, 0.0);
        chol_inv_small(f.blk, f.inv, rh, f.diagv, f.bad, f.red, f.tmp);
        if (*f.bad && threadIdx.x == 0) set_err(tp.err, m, t);
        store_block_full(f.inv, R, ldR, rh);
        __syncthreads();
        // -U = -L^{-1} V  (in place over the V blocks; single row tile)
        if (m > 1)
            cta_gemm<MEMN, MEMT, MEMN, MEMN>(rh, (m - 1) * rh, 0, op_mem(R, ldR), op_mem(R + rh, ldR), rh,
                                             op_mem(R, ldR), op_mem(R, ldR), 0, ci_zero(), -1.0, R + rh, ldR, cp,
                                             smem);
    }
}

// --------------------------------------------------------------------------- merge
__global__ void __launch_bounds__(NT, MRA_MINB)
k_merge(TreeParams tp, TREG, int m, long long t_first, long long t_count, const double* child_out, long long child_first,
        double* out, long long out_first, int q, double* ws, long long ws_stride, unsigned long long* counter,
        int presummed) {
    double* smem = dyn_smem();
    ENGINE_INIT_NOREG(smem);
    const CovP cp = covp_of(tp);
    const int J = tp.J, rh = tp.rh;
    const int qc = m * rh + 1;
    const int ldA = qc + (qc & 1);   // even leading dimension -> 16-byte cp.async rows
    double* Aws = ws + (long long)blockIdx.x * ws_stride;
    double* F = Aws + (long long)qc * ldA;
    double* Li = F + (long long)q * rh;
    FacSmem f = fac_view(smem);
    const long long qc2 = (long long)qc * qc;
    for (;;) {
        const long long it = next_item(counter, smem);
        if (it >= t_count) break;
        if (threadIdx.x == 0) *f.bad = 0;
        const long long t = t_first + it;
        const double* C0 = child_out + (t * J - child_first) * qc2;
        // presummed: k_merge_sum has already accumulated Atilde into the first child's block (ld qc)
        const double* A = presummed ? C0 : Aws;
        const long long lda = presummed ? qc : ldA;
        if (!presummed)
        // Atilde = sum of the J children (lower triangle): one warp per row, lanes along the row, U column
        // groups per pass so every lane has U*J independent streaming loads in flight (the children's
        // outputs are read exactly once: evict-first)
        {
            constexpr int U = 4;
            const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
            for (int i = warp; i < qc; i += NT / 32) {
                const double* ci = C0 + (long long)i * qc;
                double* Ai = Aws + (long long)i * ldA;
                for (int j0 = 0; j0 <= i; j0 += 32 * U) {
                    double v[U];
#pragma unroll
                    for (int u = 0; u < U; u++) {
                        const int j = j0 + lane + 32 * u;
                        double sacc = 0.0;
                        if (j <= i) {
                            const double* p = ci + j;
                            if (J == 4) {
                                const double a0 = __ldcs(p), a1 = __ldcs(p + qc2), a2 = __ldcs(p + 2 * qc2),
                                             a3 = __ldcs(p + 3 * qc2);
                                sacc = (((sacc + a0) + a1) + a2) + a3;
                            } else {
                                for (int c = 0; c < J; c++) sacc += __ldcs(p + c * qc2);
                            }
                        }
                        v[u] = sacc;
                    }
#pragma unroll
                    for (int u = 0; u < U; u++) {
                        const int j = j0 + lane + 32 * u;
                        if (j <= i) Ai[j] = v[u];
                    }
                }
            }
        }
        __syncthreads();
        double* O = out + (t - out_first) * (long long)q * q;
        const double ldm = merge_core(A, rh, lda, O, q, F, Li, tp.err, m, t, cp, smem);
        const long long id = lvl_first(J, m) + t;
        if (threadIdx.x == 0) {
            const long long c0 = lvl_first(J, m + 1) + t * J;
            double ds = 0.0;
            for (int c = 0; c < J; c++) ds += tp.dreg[c0 + c];
            tp.dreg[id] = ds + ldm;
            tp.ureg[id] = O[(long long)(q - 1) * q + q - 1];
        }
        save_post(tp, m, t, q, Li, F);
    }
}

// Atilde of every level-m region of [t_first, t_first + t_count), accumulated IN PLACE into its first child's
// output block (lower triangle, ld qc): a grid-wide streaming pass (one warp per row, U column groups per
// lane, J evict-first loads each) for the large levels, where the per-region sum inside k_merge left HBM idle
// while the CTA factored and multiplied. The children's outputs have no other consumer.
__global__ void __launch_bounds__(256)
k_merge_sum(int J, int qc, long long t_first, long long t_count, double* child_out, long long child_first) {
    constexpr int U = 4;
    const long long qc2 = (long long)qc * qc, rows = t_count * qc;
    const int lane = threadIdx.x & 31;
    const long long w0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long r = w0; r < rows; r += nw) {
        const long long t = t_first + r / qc;
        const int i = (int)(r % qc);
        double* c0 = child_out + (t * J - child_first) * qc2 + (long long)i * qc;
        for (int j0 = 0; j0 <= i; j0 += 32 * U) {
            double v[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int j = j0 + lane + 32 * u;
                double sacc = 0.0;
                if (j <= i) {
                    const double* p = c0 + j;
                    if (J == 4) {
                        const double a0 = __ldcs(p), a1 = __ldcs(p + qc2), a2 = __ldcs(p + 2 * qc2), a3 = __ldcs(p + 3 * qc2);
                        sacc = (((sacc + a0) + a1) + a2) + a3;
                    } else {
                        for (int c = 0; c < J; c++) sacc += __ldcs(p + c * qc2);
                    }
                }
                v[u] = sacc;
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int j = j0 + lane + 32 * u;
                if (j <= i) c0[j] = v[u];
            }
        }
    }
}

// resident CTAs per SM x SM count, by phase (6: mtile, 7: prior, 8: merge), per device ordinal (the smem
// attribute and occupancy are per device; computed once per device under a lock)
constexpr int MAXDEV = 64;
struct GemmAttrs {
    bool done = false;
    int resident[10] = {1, 1, 1, 1, 1, 1, 1, 1, 1, 1};
    int nsm = 148;
};
static GemmAttrs g_gemm_attrs[MAXDEV];
static std::mutex g_gemm_mu;
// the stages, or the in-place 64 x 64 factor view (diag, T00 of mtile) if larger, plus the misc area
constexpr int UNIT_SMEM_DBL = (FAC_IN_DBL > NSTAGE * STAGE_DBL ? FAC_IN_DBL : NSTAGE * STAGE_DBL) + MISC_DBL;
static int gemm_smem_bytes() { return UNIT_SMEM_DBL * (int)sizeof(double); }
static const GemmAttrs& gemm_set_attrs() {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= MAXDEV) dev = 0;
    GemmAttrs& A = g_gemm_attrs[dev];
    std::lock_guard<std::mutex> lk(g_gemm_mu);
    if (A.done) return A;
    const int b = gemm_smem_bytes();
    const void* ks[10] = {(const void*)k_wide_chain,   (const void*)k_wide_sigma, (const void*)k_wide_update,
                          (const void*)k_wide_diag,    (const void*)k_wide_panel_x, (const void*)k_wide_trsm,
                          (const void*)k_wide_mtile,   (const void*)k_prior,      (const void*)k_merge,
                          (const void*)k_wide_chsig};
    cudaDeviceGetAttribute(&A.nsm, cudaDevAttrMultiProcessorCount, dev);
    for (int i = 0; i < 10; i++) {
        cudaFuncSetAttribute(ks[i], cudaFuncAttributeMaxDynamicSharedMemorySize, b);
        int per = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, ks[i], NT, b);
        A.resident[i] = (per > 0 ? per : 1) * A.nsm;
    }
    A.done = true;
    return A;
}

// phases: 0 chain, 1 sigma, 2 update, 3 diag, 4 panel_x, 5 trsm, 6 covfill (6: mra_kernels.cu).
// `grid` is ignored for this unit's phases: a persistent grid of every resident CTA pulls the tasks.
cudaError_t launch_wide(int phase, const TreeParams& tp, const TmaReg& reg, const WideParams& wp, int step,
                        const int4* tasks, long long ntask, int grid, unsigned long long* counter, cudaStream_t st) {
    if (phase == 6) return launch_wide_main(phase, tp, wp, step, tasks, ntask, grid, counter, st);
    if (phase < 0 || phase > 6) return cudaErrorInvalidValue;
    long long g = gemm_set_attrs().resident[phase];
    if (ntask < g) g = ntask;
    if (g < 1) return cudaSuccess;
    const int b = gemm_smem_bytes();
    switch (phase) {
        case 0: ++g_kernel_launches; k_wide_chain<<<(int)g, NT, b, st>>>(tp, reg, wp, tasks, ntask, counter); break;
        case 1: ++g_kernel_launches; k_wide_sigma<<<(int)g, NT, b, st>>>(tp, reg, wp, tasks, ntask, counter); break;
        case 2: ++g_kernel_launches; k_wide_update<<<(int)g, NT, b, st>>>(tp, reg, wp, step, tasks, ntask, counter); break;
        case 3: ++g_kernel_launches; k_wide_diag<<<(int)g, NT, b, st>>>(tp, reg, wp, step, tasks, ntask, counter); break;
        case 4: ++g_kernel_launches; k_wide_panel_x<<<(int)g, NT, b, st>>>(tp, reg, wp, step, tasks, ntask, counter); break;
        case 5: ++g_kernel_launches; k_wide_trsm<<<(int)g, NT, b, st>>>(tp, reg, wp, tasks, ntask, counter); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// chain + Sigma dataflow of one sub-chunk (k_wide_chsig): leaf_done[nleaf] counters zeroed here; the grid is the
// resident CTA count (Sigma tasks wait on chain tasks claimed earlier by co-resident CTAs)
cudaError_t launch_wide_chsig(const TreeParams& tp, const TmaReg& reg, const WideParams& wp, const int4* tasks,
                              long long ntask, unsigned long long* counter, int* leaf_done, long long l0,
                              long long nleaf, cudaStream_t st) {
    long long g = gemm_set_attrs().resident[9];
    if (ntask < g) g = ntask;
    if (g < 1) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(leaf_done, 0, sizeof(int) * nleaf, st);
    if (e != cudaSuccess) return e;
    ++g_kernel_launches;
    k_wide_chsig<<<(int)g, NT, gemm_smem_bytes(), st>>>(tp, reg, wp, tasks, ntask, counter, leaf_done, l0);
    return cudaGetLastError();
}

// the level-(M-1) merge tile dataflow: every CTA of the grid must be resident (consumers spin on tasks
// claimed earlier by co-resident CTAs), so the grid is exactly the resident CTA count
cudaError_t launch_wide_mtile(const TreeParams& tp, const TmaReg& reg, const WideParams& wp, long long g_first,
                              long long g_count,
                              double* out, long long out_first, int q, const int4* tasks, long long ntask, int grid,
                              unsigned long long* counter, const MergeRing& ring, cudaStream_t st) {
    (void)grid;
    (void)g_count;
    long long gr = gemm_set_attrs().resident[6];
    if (ntask < gr) gr = ntask;
    if (gr < 1) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(ring.flags, 0, sizeof(int) * 3 * ring.maxg, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(ring.slot_done, 0, sizeof(long long) * ring.ns, st);
    if (e != cudaSuccess) return e;
    ++g_kernel_launches;
    k_wide_mtile<<<(int)gr, NT, gemm_smem_bytes(), st>>>(tp, reg, wp, g_first, out, out_first, q, tasks, ntask, counter,
                                                        ring);
    return cudaGetLastError();
}

cudaError_t launch_merge(const TreeParams& tp, const TmaReg& reg, int m, long long t_first, long long t_count, const double* child_out,
                         long long child_first, double* out, long long out_first, int q, int grid, double* ws,
                         long long ws_stride, unsigned long long* counter, cudaStream_t st) {
    const GemmAttrs& A = gemm_set_attrs();
    grid = (int)std::min<long long>({(long long)grid, (long long)A.resident[8], t_count});
    if (grid < 1) return cudaSuccess;
    // large levels (several regions per CTA): the child sums as one streaming pass first
    const int presummed = t_count >= 4LL * grid ? 1 : 0;
    if (presummed) {
        const int nsm = A.nsm;
        const int qc = m * tp.rh + 1;
        const long long rows = t_count * qc;
        const int sg = (int)std::min<long long>((rows + 7) / 8, 8LL * nsm);
        ++g_kernel_launches;
        k_merge_sum<<<sg, 256, 0, st>>>(tp.J, qc, t_first, t_count, const_cast<double*>(child_out), child_first);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    ++g_kernel_launches;
    k_merge<<<grid, NT, gemm_smem_bytes(), st>>>(tp, reg, m, t_first, t_count, child_out, child_first, out, out_first, q, ws,
                                           ws_stride, counter, presummed);
    return cudaGetLastError();
}

// k_prior of one level (the covariance blocks are filled first by launch_prior in mra_kernels.cu)
cudaError_t launch_prior_unit(const TreeParams& tp, const TmaReg& reg, int m, long long t_first, long long t_count,
                              int grid, double* ws, long long ws_stride, unsigned long long* counter, cudaStream_t st) {
    grid = (int)std::min<long long>({(long long)grid, (long long)gemm_set_attrs().resident[7], t_count});
    if (grid < 1) return cudaSuccess;
    ++g_kernel_launches;
    k_prior<<<grid, NT, gemm_smem_bytes(), st>>>(tp, reg, m, t_first, t_count, ws, ws_stride, counter);
    return cudaGetLastError();
}

// resident CTAs per SM of this unit's kernels (the plan sizes its per-CTA workspace slots with it)
int unit_ctas_per_sm() {
    const GemmAttrs& A = gemm_set_attrs();
    return std::max(1, A.resident[8] / A.nsm);
}

// -DMRA_PHASE_TIMING diagnostics of this unit's kernels (g_phase_cycles is per translation unit)
void phase_cycles_unit(unsigned long long* out32, bool reset) {
    cudaMemcpyFromSymbol(out32, g_phase_cycles, sizeof(unsigned long long) * 32);
    if (reset) {
        unsigned long long z[32] = {0};
        cudaMemcpyToSymbol(g_phase_cycles, z, sizeof z);
    }
}

// Host encoding of a registry entry (cuTensorMapEncodeTiled through the runtime's driver entry point, so the
// library has no link-time dependency on libcuda). MEMN: 2-D (ld columns, rows), row stride ld, box (16, 64),
// 128-byte swizzle; MEMT: 3-D (8, rows, ceil(ld / 8)), strides (ld, 8) doubles, box (8, 16, 8), no swizzle.
bool tma_register(TmaReg& reg, int kind, const double* base, long long ld, long long rows) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    });
    if (!encode || reg.n >= TMA_NREG || !base || ld <= 0 || (ld & 1) || rows <= 0 ||
        (reinterpret_cast<uintptr_t>(base) & 15))
        return false;
    CUtensorMap* m = &reg.map[reg.n];
    CUresult r;
    if (kind == 0) {
        cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
        cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
        cuuint32_t box[2] = {16, 64};
        cuuint32_t es[2] = {1, 1};
        r = encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
        cuuint64_t dims[3] = {8, (cuuint64_t)rows, (cuuint64_t)((ld + 7) / 8)};
        cuuint64_t strides[2] = {(cuuint64_t)ld * 8, 64};
        cuuint32_t box[3] = {8, 16, 8};
        cuuint32_t es[3] = {1, 1, 1};
        r = encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_64B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r != CUDA_SUCCESS) return false;
    reg.base[reg.n] = reinterpret_cast<unsigned long long>(base);
    reg.bytes[reg.n] = (unsigned long long)(ld * rows * 8);
    reg.ld[reg.n] = ld;
    reg.kind[reg.n] = kind;
    reg.n++;
    return true;
}

void init_kernel_attrs_main();   // mra_kernels.cu
void init_kernel_attrs() {
    gemm_set_attrs();
    init_kernel_attrs_main();
}

// resident CTAs of the merge tile dataflow (the host sizes its look-ahead D1 with it)
int wide_mtile_resident() {
    return gemm_set_attrs().resident[6];
}

}  // namespace mra
