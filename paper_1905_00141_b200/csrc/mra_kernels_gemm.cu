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

#include <cuda_runtime.h>

#include <algorithm>

#include "mra_device.cuh"
#include "mra_internal.h"
#include "mra_kcommon.cuh"

namespace mra {

// V chain for 64 rows of one leaf (covariance blocks in place from k_wide_covfill)
__global__ void __launch_bounds__(NT, MRA_MINB)
k_wide_chain(TreeParams tp, WideParams wp, const int4* tasks, long long ntask, unsigned long long* counter) {
    double* smem = dyn_smem();
    const CovP cp = to_covp(tp.cp);
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
k_wide_sigma(TreeParams tp, WideParams wp, const int4* tasks, long long ntask, unsigned long long* counter) {
    double* smem = dyn_smem();
    const CovP cp = to_covp(tp.cp);
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
        cta_gemm<MEMN, MEMN, MEMN, MEMN>(min(64, n - 64 * i), min(64, n - 64 * k), i == k, op_mem(Gi, wp.ldG),
                                         op_mem(Gk, wp.ldG), Pg, op_mem(Gi, 0), op_mem(Gi, 0), 0,
                                         ci_cov(tp.pxy + 2 * (o + 64LL * i), tp.pxy + 2 * (o + 64LL * k),
                                                i == k ? tp.tau2 : 0.0),
                                         -1.0, C, ld, cp, smem);
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
k_wide_update(TreeParams tp, WideParams wp, int s, const int4* tasks, long long ntask, unsigned long long* counter) {
    double* smem = dyn_smem();
    const CovP cp = to_covp(tp.cp);
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
k_wide_panel_x(TreeParams tp, WideParams wp, int s, const int4* tasks, long long ntask, unsigned long long* counter) {
    double* smem = dyn_smem();
    const CovP cp = to_covp(tp.cp);
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
k_wide_trsm(TreeParams tp, WideParams wp, const int4* tasks, long long ntask, unsigned long long* counter) {
    double* smem = dyn_smem();
    const CovP cp = to_covp(tp.cp);
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
            // and the inverted diagonal block; row chunks descending so g can overwrite y in place
            double* gcol = wp.G + (tp.leaf_off[l] - wp.G_base) * wp.ldG + (ncol - 1);
            for (int base = ((n - 1) / NT) * NT; base >= 0; base -= NT) {
                const int i = base + threadIdx.x;
                double v = 0.0;
                if (i < n) {
                    const int bi = i / 64, i0 = 64 * bi;
                    double s0 = 0.0, s1 = 0.0;
                    int k = 0;
                    for (; k + 1 < i0; k += 2) {
                        s0 += Sl[(long long)k * ld + i] * gcol[(long long)k * wp.ldG];
                        s1 += Sl[(long long)(k + 1) * ld + i] * gcol[(long long)(k + 1) * wp.ldG];
                    }
                    if (k < i0) s0 += Sl[(long long)k * ld + i] * gcol[(long long)k * wp.ldG];
                    const double* Di = wp.D + wp.D_off[l] + 4096LL * bi + (long long)(i - i0) * 64;
                    for (int kk = 0; kk <= i - i0; kk++) s1 += Di[kk] * gcol[(long long)(i0 + kk) * wp.ldG];
                    v = s0 + s1;
                }
                __syncthreads();
                if (i < n) gcol[(long long)i * wp.ldG] = v;
                __syncthreads();
            }
            continue;
        }
        const int c0 = 64 * tk.y, nc = min(64, ncol - c0);
        double* Gl = wp.G + (tp.leaf_off[l] - wp.G_base) * wp.ldG + c0;
        for (int i = (n - 1) / 64; i >= 0; i--) {
            const int i0 = 64 * i, nb = min(64, n - i0);
            const double* Di = wp.D + wp.D_off[l] + 4096LL * i;
            cta_gemm<MEMT, MEMT, MEMN, MEMT>(nb, nc, 0, op_mem(Sl + i0, ld), op_mem(Gl, wp.ldG), i0, op_mem(Di, 64),
                                             op_mem(Gl + (long long)i0 * wp.ldG, wp.ldG), nb, ci_zero(), 1.0,
                                             Gl + (long long)i0 * wp.ldG, wp.ldG, cp, smem);
        }
    }
}

static int g_gemm_resident[6] = {1, 1, 1, 1, 1, 1};   // resident CTAs per SM x SM count, by phase
static bool g_gemm_attr_done = false;
static int gemm_smem_bytes() { return GEMM_SMEM_DBL * (int)sizeof(double); }
static void gemm_set_attrs() {
    if (g_gemm_attr_done) return;
    const int b = gemm_smem_bytes();
    const void* ks[6] = {(const void*)k_wide_chain, (const void*)k_wide_sigma, (const void*)k_wide_update,
                         nullptr, (const void*)k_wide_panel_x, (const void*)k_wide_trsm};
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    for (int i = 0; i < 6; i++) {
        if (!ks[i]) continue;
        cudaFuncSetAttribute(ks[i], cudaFuncAttributeMaxDynamicSharedMemorySize, b);
        int per = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, ks[i], NT, b);
        g_gemm_resident[i] = (per > 0 ? per : 1) * nsm;
    }
    g_gemm_attr_done = true;
}

// phases: 0 chain, 1 sigma, 2 update, 3 diag, 4 panel_x, 5 trsm, 6 covfill (3 and 6: mra_kernels.cu).
// `grid` is ignored for this unit's phases: a persistent grid of every resident CTA pulls the tasks.
cudaError_t launch_wide(int phase, const TreeParams& tp, const WideParams& wp, int step, const int4* tasks,
                        long long ntask, int grid, unsigned long long* counter, cudaStream_t st) {
    if (phase == 3 || phase == 6) return launch_wide_main(phase, tp, wp, step, tasks, ntask, grid, counter, st);
    if (phase < 0 || phase > 6) return cudaErrorInvalidValue;
    gemm_set_attrs();
    long long g = g_gemm_resident[phase];
    if (ntask < g) g = ntask;
    if (g < 1) return cudaSuccess;
    const int b = gemm_smem_bytes();
    switch (phase) {
        case 0: k_wide_chain<<<(int)g, NT, b, st>>>(tp, wp, tasks, ntask, counter); break;
        case 1: k_wide_sigma<<<(int)g, NT, b, st>>>(tp, wp, tasks, ntask, counter); break;
        case 2: k_wide_update<<<(int)g, NT, b, st>>>(tp, wp, step, tasks, ntask, counter); break;
        case 4: k_wide_panel_x<<<(int)g, NT, b, st>>>(tp, wp, step, tasks, ntask, counter); break;
        case 5: k_wide_trsm<<<(int)g, NT, b, st>>>(tp, wp, tasks, ntask, counter); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace mra
