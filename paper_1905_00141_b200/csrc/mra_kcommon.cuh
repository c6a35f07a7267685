// mra_kcommon.cuh -- device helpers shared by the kernel translation units (mra_kernels.cu: default
// engine; mra_kernels_gemm.cu: the GEMM-only wide-path kernels, built with their own engine shape).
// Include after mra_device.cuh and mra_internal.h.
#pragma once

#ifndef MRA_MINB
#define MRA_MINB 2   // resident CTAs per SM the register allocation is sized for (256-thread CTAs)
#endif

namespace mra {
inline namespace MRA_ENG_NS {

#ifdef MRA_PHASE_TIMING
#define PHASE_MARK(var) long long var = clock64()
#define PHASE_ADD(idx, from)                                                                  \
    do {                                                                                      \
        if (threadIdx.x == 0) atomicAdd(&g_phase_cycles[idx], (unsigned long long)(clock64() - (from))); \
    } while (0)
#else
#define PHASE_MARK(var)
#define PHASE_ADD(idx, from)
#endif

__device__ __forceinline__ long long lvl_first(int J, int m) {
    long long p = 1;
    for (int i = 1; i < m; i++) p *= J;
    return (p - 1) / (J - 1);
}

__device__ __forceinline__ CovP to_covp(const CovParams& c) {
    CovP p;
    p.kind = c.kind; p.s2 = c.s2; p.rho = c.rho; p.xs = c.xs; p.ys = c.ys;
    p.ir = (c.kind == 0 ? 1.0 : 1.7320508075688772935) / c.rho;
    return p;
}
// theta of the evaluation: by value in TreeParams, or -- for an evaluation replayed as a CUDA graph -- read from the
// plan's device buffer {sigma2, rho, tau2} that the host refreshes before each replay (the covariance family is
// part of the graph's key)
__device__ __forceinline__ CovP covp_of(const TreeParams& tp) {
    CovParams c = tp.cp;
    if (tp.theta_dev) {
        c.s2 = tp.theta_dev[0];
        c.rho = tp.theta_dev[1];
    }
    return to_covp(c);
}
__device__ __forceinline__ double tau2_of(const TreeParams& tp) { return tp.theta_dev ? tp.theta_dev[2] : tp.tau2; }

__device__ __forceinline__ void set_err(int* err, int level, long long idx) {
    if (atomicCAS(err, 0, 1) == 0) {
        err[1] = level;
        *reinterpret_cast<long long*>(err + 2) = idx;
    }
}

// persistent work queue: returns the next item index (uniform across the CTA)
__device__ __forceinline__ long long next_item(unsigned long long* counter, double* smem) {
    long long* slot = reinterpret_cast<long long*>(misc_smem(smem) + 18);
    __syncthreads();
    if (threadIdx.x == 0) *slot = (long long)atomicAdd(counter, 1ULL);
    __syncthreads();
    long long v = *slot;
    return v;
}

__device__ __forceinline__ const double* chain_row(const TreeParams& tp, int k, long long ak) {
    return tp.prior + tp.prior_base[k] + (ak - tp.prior_first[k]) * (long long)k * tp.rh * tp.rh;
}

// V chain of a point set P (n points inside level-m region t): for k = 1..m
//   V^k(P) = [ C(P, Q_{a_k}) | V^{k-1}(P) .. V^1(P) ] R_{a_k}^T        (K = k * rh)
// written into Gc at column block m-k (levels in descending order), ld ldg.
__device__ void point_chain(const TreeParams& tp, int m, long long t, int n, const double* pts, double* Gc,
                            long long ldg, const CovP& cp, double* smem) {
    const int rh = tp.rh;
    for (int k = 1; k <= m; k++) {
        const long long ak = t >> (tp.lj * (m - k));
        const long long akid = lvl_first(tp.J, k) + ak;
        const long long ldk = (long long)k * rh;
        const double* Rk = chain_row(tp, k, ak);
        PHASE_MARK(pc0);
        cta_gemm<COVK, MEMN, MEMN, MEMN>(n, rh, 0, op_cov(pts, tp.kxy + 2 * akid * rh),
                                         op_mem(Rk, ldk), rh, op_mem(Gc + (long long)(m - k + 1) * rh, ldg),
                                         op_mem(Rk + rh, ldk), (k - 1) * rh, ci_zero(), 1.0,
                                         Gc + (long long)(m - k) * rh, ldg, cp, smem);
        PHASE_ADD(26, pc0);
#ifdef MRA_PHASE_TIMING
        if (threadIdx.x == 0) atomicAdd(&g_phase_cycles[27], (unsigned long long)k);   // sum of k (= K / rh)
#endif
    }
}

// V chain over covariance blocks already in place: Gc's column block m-k holds C(P, Q_{a_k}) on entry
// (k_wide_covfill) and V^k on exit. Each step is one single-segment GEMM over the contiguous columns
// [C_k | V^{k-1} .. V^1] that overwrites C_k (every output tile reads only its own rows).
__device__ void point_chain_pre(const TreeParams& tp, int m, long long t, int n, double* Gc, long long ldg,
                                const CovP& cp, double* smem) {
    const int rh = tp.rh;
    for (int k = 1; k <= m; k++) {
        const long long ak = t >> (tp.lj * (m - k));
        const long long ldk = (long long)k * rh;
        const double* Rk = chain_row(tp, k, ak);
        double* Ck = Gc + (long long)(m - k) * rh;
        cta_gemm<MEMN, MEMN, MEMN, MEMN>(n, rh, 0, op_mem(Ck, ldg), op_mem(Rk, ldk), k * rh, op_mem(Ck, ldg),
                                         op_mem(Ck, ldg), 0, ci_zero(), 1.0, Ck, ldg, cp, smem);
    }
}

// --------------------------------------------------------------------------- prior
// Covariance blocks of the prior chains of level-m regions, in place of the chain row R (ld m rh):
// block 0 <- C(Q_R, Q_R) (k_prior turns it into W^m, then overwrites it with L^{-1}), block m-k <-
// C(Q_R, Q_{a_k}) for k < m (turned into V^k, then -U^k). Own phase, like k_wide_covfill: no DMMA shares
// the fp64 pipe with the sqrt / exp chains.
constexpr int CFT = 256;   // threads of the covariance-generation kernels (independent of the engine's NT)

__device__ __forceinline__ int leaf_n(const TreeParams& tp, long long l) {
    return (int)(tp.leaf_off[l + 1] - tp.leaf_off[l]);
}


// factor view of the smem main area: out of place (mra_kernels.cu: L and L^{-1} both kept, 76 KB) or in
// place (mra_kernels_gemm.cu: L^{-1} overwrites L, 42 KB), chosen per translation unit
#ifndef MRA_FAC_INPLACE
#define MRA_FAC_INPLACE 0
#endif
__device__ __forceinline__ FacSmem fac_view(double* smem) {
    return MRA_FAC_INPLACE ? fac_smem_inplace(smem) : fac_smem(smem);
}

// merge of region with Atilde (ncol x ncol lower, ld ldA): Lt = chol(I + A_oo), Li = Lt^{-1},
// F = A_ro Li^T, O = A_rr - F F^T (q = ncol - rh). Returns log|I + A_oo|.
__device__ double merge_core(const double* A, int rh, long long ldA, double* O, int q, double* F, double* Li,
                             int* err, int level, long long t, const CovP& cp, double* smem) {
    FacSmem f = fac_view(smem);
    load_block_lower(f.blk, A, ldA, rh, 1.0);
    const double ld = chol_inv_small(f.blk, f.inv, rh, f.diagv, f.bad, f.red, f.tmp);
    if (*f.bad && threadIdx.x == 0) set_err(err, level, t);
    store_block_full(f.inv, Li, rh, rh);
    __syncthreads();
    cta_gemm<MEMN, MEMN, MEMN, MEMN>(q, rh, 0, op_mem(A + (long long)rh * ldA, ldA), op_mem(Li, rh), rh,
                                     op_mem(Li, rh), op_mem(Li, rh), 0, ci_zero(), 1.0, F, rh, cp, smem);
    cta_gemm<MEMN, MEMN, MEMN, MEMN>(q, q, 1, op_mem(F, rh), op_mem(F, rh), rh, op_mem(F, rh), op_mem(F, rh), 0,
                                     ci_mem(A + (long long)rh * ldA + rh, ldA), -1.0, O, q, cp, smem);
    return ld;
}

__device__ __forceinline__ void save_post(const TreeParams& tp, int m, long long t, int q, const double* Li,
                                          const double* F) {
    if (!tp.post) return;
    const int rh = tp.rh;
    double* P = tp.post + tp.post_base[m] + t * ((long long)rh * rh + (long long)q * rh);
    for (int e = threadIdx.x; e < rh * rh; e += NT) P[e] = Li[e];
    for (int e = threadIdx.x; e < q * rh; e += NT) P[rh * rh + e] = F[e];
}

}  // inline namespace MRA_ENG_NS
}  // namespace mra
