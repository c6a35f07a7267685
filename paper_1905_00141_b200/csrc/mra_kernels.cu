// mra_kernels.cu -- sm_100a kernels of the MRA log-likelihood hot path.
//
// Whitened formulation: every pre-finest region R at level m stores its chain row
//   R_R = [ L_R^{-1} | -L_R^{-1} V^{m-1}_R | ... | -L_R^{-1} V^1_R ]           (rh x m*rh)
// where L_R = chol(W^m_R) and V^k_R = W^k_R L_{a_k}^{-T} (north_star W-recursion).
// For any point set P inside R's subtree the chain block V^k(P) = [C(P, Q_{a_k}) | V^{k-1}(P)..V^1(P)]
// R_{a_k}^T is ONE GEMM whose first K-segment is generated covariance (fused covgen).
// The posterior pass then works with identity priors: Ktilde^{-1} = I + Atilde^{mm} and
// d_R = sum d_c + log|I + Atilde^{mm}| (equal to the paper's log|W^m + A^{mm}| - log|W^m|).
//
// Kernels (persistent CTAs of 256 threads, one work item = one region, dynamic atomic queue):
//   k_prior   level m: V chain + W^m = C(Q,Q) - V V^T, chol, inverse, U = L^{-1} V
//   k_bottom  one level-(M-1) region p with its J leaves: per leaf V (chain GEMMs with fused
//             covariance), Sigma_j = C(S,S) + tau2 I - V V^T, blocked Cholesky, G = L^{-1}[V|y];
//             then Atilde_p = G_stack^T G_stack (stacked SYRK over the J leaves, no per-leaf ATilde
//             is ever stored) and the merge of p.
//   k_merge   level m < M-1: Atilde = sum of J child outputs, merge.
//   k_mu / k_smooth   posterior state (top-down), only when requested.
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>

#include "mra_device.cuh"
#include "mra_internal.h"

#include "mra_kcommon.cuh"

namespace mra {

__global__ void __launch_bounds__(CFT)
k_prior_covfill(TreeParams tp, int m, long long t_first, long long nitems) {
    __shared__ double2 pts_s[64];
    __shared__ double2 knots_s[MAXM * 64];
    const CovP cp = covp_of(tp);
    const int rh = tp.rh, W = m * rh;
    const long long ldR = (long long)m * rh;
    for (long long it = blockIdx.x; it < nitems; it += gridDim.x) {
        const long long t = t_first + it;
        const long long id = lvl_first(tp.J, m) + t;
        __syncthreads();
        if (threadIdx.x < rh) pts_s[threadIdx.x] = ldpt(tp.kxy + 2 * id * rh, threadIdx.x);
        for (int c = threadIdx.x; c < W; c += CFT) {   // column block b holds level m - b (b = 0: R itself)
            const int b = c / rh, k = m - b;
            const long long akid = lvl_first(tp.J, k) + (t >> (tp.lj * (m - k)));
            knots_s[c] = ldpt(tp.kxy + 2 * akid * rh, c - b * rh);
        }
        __syncthreads();
        double* R = tp.prior + tp.prior_base[m] + (t - tp.prior_first[m]) * ldR * rh;
        int i = 0, c = threadIdx.x;
        while (c >= W) { c -= W; i++; }
        const int di = CFT / W, dc = CFT - di * W;
#pragma unroll 4
        for (int e = threadIdx.x; e < rh * W; e += CFT) {
            const double2 pp = pts_s[i], q = knots_s[c];
            R[(long long)i * ldR + c] = covf(cp, pp.x, pp.y, q.x, q.y);
            i += di;
            c += dc;
            if (c >= W) { c -= W; i++; }
        }
    }
}




// Atilde_p = G_stack^T G_stack over the group's leaves (lower), then the merge of level-(M-1) region t
__device__ void group_tail(const TreeParams& tp, int m, long long t, const double* G, long long ldG, int ng,
                           double dsum, double* out, long long out_first, int q, double* A, long long ldA, double* F,
                           double* Li, const CovP& cp, double* smem) {
    const int ncol = m * tp.rh + 1;
    PHASE_MARK(c4);
    cta_gemm<MEMT, MEMT, MEMN, MEMN>(ncol, ncol, 1, op_mem(G, ldG), op_mem(G, ldG), ng, op_mem(G, 0), op_mem(G, 0), 0,
                                     ci_zero(), 1.0, A, ldA, cp, smem);
    PHASE_ADD(4, c4);
    PHASE_MARK(c5);
    double* O = out + (t - out_first) * (long long)q * q;
    const double ldm = merge_core(A, tp.rh, ldA, O, q, F, Li, tp.err, m, t, cp, smem);
    PHASE_ADD(5, c5);
    const long long id = lvl_first(tp.J, m) + t;
    if (threadIdx.x == 0) {
        tp.dreg[id] = dsum + ldm;
        tp.ureg[id] = O[(long long)(q - 1) * q + q - 1];
    }
    save_post(tp, m, t, q, Li, F);
}

// -------------------------------------------------------------------------- bottom
__global__ void __launch_bounds__(NT, MRA_MINB)
k_bottom(TreeParams tp, long long g_first, long long g_count, double* out, long long out_first, int q, double* ws,
         WsLayout L, unsigned long long* counter) {
    double* smem = dyn_smem();
    const CovP cp = covp_of(tp);
    const int M = tp.M, J = tp.J, rh = tp.rh;
    const int m = M - 1;                 // group level; 0 when M == 1 (the root is the only leaf)
    const int Jc = (M == 1) ? 1 : J;     // leaves per group
    const int Pg = m * rh, ncol = Pg + 1;
    double* base = ws + (long long)blockIdx.x * L.stride;
    double *G = base + L.oG, *S = base + L.oS, *D = base + L.oD, *A = base + L.oA, *F = base + L.oF,
           *Li = base + L.oL;
    FacSmem f = fac_smem(smem);
    double* red = misc_smem(smem);
    const long long leaf_id0 = lvl_first(J, M);
    PHASE_MARK(kstart);
    for (;;) {
        const long long it = next_item(counter, smem);
        if (it >= g_count) break;
        if (threadIdx.x == 0) *f.bad = 0;
        const long long t = g_first + it;
        const long long l0 = t * Jc;
        const long long obase = tp.leaf_off[l0];
        const long long ng = tp.leaf_off[l0 + Jc] - obase;
        double dsum = 0.0, ulast = 0.0;
        for (int c = 0; c < Jc; c++) {
            const long long l = l0 + c;
            const long long o0 = tp.leaf_off[l];
            const int n = (int)(tp.leaf_off[l + 1] - o0);
            if (n == 0) {   // empty leaf: zero contribution (reading R10)
                if (threadIdx.x == 0) { tp.dreg[leaf_id0 + l] = 0.0; tp.ureg[leaf_id0 + l] = 0.0; }
                continue;
            }
            double* Gc = G + (o0 - obase) * L.ldG;
            const double* pts = tp.pxy + 2 * o0;
            PHASE_MARK(c0);
            point_chain(tp, m, t, n, pts, Gc, L.ldG, cp, smem);
            for (int i = threadIdx.x; i < n; i += NT) Gc[(long long)i * L.ldG + Pg] = tp.zs[o0 + i];
            __syncthreads();
            PHASE_ADD(0, c0);
            PHASE_MARK(c1);
            // Sigma_j = C(S,S) + tau2 I - V V^T  (nugget on the observation diagonal only, reading R2)
            cta_gemm<MEMN, MEMN, MEMN, MEMN, 1>(n, n, 1, op_mem(Gc, L.ldG), op_mem(Gc, L.ldG), Pg, op_mem(Gc, L.ldG),
                                             op_mem(Gc, L.ldG), 0, ci_cov(pts, pts, tau2_of(tp)), -1.0, S,
                                             L.ldS, cp, smem);
            PHASE_ADD(1, c1);
            PHASE_MARK(c2);
            const double ldet = chol_blocked(S, n, L.ldS, D, cp, smem);
            if (*f.bad && threadIdx.x == 0) set_err(tp.err, M, l);
            PHASE_ADD(2, c2);
            PHASE_MARK(c3);
            fwd_subst(S, n, L.ldS, D, Gc, ncol, L.ldG, cp, smem);
            PHASE_ADD(3, c3);
            double u = 0.0;
            for (int i = threadIdx.x; i < n; i += NT) {
                const double g = Gc[(long long)i * L.ldG + Pg];
                u += g * g;
            }
            u = cta_sum(u, red);
            if (threadIdx.x == 0) { tp.dreg[leaf_id0 + l] = ldet; tp.ureg[leaf_id0 + l] = u; }
            dsum += ldet;
            ulast = u;
        }
        if (m == 0) {   // M == 1: the leaf is the root
            if (threadIdx.x == 0) { tp.dreg[0] = dsum; tp.ureg[0] = ulast; }
            continue;
        }
        group_tail(tp, m, t, G, L.ldG, (int)ng, dsum, out, out_first, q, A, L.ldA, F, Li, cp, smem);
    }
    PHASE_ADD(12, kstart);
}


// log L = -1/2 (N log 2 pi + d_root + u_root)
__global__ void k_final(TreeParams tp, double N, double* loglik) {
    if (threadIdx.x == 0 && blockIdx.x == 0)
        *loglik = -0.5 * (N * log(2.0 * 3.14159265358979323846) + tp.dreg[0] + tp.ureg[0]);
}

__global__ void k_gather(const double* z, const long long* perm, double* zs, long long N) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x)
        zs[i] = z[perm[i]];
}

__global__ void k_fill(double* p, long long n, double v) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        p[i] = v;
}

__global__ void k_scatter(const double* zs, const long long* perm, double* z, long long N) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x)
        z[perm[i]] = zs[i];
}

// ------------------------------------------------------------- exchange buffer (subtree sharding)
// packed layout (include/mra.h mra_shard_size): ns lower triangles of q x q, row by row (i(i+1)/2 + j),
// then d[ns], u[ns], then one error flag. Row of packed index r: i = floor((sqrt(8r+1)-1)/2), fixed up
// in integers (the fp64 estimate is exact or off by one for r < 2^50).
__device__ __forceinline__ void tri_rc(long long r, int* i, int* j) {
    long long ii = (long long)((sqrt(8.0 * (double)r + 1.0) - 1.0) * 0.5);
    while (ii * (ii + 1) / 2 > r) ii--;
    while ((ii + 1) * (ii + 2) / 2 <= r) ii++;
    *i = (int)ii;
    *j = (int)(r - ii * (ii + 1) / 2);
}
__global__ void k_pack_exchange(const double* out, long long ns, int q, const double* d, const double* u,
                                const int* err, double* xbuf) {
    const long long qq = (long long)q * (q + 1) / 2, tot = ns * qq;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot + 2 * ns + 1;
         e += (long long)gridDim.x * blockDim.x) {
        if (e < tot) {
            const long long t = e / qq;
            int i, j;
            tri_rc(e - t * qq, &i, &j);
            xbuf[e] = out[t * q * q + (long long)i * q + j];
        } else if (e < tot + ns) {
            xbuf[e] = d[e - tot];
        } else if (e < tot + 2 * ns) {
            xbuf[e] = u[e - tot - ns];
        } else {
            xbuf[e] = err[0] ? 1.0 : 0.0;
        }
    }
}
__global__ void k_unpack_exchange(const double* xbuf, long long ns, int q, double* out, double* d, double* u) {
    const long long qq = (long long)q * (q + 1) / 2, tot = ns * qq;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot + 2 * ns;
         e += (long long)gridDim.x * blockDim.x) {
        if (e < tot) {
            const long long t = e / qq;
            int i, j;
            tri_rc(e - t * qq, &i, &j);
            out[t * q * q + (long long)i * q + j] = xbuf[e];
        } else if (e < tot + ns) {
            d[e - tot] = xbuf[e];
        } else {
            u[e - tot - ns] = xbuf[e];
        }
    }
}

// ----------------------------------------------------------------- posterior state
// muhat_R = Lt^{-T} (h - sum_k H^k muhat_{a_k})   (whitened), mu_R = L_R^{-T} muhat_R (paper's eta)
__global__ void k_mu(TreeParams tp, int m, double* muhat, double* mu, long long t_first, long long t_count) {
    __shared__ double tv[64], mh[64];
    const int rh = tp.rh, q = (m - 1) * rh + 1;
    for (long long t = t_first + blockIdx.x; t < t_first + t_count; t += gridDim.x) {
        const long long id = lvl_first(tp.J, m) + t;
        const double* Li = tp.post + tp.post_base[m] + t * ((long long)rh * rh + (long long)q * rh);
        const double* F = Li + rh * rh;
        for (int a = threadIdx.x; a < rh; a += blockDim.x) {
            double s = F[(long long)(q - 1) * rh + a];
            for (int b = 0; b < q - 1; b++) {
                const int bi = b / rh, lev = m - 1 - bi;
                const long long anc = lvl_first(tp.J, lev) + (t >> (tp.lj * (m - lev)));
                s -= F[(long long)b * rh + a] * muhat[anc * rh + (b - bi * rh)];
            }
            tv[a] = s;
        }
        __syncthreads();
        for (int a = threadIdx.x; a < rh; a += blockDim.x) {
            double s = 0.0;
            for (int b = 0; b < rh; b++) s += Li[b * rh + a] * tv[b];
            mh[a] = s;
        }
        __syncthreads();
        const double* Rr = chain_row(tp, m, t);
        const long long ldR = (long long)m * rh;
        for (int a = threadIdx.x; a < rh; a += blockDim.x) {
            muhat[id * rh + a] = mh[a];
            double s = 0.0;
            for (int b = 0; b < rh; b++) s += Rr[(long long)b * ldR + a] * mh[b];
            if (mu) mu[id * rh + a] = s;
        }
        __syncthreads();
    }
}

// E[X(S_j)|y] = y_j - tau2 Sigma_j^{-1} (y_j - sum_k V^k muhat_{a_k})   (recomputes V, Sigma_j, L_j)
__global__ void __launch_bounds__(NT, MRA_MINB)
k_smooth(TreeParams tp, const double* muhat, const long long* perm, double* smooth, double* ws, WsLayout L,
         unsigned long long* counter, long long l_first, long long l_count) {
    double* smem = dyn_smem();
    const CovP cp = covp_of(tp);
    const int M = tp.M, rh = tp.rh, m = M - 1, Pg = m * rh;
    double* base = ws + (long long)blockIdx.x * L.stride;
    double *G = base + L.oG, *S = base + L.oS, *D = base + L.oD, *r = base + L.oV;
    FacSmem f = fac_smem(smem);
    double* tmp = misc_smem(smem);   // not used for vectors; vectors live in r
    (void)tmp;
    long long nleaves = 1;
    for (int i = 1; i < M; i++) nleaves *= tp.J;
    for (;;) {
        const long long l = l_first + next_item(counter, smem);
        if (l >= l_first + l_count) break;
        if (threadIdx.x == 0) *f.bad = 0;
        const long long t = (M == 1) ? 0 : (l >> tp.lj);
        const long long o0 = tp.leaf_off[l];
        const int n = (int)(tp.leaf_off[l + 1] - o0);
        if (n == 0) continue;
        const double* pts = tp.pxy + 2 * o0;
        point_chain(tp, m, t, n, pts, G, L.ldG, cp, smem);
        cta_gemm<MEMN, MEMN, MEMN, MEMN, 1>(n, n, 1, op_mem(G, L.ldG), op_mem(G, L.ldG), Pg, op_mem(G, L.ldG),
                                         op_mem(G, L.ldG), 0, ci_cov(pts, pts, tau2_of(tp)), -1.0, S, L.ldS, cp,
                                         smem);
        chol_blocked(S, n, L.ldS, D, cp, smem);
        if (*f.bad && threadIdx.x == 0) set_err(tp.err, M, l);
        // r = y - V muhat_chain
        for (int i = threadIdx.x; i < n; i += NT) {
            double s = tp.zs[o0 + i];
            for (int col = 0; col < Pg; col++) {
                const int b = col / rh, lev = m - b;
                const long long anc = lvl_first(tp.J, lev) + (t >> (tp.lj * (m - lev)));
                s -= G[(long long)i * L.ldG + col] * muhat[anc * rh + (col - b * rh)];
            }
            r[i] = s;
        }
        __syncthreads();
        double* w = f.blk;   // smem scratch [64]
        // forward: r <- L^{-1} r
        for (int i0 = 0; i0 < n; i0 += 64) {
            const int nb = min(64, n - i0);
            for (int ii = threadIdx.x; ii < nb; ii += NT) {
                double s = r[i0 + ii];
                for (int k = 0; k < i0; k++) s -= S[(long long)(i0 + ii) * L.ldS + k] * r[k];
                w[ii] = s;
            }
            __syncthreads();
            const double* Di = D + (long long)(i0 / 64) * 4096;
            for (int ii = threadIdx.x; ii < nb; ii += NT) {
                double s = 0.0;
                for (int k = 0; k <= ii; k++) s += Di[ii * 64 + k] * w[k];
                r[i0 + ii] = s;
            }
            __syncthreads();
        }
        // backward: r <- L^{-T} r
        const int nblk = (n + 63) / 64;
        for (int bb = nblk - 1; bb >= 0; bb--) {
            const int i0 = bb * 64, nb = min(64, n - i0);
            for (int ii = threadIdx.x; ii < nb; ii += NT) {
                double s = r[i0 + ii];
                for (int k = i0 + nb; k < n; k++) s -= S[(long long)k * L.ldS + i0 + ii] * r[k];
                w[ii] = s;
            }
            __syncthreads();
            const double* Di = D + (long long)bb * 4096;
            for (int ii = threadIdx.x; ii < nb; ii += NT) {
                double s = 0.0;
                for (int k = ii; k < nb; k++) s += Di[k * 64 + ii] * w[k];
                r[i0 + ii] = s;
            }
            __syncthreads();
        }
        for (int i = threadIdx.x; i < n; i += NT) smooth[perm[o0 + i]] = tp.zs[o0 + i] - tau2_of(tp) * r[i];
    }
}


// ---------------------------------------------------------------- prediction
// Posterior mean and variance of the noise-free X at query points P of leaf j (the
// "prediction" mode of PAPER.md:228; oracle: predict_all). With the whitened basis v(p) = V(p) of the
// query (same chain as the observations), E = L_j^{-1} C_M(S_j, P), C_M(S, P) = C(S, P) - V_S V(P)^T:
//   mean(p) = v(p) muhat + E_p^T (g - G_V muhat)
//   var(p)  = sigma^2 - |v(p)|^2 - |E_p|^2 + |U^{-T} b(p)|^2,  b(p) = v(p) - G_V^T E_p,
// where U^{-T} is the back substitution along the ancestor chain with the merge factors kept by the
// posterior pass (Ltilde^{-1} and F = H^T per region): s_m = Li_m b_m, s_k = Li_k (b_k - sum_{j>k} F_j[k] s_j)
// (the chain's posterior covariance, the paper's BTilde, is U^{-1} U^{-T} in the whitened basis).
__global__ void __launch_bounds__(NT, MRA_MINB)
k_predict(TreeParams tp, PredParams pp, double* ws, WsLayout L, unsigned long long* counter) {
    double* smem = dyn_smem();
    const CovP cp = covp_of(tp);
    const int M = tp.M, J = tp.J, rh = tp.rh, m = M - 1, Pg = m * rh, ncol = Pg + 1;
    double* base = ws + (long long)blockIdx.x * L.stride;
    double *G = base + L.oG, *S = base + L.oS, *D = base + L.oD, *r = base + L.oV, *Q = base + L.oQ,
           *E = base + L.oE, *W = base + L.oW;
    FacSmem f = fac_smem(smem);
    auto mu_chain = [&](long long t, int col) -> double {   // muhat of the ancestor owning G column col
        const int b = col / rh, lev = m - b;
        const long long anc = lvl_first(J, lev) + (t >> (tp.lj * (m - lev)));
        return pp.muhat[anc * rh + (col - b * rh)];
    };
    for (;;) {
        const long long it = next_item(counter, smem);
        if (it >= pp.n_leaves) break;
        if (threadIdx.x == 0) *f.bad = 0;
        const long long l = pp.leaves[it];
        const long long t = (M == 1) ? 0 : (l >> tp.lj);
        const long long o0 = tp.leaf_off[l];
        const int n = (int)(tp.leaf_off[l + 1] - o0);
        const double* pts = tp.pxy + 2 * o0;
        if (n > 0) {   // the leaf's posterior-pass quantities: G = L^{-1}[V | y], L (blocked), r = g - G_V muhat
            point_chain(tp, m, t, n, pts, G, L.ldG, cp, smem);
            for (int i = threadIdx.x; i < n; i += NT) G[(long long)i * L.ldG + Pg] = tp.zs[o0 + i];
            __syncthreads();
            cta_gemm<MEMN, MEMN, MEMN, MEMN, 1>(n, n, 1, op_mem(G, L.ldG), op_mem(G, L.ldG), Pg, op_mem(G, L.ldG),
                                             op_mem(G, L.ldG), 0, ci_cov(pts, pts, tau2_of(tp)), -1.0, S, L.ldS, cp,
                                             smem);
            chol_blocked(S, n, L.ldS, D, cp, smem);
            if (*f.bad && threadIdx.x == 0) set_err(tp.err, M, l);
            fwd_subst(S, n, L.ldS, D, G, ncol, L.ldG, cp, smem);
            for (int i = threadIdx.x; i < n; i += NT) {
                double s = G[(long long)i * L.ldG + Pg];
                for (int col = 0; col < Pg; col++) s -= G[(long long)i * L.ldG + col] * mu_chain(t, col);
                r[i] = s;
            }
            __syncthreads();
        }
        const long long q0 = pp.q_off[l], nq = pp.q_off[l + 1] - q0;
        for (long long qt = 0; qt < nq; qt += 64) {
            const int nt = (int)min(64LL, nq - qt);
            const double* qp = pp.qxy + 2 * (q0 + qt);
            point_chain(tp, m, t, nt, qp, Q, L.ldG, cp, smem);   // v(p), rows of Q
            if (n > 0) {
                // E = L^{-1} C_M(S, P) = L^{-1} C(S, P) - G_V V(P)^T   (G already holds L^{-1} V)
                cta_gemm<MEMN, MEMN, MEMN, MEMN, 1>(n, nt, 0, op_mem(G, L.ldG), op_mem(Q, L.ldG), 0, op_mem(G, 0),
                                                 op_mem(G, 0), 0, ci_cov(pts, qp, 0.0), 1.0, E, 64, cp, smem);
                fwd_subst(S, n, L.ldS, D, E, nt, 64, cp, smem);
                if (Pg > 0)
                    cta_gemm<MEMN, MEMN, MEMN, MEMN>(n, nt, 0, op_mem(G, L.ldG), op_mem(Q, L.ldG), Pg, op_mem(G, 0),
                                                     op_mem(G, 0), 0, ci_mem(E, 64), -1.0, E, 64, cp, smem);
            }
            __syncthreads();
            double mean = 0.0, var = 0.0;
            if (threadIdx.x < nt) {
                const int i = threadIdx.x;
                double vv = 0.0, ee = 0.0;
                for (int col = 0; col < Pg; col++) {
                    const double v = Q[(long long)i * L.ldG + col];
                    mean += v * mu_chain(t, col);
                    vv += v * v;
                }
                for (int k = 0; k < n; k++) {
                    const double e = E[(long long)k * 64 + i];
                    mean += e * r[k];
                    ee += e * e;
                }
                var = cp.s2 - vv - ee;
            }
            if (m >= 1) {
                // b = v - G_V^T E  (in place over Q)
                if (n > 0)
                    cta_gemm<MEMT, MEMT, MEMN, MEMN>(nt, Pg, 0, op_mem(E, 64), op_mem(G, L.ldG), n, op_mem(E, 0),
                                                     op_mem(E, 0), 0, ci_mem(Q, L.ldG), -1.0, Q, L.ldG, cp, smem);
                // chain back substitution, levels m..1 (G column block of level k: (m - k) rh)
                for (int k = m; k >= 1; k--) {
                    const int cb = (m - k) * rh, qk = (k - 1) * rh + 1;
                    const long long ak = t >> (tp.lj * (m - k));
                    const double* Lik = tp.post + tp.post_base[k] + ak * ((long long)rh * rh + (long long)qk * rh);
                    const double* Tk = Q + cb;
                    for (int j = k + 1; j <= m; j++) {
                        const int qj = (j - 1) * rh + 1;
                        const long long aj = t >> (tp.lj * (m - j));
                        const double* Fj = tp.post + tp.post_base[j] + aj * ((long long)rh * rh + (long long)qj * rh) +
                                           (long long)rh * rh + (long long)(j - 1 - k) * rh * rh;
                        cta_gemm<MEMN, MEMN, MEMN, MEMN>(nt, rh, 0, op_mem(W + (m - j) * rh, L.ldG), op_mem(Fj, rh),
                                                         rh, op_mem(Fj, 0), op_mem(Fj, 0), 0, ci_mem(Tk, L.ldG), -1.0,
                                                         W + cb, L.ldG, cp, smem);
                        Tk = W + cb;
                    }
                    cta_gemm<MEMN, MEMN, MEMN, MEMN>(nt, rh, 0, op_mem(Tk, L.ldG), op_mem(Lik, rh), rh,
                                                     op_mem(Lik, 0), op_mem(Lik, 0), 0, ci_zero(), 1.0, W + cb, L.ldG,
                                                     cp, smem);
                }
                __syncthreads();
                if (threadIdx.x < nt)
                    for (int col = 0; col < Pg; col++) {
                        const double s2 = W[(long long)threadIdx.x * L.ldG + col];
                        var += s2 * s2;
                    }
            }
            if (threadIdx.x < nt) {
                const long long dst = pp.q_perm[q0 + qt + threadIdx.x];
                pp.mean[dst] = mean;
                pp.var[dst] = var;
            }
            __syncthreads();
        }
    }
}

// ====================================================================== wide (big-leaf) path
// Leaves too large for one CTA (C4: up to ~9k observations) are processed by all CTAs together,
// phase by phase, from precomputed task lists: row-tile V chains, Sigma tiles, a
// left-looking batched blocked Cholesky (per step s: column update with K = 64 s, diagonal factor
// per leaf, panel solve), batched block forward substitution, per-leaf d/u, then per group the
// stacked SYRK + merge. Tasks are int4 {leaf, i, k, 0}.


// Covariance blocks C(P, Q_{a_k}), k = 1..M-1, of 64 rows of one leaf into G's column blocks (M-1-k)
// and the y column: a phase of its own, with no DMMA work sharing the fp64 pipe (generated inside the
// chain GEMMs, every dependent sqrt / exp chain queued behind the other CTA's DMMAs: ~9k cycles per
// 64 x 32 stage). Same covf arithmetic as the fused path.
__global__ void __launch_bounds__(CFT)
k_wide_covfill(TreeParams tp, WideParams wp, const int4* tasks, long long ntask) {
    __shared__ double2 pts_s[64];
    __shared__ double2 knots_s[MAXM * 64];
    const CovP cp = covp_of(tp);
    const int rh = tp.rh, m = tp.M - 1, Pg = m * rh;
    for (long long it = blockIdx.x; it < ntask; it += gridDim.x) {
        const int4 tk = tasks[it];
        const long long l = tk.x, t = l >> tp.lj;
        const long long o0 = tp.leaf_off[l] + 64LL * tk.y;
        const int n = min(64, leaf_n(tp, l) - 64 * tk.y);
        __syncthreads();
        if (threadIdx.x < n) pts_s[threadIdx.x] = ldpt(tp.pxy, o0 + threadIdx.x);
        // the knots of every ancestor, in G's column order (block b = level m - b)
        for (int c = threadIdx.x; c < Pg; c += CFT) {
            const int b = c / rh, k = m - b;
            const long long akid = lvl_first(tp.J, k) + (t >> (tp.lj * (m - k)));
            knots_s[c] = ldpt(tp.kxy + 2 * akid * rh, c - b * rh);
        }
        __syncthreads();
        double* Gr = wp.G + (o0 - wp.G_base) * wp.ldG;
        // work items (column c, run of 16 rows): consecutive threads take consecutive columns (coalesced stores),
        // the knot sits in registers for the whole run and the point is a broadcast shared load; a 64-row tile of
        // Pg = 9 x 64 columns is 2304 items = 9 per thread
        const int nch = (n + 15) >> 4;
        for (int it = threadIdx.x; it < Pg * nch; it += CFT) {
            const int ch = it / Pg, c = it - ch * Pg;
            const double2 q = knots_s[c];
            const int i1 = min(16 * ch + 16, n);
            double* out = Gr + (long long)(16 * ch) * wp.ldG + c;
#pragma unroll 4
            for (int i = 16 * ch; i < i1; i++, out += wp.ldG) {
                const double2 pp = pts_s[i];
                *out = covf(cp, pp.x, pp.y, q.x, q.y);
            }
        }
        for (int r = threadIdx.x; r < n; r += CFT) Gr[(long long)r * wp.ldG + Pg] = tp.zs[o0 + r];
    }
}









// ------------------------------------------------------------------------ launchers
int smem_bytes() { return SMEM_DBL * (int)sizeof(double); }
int resident_ctas_per_sm();

// per host thread: a plan is single-entrant and a call runs on the calling thread, so the difference of this
// counter around a call is exactly that call's launches even when other threads drive other plans
thread_local unsigned long long g_kernel_launches = 0;

void phase_cycles(unsigned long long* out32, bool reset) {
    cudaMemcpyFromSymbol(out32, g_phase_cycles, sizeof(unsigned long long) * 32);
    if (reset) {
        unsigned long long z[32] = {0};
        cudaMemcpyToSymbol(g_phase_cycles, z, sizeof z);
    }
}

// occupancy and the >48 KB dynamic-smem attribute are per device: cached per device ordinal (a plan may
// live on any device of the process, opts.device), computed once under a lock
constexpr int MAXDEV = 64;
struct DevAttrs {
    bool done = false;
    int resident[12] = {1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1};   // resident CTAs per SM x SM count
    int cf_prior = 1, cf_wide = 1;                             // covariance-fill grids
};
static DevAttrs g_dev_attrs[MAXDEV];
static std::mutex g_attr_mu;
static const DevAttrs& set_attrs() {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= MAXDEV) dev = 0;
    DevAttrs& A = g_dev_attrs[dev];
    std::lock_guard<std::mutex> lk(g_attr_mu);
    if (A.done) return A;
    const int b = smem_bytes();
    const void* ks[12] = {(const void*)k_bottom,      (const void*)k_bottom,      (const void*)k_bottom,
                          (const void*)k_smooth,      (const void*)k_bottom,       (const void*)k_bottom,
                          (const void*)k_bottom,       (const void*)k_bottom,       (const void*)k_bottom,
                          (const void*)k_bottom,       (const void*)k_bottom,       (const void*)k_predict};
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    for (int i = 0; i < 12; i++) {
        cudaFuncSetAttribute(ks[i], cudaFuncAttributeMaxDynamicSharedMemorySize, b);
        int per = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, ks[i], NT, b);
        A.resident[i] = (per > 0 ? per : 1) * nsm;
    }
    int per = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_prior_covfill, CFT, 0);
    A.cf_prior = (per > 0 ? per : 1) * nsm;
    per = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_wide_covfill, CFT, 0);
    A.cf_wide = (per > 0 ? per : 1) * nsm;
    A.done = true;
    return A;
}
void init_kernel_attrs_main() { set_attrs(); }

// persistent grid: never more CTAs than can be resident at once (they pull work from a queue)
static int clamp_grid(int grid, long long items, int kidx) {
    const int res = set_attrs().resident[kidx];
    if (grid > res) grid = res;
    if (items < grid) grid = (int)items;
    return grid;
}

cudaError_t launch_gather(const double* z, const long long* perm, double* zs, long long N, cudaStream_t st) {
    long long blocks = (N + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    if (blocks < 1) blocks = 1;
    ++g_kernel_launches;
    k_gather<<<(int)blocks, 256, 0, st>>>(z, perm, zs, N);
    return cudaGetLastError();
}
cudaError_t launch_scatter(const double* zs, const long long* perm, double* z, long long N, cudaStream_t st) {
    long long blocks = (N + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    if (blocks < 1) blocks = 1;
    ++g_kernel_launches;
    k_scatter<<<(int)blocks, 256, 0, st>>>(zs, perm, z, N);
    return cudaGetLastError();
}
cudaError_t launch_pack_exchange(const double* out, long long ns, int q, const double* d, const double* u,
                                 const int* err, double* xbuf, cudaStream_t st) {
    const long long n = ns * (long long)q * (q + 1) / 2 + 2 * ns + 1;
    const long long blocks = std::min<long long>(4096, (n + 255) / 256);
    ++g_kernel_launches;
    k_pack_exchange<<<(int)blocks, 256, 0, st>>>(out, ns, q, d, u, err, xbuf);
    return cudaGetLastError();
}
cudaError_t launch_unpack_exchange(const double* xbuf, long long ns, int q, double* out, double* d, double* u,
                                   cudaStream_t st) {
    const long long n = ns * (long long)q * (q + 1) / 2 + 2 * ns;
    const long long blocks = std::min<long long>(4096, (n + 255) / 256);
    ++g_kernel_launches;
    k_unpack_exchange<<<(int)blocks, 256, 0, st>>>(xbuf, ns, q, out, d, u);
    return cudaGetLastError();
}
cudaError_t launch_fill(double* p, long long n, double v, cudaStream_t st) {
    long long blocks = (n + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    if (blocks < 1) blocks = 1;
    ++g_kernel_launches;
    k_fill<<<(int)blocks, 256, 0, st>>>(p, n, v);
    return cudaGetLastError();
}
cudaError_t launch_prior(const TreeParams& tp, const TmaReg& reg, int m, long long t_first, long long t_count, int grid,
                         double* ws, long long ws_stride, unsigned long long* counter, cudaStream_t st) {
    if (t_count > 0) {
        const int cf_grid = set_attrs().cf_prior;
        ++g_kernel_launches;
        k_prior_covfill<<<(int)std::min<long long>(cf_grid, t_count), CFT, 0, st>>>(tp, m, t_first, t_count);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return launch_prior_unit(tp, reg, m, t_first, t_count, grid, ws, ws_stride, counter, st);
}
cudaError_t launch_bottom(const TreeParams& tp, long long g_first, long long g_count, double* out, long long out_first,
                          int q, int grid, double* ws, const WsLayout& L, unsigned long long* counter,
                          cudaStream_t st) {
    set_attrs();
    grid = clamp_grid(grid, g_count, 1);
    if (grid < 1) return cudaSuccess;
    ++g_kernel_launches;
    k_bottom<<<grid, NT, smem_bytes(), st>>>(tp, g_first, g_count, out, out_first, q, ws, L, counter);
    return cudaGetLastError();
}
cudaError_t launch_final(const TreeParams& tp, double N, double* d_loglik, cudaStream_t st) {
    ++g_kernel_launches;
    k_final<<<1, 32, 0, st>>>(tp, N, d_loglik);
    return cudaGetLastError();
}
cudaError_t launch_mu(const TreeParams& tp, int m, double* muhat, double* mu, long long t_first, long long t_count,
                      cudaStream_t st) {
    if (t_count < 1) return cudaSuccess;
    int grid = (int)(t_count < 4096 ? t_count : 4096);
    ++g_kernel_launches;
    k_mu<<<grid, 64, 0, st>>>(tp, m, muhat, mu, t_first, t_count);
    return cudaGetLastError();
}
cudaError_t launch_smooth(const TreeParams& tp, const double* muhat, const long long* perm, double* smooth, int grid,
                          double* ws, const WsLayout& L, unsigned long long* counter, long long l_first,
                          long long l_count, cudaStream_t st) {
    set_attrs();
    grid = clamp_grid(grid, l_count, 3);
    if (grid < 1) return cudaSuccess;
    ++g_kernel_launches;
    k_smooth<<<grid, NT, smem_bytes(), st>>>(tp, muhat, perm, smooth, ws, L, counter, l_first, l_count);
    return cudaGetLastError();
}

}  // namespace mra

namespace mra {
// the wide-path phase that runs outside the GEMM unit: 6 = covariance fill (no engine)
// (launch_wide in mra_kernels_gemm.cu forwards them here)
cudaError_t launch_wide_main(int phase, const TreeParams& tp, const WideParams& wp, int step, const int4* tasks,
                             long long ntask, int grid, unsigned long long* counter, cudaStream_t st) {
    set_attrs();
    grid = clamp_grid(grid, ntask, phase == 6 ? 4 : 4 + phase);
    if (grid < 1) return cudaSuccess;
    const int b = smem_bytes();
    switch (phase) {
        case 6: {
            const int cf_grid = set_attrs().cf_wide;
            ++g_kernel_launches;
            k_wide_covfill<<<(int)std::min<long long>(cf_grid, ntask), CFT, 0, st>>>(tp, wp, tasks, ntask);
            break;
        }
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}
}  // namespace mra



namespace mra {
cudaError_t launch_predict(const TreeParams& tp, const PredParams& pp, int grid, double* ws, const WsLayout& L,
                           unsigned long long* counter, cudaStream_t st) {
    set_attrs();
    grid = clamp_grid(grid, pp.n_leaves, 11);
    if (grid < 1) return cudaSuccess;
    ++g_kernel_launches;
    k_predict<<<grid, NT, smem_bytes(), st>>>(tp, pp, ws, L, counter);
    return cudaGetLastError();
}
}  // namespace mra

namespace mra {
// resident CTAs per SM of the engine kernels (occupancy of k_bottom at the engine's smem size)
int resident_ctas_per_sm() {
    int per = 1;
    cudaFuncSetAttribute(k_bottom, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_bottom, NT, smem_bytes());
    return per > 0 ? per : 1;
}
}  // namespace mra
