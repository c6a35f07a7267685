// mra_device.cuh -- CTA-level fp64 building blocks for the MRA hot path on sm_100a.
//
// Everything here is executed by one CTA of NT = 256 threads on matrices that live in
// global memory (L2-resident per-CTA workspaces) and are staged through shared memory:
//   cta_gemm      C = init + alpha * sum_seg opA(seg) opB(seg)^T, 64x64 output tiles,
//                 fp64 tensor-core MMA (mma.sync.m8n8k4.f64 -> DMMA), operands either
//                 loaded from memory (row- or column-contiguous) or GENERATED on the fly
//                 as covariance blocks C(P, Q) (fused covariance generation)
//   chol_small    in-smem Cholesky of an n <= 64 block (+ log-determinant)
//   trinv_small   in-smem inverse of an n <= 64 lower-triangular block
//   chol_blocked  right-looking blocked Cholesky of an n x n global matrix (64-wide panels),
//                 keeps the inverted diagonal blocks for the triangular solves
//   fwd_subst     G <- L^{-1} G with the blocked factor (GEMM updates + inverted diagonals)
// fp64 is the method's precision; tcgen05 has no f64 kind, so the fp64
// tensor path on sm_100a is the warp-level DMMA.
#pragma once
#include <cstdint>

namespace mra {

constexpr int NT = 256;         // threads per CTA (8 warps)
constexpr int TM = 64;          // output tile rows
constexpr int TN = 64;          // output tile cols
constexpr int TK = 32;          // K per smem stage
constexpr int LDN = 36;         // smem ld of a [row][k] tile (== 4 mod 16 -> conflict-free frags)
constexpr int LDT = 68;         // smem ld of a [k][row] tile (== 4 mod 16)
constexpr int TILE_DBL = 2304;  // max(64*36, 32*68) doubles per operand tile
constexpr int LDB = 65;         // smem ld of a 64x64 factor block

enum Kind { MEMN = 0, MEMT = 1, COVK = 2 };

// covariance parameters (exponential / Matern-3/2), planar Euclidean distance
struct CovP {
    int kind;
    double s2, rho, xs, ys;
};

// one logical operand of size rows x K:
//   MEMN: X[i][k] = p[i*ld + k]     MEMT: X[i][k] = p[k*ld + i]
//   COVK: X[i][k] = C((rx[i], ry[i]), (cx[k], cy[k]))
struct Op {
    const double* p;
    long long ld;
    const double *rx, *ry, *cx, *cy;
};

// epilogue initial value: ZERO, MEM (p[i*ld+j], may alias C), COV (+ diag on i == j)
struct CInit {
    int kind;  // 0 zero, 1 mem, 2 cov
    const double* p;
    long long ld;
    const double *rx, *ry, *cx, *cy;
    double diag;
};

__device__ __forceinline__ Op op_mem(const double* p, long long ld) {
    Op o; o.p = p; o.ld = ld; o.rx = o.ry = o.cx = o.cy = nullptr; return o;
}
__device__ __forceinline__ Op op_cov(const double* rx, const double* ry, const double* cx, const double* cy) {
    Op o; o.p = nullptr; o.ld = 0; o.rx = rx; o.ry = ry; o.cx = cx; o.cy = cy; return o;
}
__device__ __forceinline__ CInit ci_zero() {
    CInit c; c.kind = 0; c.p = nullptr; c.ld = 0; c.rx = c.ry = c.cx = c.cy = nullptr; c.diag = 0; return c;
}
__device__ __forceinline__ CInit ci_mem(const double* p, long long ld) {
    CInit c = ci_zero(); c.kind = 1; c.p = p; c.ld = ld; return c;
}
__device__ __forceinline__ CInit ci_cov(const double* rx, const double* ry, const double* cx, const double* cy, double diag) {
    CInit c = ci_zero(); c.kind = 2; c.rx = rx; c.ry = ry; c.cx = cx; c.cy = cy; c.diag = diag; return c;
}

__device__ __forceinline__ double covf(const CovP& c, double x1, double y1, double x2, double y2) {
    double dx = (x1 - x2) * c.xs, dy = (y1 - y2) * c.ys;
    double d = sqrt(dx * dx + dy * dy);
    if (c.kind == 0) return c.s2 * exp(-d / c.rho);
    double a = 1.7320508075688772935 * d / c.rho;
    return c.s2 * (1.0 + a) * exp(-a);
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// stage rows [r0, r0+nr) x k [k0, k0+nk) of an operand into smem (zero-padded to 64 x 32)
template <int KIND>
__device__ __forceinline__ void load_tile(double* s, const Op& op, int r0, int nr, int k0, int nk,
                                          const CovP& cp) {
    const int tid = threadIdx.x;
    if (KIND == MEMT) {
#pragma unroll 4
        for (int e = tid; e < TM * TK; e += NT) {
            int kk = e >> 6, row = e & 63;
            double v = 0.0;
            if (row < nr && kk < nk) v = op.p[(long long)(k0 + kk) * op.ld + r0 + row];
            s[kk * LDT + row] = v;
        }
    } else if (KIND == MEMN) {
#pragma unroll 4
        for (int e = tid; e < TM * TK; e += NT) {
            int row = e >> 5, kk = e & 31;
            double v = 0.0;
            if (row < nr && kk < nk) v = op.p[(long long)(r0 + row) * op.ld + k0 + kk];
            s[row * LDN + kk] = v;
        }
    } else {
#pragma unroll 2
        for (int e = tid; e < TM * TK; e += NT) {
            int row = e >> 5, kk = e & 31;
            double v = 0.0;
            if (row < nr && kk < nk)
                v = covf(cp, op.rx[r0 + row], op.ry[r0 + row], op.cx[k0 + kk], op.cy[k0 + kk]);
            s[row * LDN + kk] = v;
        }
    }
}

template <int KIND>
__device__ __forceinline__ double frag(const double* s, int row, int k) {
    return KIND == MEMT ? s[k * LDT + row] : s[row * LDN + k];
}

// accumulate one K-segment into the warp's 16x32 sub-tile of output tile (r0, c0)
template <int KA, int KB>
__device__ __forceinline__ void gemm_segment(double (&acc)[2][4][2], const Op& A, const Op& B, int K,
                                             int r0, int nr, int c0, int nc, const CovP& cp,
                                             double* As, double* Bs) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int wr = (warp >> 1) * 16, wc = (warp & 1) * 32;
    for (int k0 = 0; k0 < K; k0 += TK) {
        const int nk = min(TK, K - k0);
        __syncthreads();
        load_tile<KA>(As, A, r0, nr, k0, nk, cp);
        load_tile<KB>(Bs, B, c0, nc, k0, nk, cp);
        __syncthreads();
        const int nk4 = (nk + 3) & ~3;
        for (int kk = 0; kk < nk4; kk += 4) {
            double a[2], b[4];
#pragma unroll
            for (int mi = 0; mi < 2; mi++) a[mi] = frag<KA>(As, wr + mi * 8 + g, kk + t);
#pragma unroll
            for (int ni = 0; ni < 4; ni++) b[ni] = frag<KB>(Bs, wc + ni * 8 + g, kk + t);
#pragma unroll
            for (int mi = 0; mi < 2; mi++)
#pragma unroll
                for (int ni = 0; ni < 4; ni++) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
        }
    }
}

// C[Mr x Nc] = init + alpha * (A0 B0^T [K0] + A1 B1^T [K1]); lower != 0 -> only i >= j written.
// In-place use (C aliasing the operands / init) is safe when every output tile reads only its own
// rows (A side) / columns (B side) of the aliased region -- see DESIGN.md §5.
template <int KA0, int KB0, int KA1, int KB1>
__device__ void cta_gemm(int Mr, int Nc, int lower, const Op& A0, const Op& B0, int K0, const Op& A1,
                         const Op& B1, int K1, const CInit& ci, double alpha, double* C, long long ldc,
                         const CovP& cp, double* smem) {
    double* As = smem;
    double* Bs = smem + TILE_DBL;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int wr = (warp >> 1) * 16, wc = (warp & 1) * 32;
    const int tiles_m = (Mr + TM - 1) / TM, tiles_n = (Nc + TN - 1) / TN;
    for (int tm = 0; tm < tiles_m; tm++) {
        for (int tn = 0; tn < tiles_n; tn++) {
            if (lower && tn > tm) continue;
            const int r0 = tm * TM, c0 = tn * TN;
            const int nr = min(TM, Mr - r0), nc = min(TN, Nc - c0);
            double acc[2][4][2];
#pragma unroll
            for (int mi = 0; mi < 2; mi++)
#pragma unroll
                for (int ni = 0; ni < 4; ni++) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
            if (K0 > 0) gemm_segment<KA0, KB0>(acc, A0, B0, K0, r0, nr, c0, nc, cp, As, Bs);
            if (K1 > 0) gemm_segment<KA1, KB1>(acc, A1, B1, K1, r0, nr, c0, nc, cp, As, Bs);
#pragma unroll
            for (int mi = 0; mi < 2; mi++)
#pragma unroll
                for (int ni = 0; ni < 4; ni++)
#pragma unroll
                    for (int e = 0; e < 2; e++) {
                        const int i = r0 + wr + mi * 8 + g, j = c0 + wc + ni * 8 + 2 * t + e;
                        if (i < Mr && j < Nc && (!lower || j <= i)) {
                            double v;
                            if (ci.kind == 0) v = 0.0;
                            else if (ci.kind == 1) v = ci.p[(long long)i * ci.ld + j];
                            else v = covf(cp, ci.rx[i], ci.ry[i], ci.cx[j], ci.cy[j]) + (i == j ? ci.diag : 0.0);
                            C[(long long)i * ldc + j] = v + alpha * acc[mi][ni][e];
                        }
                    }
        }
    }
    __syncthreads();
}

// ---------------------------------------------------------------- small factor blocks
// a: smem n x n (ld LDB), lower Cholesky in place; returns log|A| in *logdet (all threads);
// sets *bad (smem flag) if not positive definite. diagv: smem scratch [64].
__device__ void chol_small(double* a, int n, double* diagv, int* bad, double* red, double* logdet) {
    const int tid = threadIdx.x;
    for (int j = 0; j < n; j++) {
        const double ajj = a[j * LDB + j];
        const double ljj = sqrt(ajj > 0.0 ? ajj : 1.0);
        if (tid == 0) {
            if (!(ajj > 0.0)) *bad = 1;
            diagv[j] = ljj;
        }
        const double inv = 1.0 / ljj;
        for (int i = j + 1 + tid; i < n; i += NT) a[i * LDB + j] *= inv;
        __syncthreads();
        const int m = n - j - 1;
        for (int e = tid; e < m * m; e += NT) {
            const int ii = e / m, kk = e - ii * m;
            if (kk <= ii) a[(j + 1 + ii) * LDB + j + 1 + kk] -= a[(j + 1 + ii) * LDB + j] * a[(j + 1 + kk) * LDB + j];
        }
        __syncthreads();
    }
    for (int j = tid; j < n; j += NT) a[j * LDB + j] = diagv[j];
    // log-determinant: warp 0 reduces 2 sum log L_jj
    if (tid < 32) {
        double s = 0.0;
        for (int j = tid; j < n; j += 32) s += log(diagv[j]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (tid == 0) *red = 2.0 * s;
    }
    __syncthreads();
    *logdet = *red;
    __syncthreads();
}

// x = L^{-1} (lower triangular, n <= 64), both in smem with ld LDB; upper part of x zeroed
__device__ void trinv_small(const double* L, double* x, int n) {
    const int tid = threadIdx.x;
    const int c = tid & 63, part = tid >> 6;  // 4 threads per column: part 0 computes, others zero-fill
    if (part == 0 && c < n) {
        for (int i = 0; i < c; i++) x[i * LDB + c] = 0.0;
        x[c * LDB + c] = 1.0 / L[c * LDB + c];
        for (int i = c + 1; i < n; i++) {
            double s = 0.0;
            for (int k = c; k < i; k++) s += L[i * LDB + k] * x[k * LDB + c];
            x[i * LDB + c] = -s / L[i * LDB + i];
        }
    }
    __syncthreads();
}

// smem layout (doubles): [ main: GEMM tiles | factor blocks ] [ misc: 32 doubles ]
//   factor view of main: blk[64*LDB] | inv[64*LDB] | diag[64]
//   misc: red[0..15] (reductions) | bad flag (int) at misc+16 | work item at misc+18
constexpr int FAC_DBL = 2 * 64 * LDB + 64;
constexpr int MAIN_DBL = (FAC_DBL > 2 * TILE_DBL) ? FAC_DBL : 2 * TILE_DBL;
constexpr int SMEM_DBL = MAIN_DBL + 32;
struct FacSmem {
    double* blk;
    double* inv;
    double* diagv;
    double* red;
    int* bad;
};
__device__ __forceinline__ double* misc_smem(double* smem) { return smem + MAIN_DBL; }
__device__ __forceinline__ FacSmem fac_smem(double* smem) {
    FacSmem f;
    f.blk = smem;
    f.inv = smem + 64 * LDB;
    f.diagv = smem + 2 * 64 * LDB;
    f.red = misc_smem(smem);
    f.bad = reinterpret_cast<int*>(misc_smem(smem) + 16);
    return f;
}

// load lower n x n block of global A (ld) into blk; add `shift` to the diagonal
__device__ __forceinline__ void load_block_lower(double* blk, const double* A, long long ld, int n, double shift) {
    for (int e = threadIdx.x; e < 64 * 64; e += NT) {
        int i = e >> 6, j = e & 63;
        if (i < n && j <= i) blk[i * LDB + j] = A[(long long)i * ld + j] + (i == j ? shift : 0.0);
    }
    __syncthreads();
}
// store lower part of blk (n x n) to global (upper part untouched)
__device__ __forceinline__ void store_block_lower(const double* blk, double* A, long long ld, int n) {
    for (int e = threadIdx.x; e < 64 * 64; e += NT) {
        int i = e >> 6, j = e & 63;
        if (i < n && j <= i) A[(long long)i * ld + j] = blk[i * LDB + j];
    }
}
// store full n x n of x (upper zeros included) to global
__device__ __forceinline__ void store_block_full(const double* x, double* A, long long ld, int n) {
    for (int e = threadIdx.x; e < 64 * 64; e += NT) {
        int i = e >> 6, j = e & 63;
        if (i < n && j < n) A[(long long)i * ld + j] = x[i * LDB + j];
    }
}

// Blocked right-looking Cholesky of S (n x n, lower, ld) in place; Dinv receives the inverted
// 64x64 diagonal blocks (block b at Dinv + b*4096, ld 64). Returns log|S| (all threads).
__device__ double chol_blocked(double* S, int n, long long ld, double* Dinv, const CovP& cp, double* smem) {
    FacSmem f = fac_smem(smem);
    double total = 0.0;
    for (int j0 = 0; j0 < n; j0 += 64) {
        const int nb = min(64, n - j0);
        load_block_lower(f.blk, S + (long long)j0 * ld + j0, ld, nb, 0.0);
        double ldet;
        chol_small(f.blk, nb, f.diagv, f.bad, f.red, &ldet);
        total += ldet;
        trinv_small(f.blk, f.inv, nb);
        double* Di = Dinv + (long long)(j0 / 64) * 4096;
        store_block_lower(f.blk, S + (long long)j0 * ld + j0, ld, nb);
        store_block_full(f.inv, Di, 64, nb);
        __syncthreads();
        const int r = n - j0 - nb;
        if (r > 0) {
            double* P = S + (long long)(j0 + nb) * ld + j0;
            // panel: L_ij = A_ij L_jj^{-T}  (in place, single column tile)
            cta_gemm<MEMN, MEMN, MEMN, MEMN>(r, nb, 0, op_mem(P, ld), op_mem(Di, 64), nb, op_mem(P, ld),
                                             op_mem(P, ld), 0, ci_zero(), 1.0, P, ld, cp, smem);
            // trailing: A_ik -= L_ij L_kj^T (lower tiles, in place)
            double* T = S + (long long)(j0 + nb) * ld + j0 + nb;
            cta_gemm<MEMN, MEMN, MEMN, MEMN>(r, r, 1, op_mem(P, ld), op_mem(P, ld), nb, op_mem(P, ld),
                                             op_mem(P, ld), 0, ci_mem(T, ld), -1.0, T, ld, cp, smem);
        }
    }
    return total;
}

// G (n x ncol, ld ldg) <- L^{-1} G with the blocked factor of chol_blocked
__device__ void fwd_subst(const double* S, int n, long long ld, const double* Dinv, double* G, int ncol,
                          long long ldg, const CovP& cp, double* smem) {
    for (int i0 = 0; i0 < n; i0 += 64) {
        const int nb = min(64, n - i0);
        double* Gi = G + (long long)i0 * ldg;
        if (i0 > 0)
            cta_gemm<MEMN, MEMT, MEMN, MEMN>(nb, ncol, 0, op_mem(S + (long long)i0 * ld, ld), op_mem(G, ldg), i0,
                                             op_mem(G, ldg), op_mem(G, ldg), 0, ci_mem(Gi, ldg), -1.0, Gi, ldg,
                                             cp, smem);
        cta_gemm<MEMN, MEMT, MEMN, MEMN>(nb, ncol, 0, op_mem(Dinv + (long long)(i0 / 64) * 4096, 64),
                                         op_mem(Gi, ldg), nb, op_mem(G, ldg), op_mem(G, ldg), 0, ci_zero(), 1.0,
                                         Gi, ldg, cp, smem);
    }
}

// CTA-wide sum (result valid in all threads)
__device__ __forceinline__ double cta_sum(double v, double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0) {
        for (int w = 0; w < NT / 32; w++) s += red[w];
        red[8] = s;
    }
    __syncthreads();
    s = red[8];
    __syncthreads();
    return s;
}

}  // namespace mra
