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
#include <type_traits>
#ifdef MRA_BULK
#include "mra_internal.h"   // TmaReg
#endif

#ifndef MRA_NT
#define MRA_NT 256
#endif
#ifndef MRA_TK
#define MRA_TK 32
#endif
#ifndef MRA_NSTAGE
#define MRA_NSTAGE 3
#endif
// every engine shape gets its own inline namespace, so translation units built with different shapes
// (mra_kernels.cu, mra_kernels_gemm.cu) can be linked into one library
#define MRA_ENG_NS_(a, b, c) eng_##a##_##b##_##c
#define MRA_ENG_NS_X(a, b, c) MRA_ENG_NS_(a, b, c)
#define MRA_ENG_NS MRA_ENG_NS_X(MRA_NT, MRA_TK, MRA_NSTAGE)

namespace mra {
inline namespace MRA_ENG_NS {
constexpr int NT = MRA_NT;      // threads per CTA: 8 warps of 16 x 32 sub-tiles, 2 CTAs per SM (default);
                                // -DMRA_NT=128 -DMRA_MINB=3 -DMRA_NSTAGE=2: 4 warps of 32 x 32, 3 CTAs per SM
                                // (faster GEMM main loop, slower latency-bound phases: DESIGN.md §5)
constexpr int TM = 64;          // output tile rows
constexpr int TN = 64;          // output tile cols
constexpr int NWARP = NT / 32;
constexpr int WN = 32;                      // warp sub-tile columns
constexpr int WM = 64 / (NWARP / (64 / WN));   // warp sub-tile rows (32 for 4 warps, 16 for 8)
constexpr int MI = WM / 8;                  // 8-row DMMA blocks per warp
static_assert(NWARP * WM * WN == 64 * 64, "warp tiling");
#ifndef MRA_TK
#define MRA_TK 32
#endif
static_assert(MRA_TK % 8 == 0 && MRA_TK <= 64, "stage depth");
constexpr int TK = MRA_TK;      // K per smem stage
constexpr int LDN = TK + 4;     // smem ld of a [row][k] tile (== 4 mod 16 -> conflict-free frags)
constexpr int LDT = 68;         // smem ld of a [k][row] tile (== 4 mod 16)
constexpr int TILE_DBL = (64 * LDN > TK * LDT) ? 64 * LDN : TK * LDT;   // doubles per operand tile
constexpr int LDB = 65;         // smem ld of a 64x64 factor block

enum Kind { MEMN = 0, MEMT = 1, COVK = 2 };

// covariance parameters (exponential / Matern-3/2), planar Euclidean distance; ir = 1/rho
// (exponential) or sqrt(3)/rho (Matern-3/2), precomputed so the per-entry path has no division
struct CovP {
    int kind;
    double s2, rho, xs, ys, ir;
};

// one logical operand of size rows x K (points are interleaved (x, y) pairs):
//   MEMN: X[i][k] = p[i*ld + k]     MEMT: X[i][k] = p[k*ld + i]
//   COVK: X[i][k] = C(p[2i], p[2i+1]; q[2k], q[2k+1])
struct Op {
    const double* p;
    const double* q;
    long long ld;
};

// epilogue initial value: ZERO, MEM (p[i*ld+j], may alias C), COV C(p_i, q_j) (+ diag on i == j)
struct CInit {
    int kind;  // 0 zero, 1 mem, 2 cov
    const double* p;
    const double* q;
    long long ld;
    double diag;
};

__device__ __forceinline__ Op op_mem(const double* p, long long ld) {
    Op o; o.p = p; o.q = nullptr; o.ld = ld; return o;
}
__device__ __forceinline__ Op op_cov(const double* rowpts, const double* kpts) {
    Op o; o.p = rowpts; o.q = kpts; o.ld = 0; return o;
}
__device__ __forceinline__ CInit ci_zero() {
    CInit c; c.kind = 0; c.p = nullptr; c.q = nullptr; c.ld = 0; c.diag = 0; return c;
}
__device__ __forceinline__ CInit ci_mem(const double* p, long long ld) {
    CInit c = ci_zero(); c.kind = 1; c.p = p; c.ld = ld; return c;
}
__device__ __forceinline__ CInit ci_cov(const double* rowpts, const double* colpts, double diag) {
    CInit c = ci_zero(); c.kind = 2; c.p = rowpts; c.q = colpts; c.diag = diag; return c;
}
__device__ __forceinline__ double2 ldpt(const double* pts, int i) {
    return reinterpret_cast<const double2*>(pts)[i];
}

// e^{-x} for x >= 0 with a short dependency chain (libm exp is ~204 dependent cycles on B200,
// tools/bench_fp64ops.cu); e^{-x} < 1e-307 is flushed to 0.
//   e^{-x} = 2^{-e} 2^{-j/32} e^{-r},  k = rint(32 x / ln 2) = 32 e + j,  r = x - k ln2/32 in [-ln2/64, ln2/64]
// (Cody-Waite split of ln2/32: the high part has 32 significant bits, exact for k < 2^21); e^{-r} by its
// degree-6 Taylor polynomial (truncation < 3.5e-18) as e^{-r} - 1; 2^{-j/32} from a 32-entry table
// (L1-resident, read with __ldg). About 16 fp64 operations (the degree-12 form without the table took
// 23); max error measured by tools/check_exp.cu.
static __device__ const double g_exp2m32[32] = {
    1.0, 0.9785720620877001, 0.9576032806985737, 0.93708381705515,
    0.9170040432046712, 0.8973545375015536, 0.8781260801866497, 0.859309649061239,
    0.8408964152537145, 0.8228777390769825, 0.8052451659746271, 0.7879904225539432,
    0.7711054127039704, 0.7545822137967114, 0.7384130729697497, 0.7225904034885233,
    0.7071067811865476, 0.691954940981916, 0.6771277734684463, 0.6626183215798707,
    0.6484197773255048, 0.6345254785958666, 0.620928906036742, 0.6076236799902345,
    0.5946035575013605, 0.5818624293887887, 0.5693943173783458, 0.5571933712979462,
    0.5452538663326288, 0.5335702003384118, 0.5221368912137069, 0.5109485743270583};
__device__ __forceinline__ double exp_neg(double x) {
    // branch-free (one basic block, so the unrolled callers interleave independent chains): x >= 708 (and NaN)
    // run the same arithmetic (meaningless there, the table index stays in range) and 0 is selected at the end
    const bool big = !(x < 708.0);
    const double K32 = 46.166241308446828384,                          // 32 / ln 2
        LN2_32_HI = 6.93147180369123816490e-01 / 32, LN2_32_LO = 1.90821492927058770002e-10 / 32,
        MAGIC = 6755399441055744.0;
    const double kt = __dadd_rn(__dmul_rn(x, K32), MAGIC);          // MAGIC + rint(32 x / ln 2)
    const double kd = kt - MAGIC;                                      // rint(32 x / ln 2)
    double s = fma(kd, LN2_32_HI, -x);                               // s = -r
    s = fma(kd, LN2_32_LO, s);
    // w = e^s - 1 = s + s^2 (1/2 + s/6 + s^2 (1/24 + s/120 + s^2/720)); the result t (1 + w) is rounded
    // once, so only t's own rounding and that final fma reach the last bits
    const double s2 = s * s;
    const double a = fma(1.0 / 6, s, 0.5), b = fma(1.0 / 120, s, 1.0 / 24);
    const double c = fma(1.0 / 720, s2, b);
    const double u = fma(c, s2, a);
    const double w = fma(u, s2, s);
    const int k = __double2loint(kt);   // = (int) kd: the integer sits in the low word (no conversion instruction)
    const double t = __ldg(g_exp2m32 + (k & 31));
    const double r = fma(t, w, t) * __hiloint2double((1023 - (k >> 5)) << 20, 0);
    return big ? 0.0 : r;
}

// sqrt(q) from the single-precision MUFU reciprocal square root, one fp64 Newton step on 1/sqrt and one
// Heron correction on sqrt: ~8 dependent operations instead of the libm routine (<= 1 ulp; equal to
// the correctly rounded sqrt on 2e7 random q in [1e-30, 1e6] in a host check). Branch-free (selects only, so
// that unrolled callers interleave independent chains): q below 2^-120 is scaled by 2^240 first (exact) and the
// result by 2^-120; q == 0 gives 0. Every q >= 2^-120 takes exactly the unscaled arithmetic.
__device__ __forceinline__ double sqrt_fast(double q) {
    const bool small = q < 0x1p-120;
    const double qs = small ? q * 0x1p240 : q;
    // q == 0: a finite seed, the result is replaced below; 0 < q < 2^-366 (distances below 1e-55) returns a value
    // below 2^-180 instead of the root (no covariance can tell the two apart)
    const float qf = fmaxf(__double2float_rn(qs), 0x1p-126f);
    double y = (double)rsqrtf(qf);
    y = y * fma(-0.5 * qs, y * y, 1.5);
    const double d = qs * y;
    const double r = fma(0.5 * y, fma(-d, d, qs), d);
    return q == 0.0 ? 0.0 : (small ? r * 0x1p-120 : r);
}

__device__ __forceinline__ double covf(const CovP& c, double x1, double y1, double x2, double y2) {
    const double dx = (x1 - x2) * c.xs, dy = (y1 - y2) * c.ys;
    const double a = sqrt_fast(dx * dx + dy * dy) * c.ir;
    const double e = exp_neg(a);
    // exponential: s2 e = (s2 * 1) e; Matern-3/2: s2 (1 + a) e -- one expression, the kind a loop-invariant factor
    const double m = c.kind == 0 ? 0.0 : 1.0;
    return c.s2 * fma(a, m, 1.0) * e;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// compile-time loop: f(integral_constant<int, I>) for I in [B, E)
template <int B, int E, typename F>
__device__ __forceinline__ void sfor(F&& f) {
    if constexpr (B < E) {
        f(std::integral_constant<int, B>());
        sfor<B + 1, E>(f);
    }
}

// ------------------------------------------------------------- async tile staging
#ifndef MRA_NSTAGE
#define MRA_NSTAGE 3
#endif
constexpr int NSTAGE = MRA_NSTAGE;         // cp.async pipeline depth
constexpr int STAGE_DBL = 2 * TILE_DBL;    // A tile + B tile

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
// 8-byte async copy global -> smem; src_bytes 0 zero-fills (the source is not read)
__device__ __forceinline__ void cp_async8(double* s, const double* g, int src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(s)), "l"(g), "r"(src_bytes));
}
// 16-byte async copy (L2 only); src_bytes in {0, 8, 16}, the rest zero-filled
__device__ __forceinline__ void cp_async16(double* s, const double* g, int src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(s)), "l"(g), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ bool op_aligned16(const Op& op) {
    return ((reinterpret_cast<uintptr_t>(op.p) & 15) == 0) && ((op.ld & 1) == 0);
}

// stage rows [r0, r0+nr) x k [k0, k0+nk) of an operand into smem (zero-padded to 64 x TK).
// Memory operands go through cp.async (16-byte copies when aligned); covariance operands are
// generated in registers (fused covariance generation) and stored.
template <int KIND>
__device__ __forceinline__ void load_tile_async(double* s, const Op& op, int r0, int nr, int k0, int nk,
                                                const CovP& cp, bool al16) {
    const int tid = threadIdx.x;
    if (KIND == MEMN) {
        if (al16) {
#pragma unroll
            for (int i = 0; i < 32 * TK / NT; i++) {   // 64 rows x TK/2 16-byte copies over NT threads
                const int e = tid + NT * i, row = e / (TK / 2), kk = (e % (TK / 2)) * 2;
                const int ok = (row < nr) ? min(2, max(0, nk - kk)) : 0;
                const double* g = ok ? op.p + (long long)(r0 + row) * op.ld + k0 + kk : op.p;
                cp_async16(s + row * LDN + kk, g, ok * 8);
            }
        } else {
#pragma unroll
            for (int i = 0; i < 64 * TK / NT; i++) {
                const int e = tid + NT * i, row = e / TK, kk = e % TK;
                const bool ok = row < nr && kk < nk;
                cp_async8(s + row * LDN + kk, ok ? op.p + (long long)(r0 + row) * op.ld + k0 + kk : op.p, ok ? 8 : 0);
            }
        }
    } else if (KIND == MEMT) {
        if (al16) {
#pragma unroll 2
            for (int i = 0; i < 32 * TK / NT; i++) {
                const int e = tid + NT * i, kk = e >> 5, row = (e & 31) * 2;
                const int ok = (kk < nk) ? min(2, max(0, nr - row)) : 0;
                const double* g = ok ? op.p + (long long)(k0 + kk) * op.ld + r0 + row : op.p;
                cp_async16(s + kk * LDT + row, g, ok * 8);
            }
        } else {
#pragma unroll
            for (int i = 0; i < 64 * TK / NT; i++) {
                const int e = tid + NT * i, kk = e >> 6, row = e & 63;
                const bool ok = row < nr && kk < nk;
                cp_async8(s + kk * LDT + row, ok ? op.p + (long long)(k0 + kk) * op.ld + r0 + row : op.p, ok ? 8 : 0);
            }
        }
    } else {
        const int kk = tid % TK, rw = tid / TK;
        const CovP cpl = cp;   // one copy into registers per stage (cp may live in shared memory)
        const bool kok = kk < nk;
        const double2 qk = kok ? ldpt(op.q, k0 + kk) : make_double2(0.0, 0.0);
#pragma unroll 4
        for (int i = 0; i < 64 * TK / NT; i++) {
            const int row = rw + (NT / TK) * i;
            // unconditional chain on a clamped (valid) row, select after: no branch splits the unrolled chains
            const double2 pr = ldpt(op.p, r0 + min(row, max(nr - 1, 0)));
            const double v = covf(cpl, pr.x, pr.y, qk.x, qk.y);
            s[row * LDN + kk] = (kok && row < nr) ? v : 0.0;
        }
    }
}

// LAY 1: the layouts TMA tensor loads produce (GEMM unit, MODE 3): MEMN [64 rows][16 k] with the 128-byte swizzle
// (16-byte chunk index ^= row & 7), MEMT [8 row octets][16 k][8 rows]; both conflict-free for the fragment loads
template <int KIND, int LAY = 0>
__device__ __forceinline__ double frag(const double* s, int row, int k) {
    if (LAY == 1)
        return KIND == MEMT ? s[(row >> 3) * 128 + k * 8 + (row & 7)]
                            : s[row * 16 + ((((k >> 1) ^ (row & 7)) << 1) | (k & 1))];
    return KIND == MEMT ? s[k * LDT + row] : s[row * LDN + k];
}

// MI x 4 DMMAs per k-step of 4 on the warp's WM x 32 sub-tile
// MASK: the ragged k-tile's fragments with k >= nk are zeroed (the bulk-copy path leaves stale values there; the
// cp.async path zero-fills, MASK = false)
// tri (TRI instantiations only: the Sigma tiles, EPI = 1): the warp's sub-tile sits on the diagonal of a lower-triangular
// output tile (WM == WN): the 8 x 8 blocks strictly above the diagonal are not needed (the epilogue never stores
// them), so their DMMAs are not issued -- the SM's fp64 pipe is shared by the co-resident CTAs, which get that
// time. (Compiled into every instantiation, the branch slowed the others by a few % through code size.)
template <int KA, int KB, bool MASK, int LAY, bool TRI, int MV>
__device__ __forceinline__ void mma_ktile_v(double (&acc)[MI][4][2], const double* As, const double* Bs, int nk,
                                            bool tri) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int wr = (warp / (64 / WN)) * WM, wc = (warp % (64 / WN)) * WN;
    auto step = [&](int kk) {
        double a[MV], b[4];
#pragma unroll
        for (int mi = 0; mi < MV; mi++) a[mi] = frag<KA, LAY>(As, wr + mi * 8 + g, kk + t);
#pragma unroll
        for (int ni = 0; ni < 4; ni++) b[ni] = frag<KB, LAY>(Bs, wc + ni * 8 + g, kk + t);
        if (TRI && WM == WN && tri) {
#pragma unroll
            for (int mi = 0; mi < MV; mi++)
#pragma unroll
                for (int ni = 0; ni < 4; ni++)
                    if (ni <= mi) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
        } else {
#pragma unroll
            for (int mi = 0; mi < MV; mi++)
#pragma unroll
                for (int ni = 0; ni < 4; ni++) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
        }
    };
    if (nk == TK) {
#pragma unroll
        for (int kk = 0; kk < TK; kk += 4) step(kk);
    } else if (!MASK) {
        const int nk4 = (nk + 3) & ~3;
        for (int kk = 0; kk < nk4; kk += 4) step(kk);
    } else {
        const int nk4 = (nk + 3) & ~3;
        for (int kk = 0; kk < nk4; kk += 4) {
            const bool kin = kk + t < nk;
            double a[MV], b[4];
#pragma unroll
            for (int mi = 0; mi < MV; mi++) a[mi] = kin ? frag<KA, LAY>(As, wr + mi * 8 + g, kk + t) : 0.0;
#pragma unroll
            for (int ni = 0; ni < 4; ni++) b[ni] = kin ? frag<KB, LAY>(Bs, wc + ni * 8 + g, kk + t) : 0.0;
#pragma unroll
            for (int mi = 0; mi < MV; mi++)
#pragma unroll
                for (int ni = 0; ni < 4; ni++)
                    if (!(TRI && WM == WN && tri) || ni <= mi) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
        }
    }
}

// act (cta_gemm_impl): bits 0-1 active / on the diagonal of a lower tile, bits 2-4 how many of the warp's 8-row
// blocks hold wanted rows. RAG: a warp whose wanted rows (a ragged last row tile) lie in the first half of its row
// blocks runs a second unrolled body without the other half's DMMAs (a branch: predicated-off DMMAs still occupy
// the pipe; one extra body, not one per count, to keep the code instruction-cache resident)
template <int KA, int KB, bool MASK = false, int LAY = 0, bool TRI = false, bool RAG = false>
__device__ __forceinline__ void mma_ktile(double (&acc)[MI][4][2], const double* As, const double* Bs, int nk,
                                          int act) {
    const bool tri = (act & 3) == 2;
    if constexpr (RAG) {
        if (2 * ((act >> 2) & 7) <= MI && !(TRI && tri)) {
            mma_ktile_v<KA, KB, MASK, LAY, false, MI / 2>(acc, As, Bs, nk, false);
            return;
        }
    }
    mma_ktile_v<KA, KB, MASK, LAY, TRI, MI>(acc, As, Bs, nk, tri);
}

// MI x 4 DMMAs per k-step of 4 on the warp's WM x 32 sub-tile
// MASK: the ragged k-tile's fragments with k >= nk are zeroed (the bulk-copy path leaves stale values there; the
// cp.async path zero-fills, MASK = false)
// tri (TRI instantiations only: the Sigma tiles, EPI = 1): the warp's sub-tile sits on the diagonal of a lower-triangular
// output tile (WM == WN): the 8 x 8 blocks strictly above the diagonal are not needed (the epilogue never stores
// them), so their DMMAs are not issued -- the SM's fp64 pipe is shared by the co-resident CTAs, which get that
// time. (Compiled into every instantiation, the branch slowed the others by a few % through code size.)
// NV: 8-column blocks of the warp's sub-tile (4; 2 for the two half-width warps of a balanced diagonal tile); the
// sub-tile's origin (wr, wc) comes from cta_gemm_impl
template <int KA, int KB, bool MASK, int LAY, bool TRI, int MV, int NV = 4>
__device__ __forceinline__ void mma_ktile_vb(double (&acc)[MI][4][2], const double* As, const double* Bs, int nk,
                                            bool tri, int wr, int wc) {
    const int lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    auto step = [&](int kk) {
        double a[MV], b[NV];
#pragma unroll
        for (int mi = 0; mi < MV; mi++) a[mi] = frag<KA, LAY>(As, wr + mi * 8 + g, kk + t);
#pragma unroll
        for (int ni = 0; ni < NV; ni++) b[ni] = frag<KB, LAY>(Bs, wc + ni * 8 + g, kk + t);
        if (TRI && WM == WN && tri) {
#pragma unroll
            for (int mi = 0; mi < MV; mi++)
#pragma unroll
                for (int ni = 0; ni < NV; ni++)
                    if (ni <= mi) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
        } else {
#pragma unroll
            for (int mi = 0; mi < MV; mi++)
#pragma unroll
                for (int ni = 0; ni < NV; ni++) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
        }
    };
    if (nk == TK) {
#pragma unroll
        for (int kk = 0; kk < TK; kk += 4) step(kk);
    } else if (!MASK) {
        const int nk4 = (nk + 3) & ~3;
        for (int kk = 0; kk < nk4; kk += 4) step(kk);
    } else {
        const int nk4 = (nk + 3) & ~3;
        for (int kk = 0; kk < nk4; kk += 4) {
            const bool kin = kk + t < nk;
            double a[MV], b[NV];
#pragma unroll
            for (int mi = 0; mi < MV; mi++) a[mi] = kin ? frag<KA, LAY>(As, wr + mi * 8 + g, kk + t) : 0.0;
#pragma unroll
            for (int ni = 0; ni < NV; ni++) b[ni] = kin ? frag<KB, LAY>(Bs, wc + ni * 8 + g, kk + t) : 0.0;
#pragma unroll
            for (int mi = 0; mi < MV; mi++)
#pragma unroll
                for (int ni = 0; ni < NV; ni++)
                    if (!(TRI && WM == WN && tri) || ni <= mi) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
        }
    }
}

// act (cta_gemm_impl): bits 0-1 active (1) / on the diagonal of a lower tile (2) / half-width sub-tile of a balanced
// diagonal tile (3), bits 2-4 how many of the warp's 8-row blocks hold wanted rows, bits 5-7 / 8-10 the sub-tile's
// row / column origin in 8-blocks. RAG: a warp whose wanted rows (a ragged last row tile) lie in the first half of its row
// blocks runs a second unrolled body without the other half's DMMAs (a branch: predicated-off DMMAs still occupy
// the pipe; one extra body, not one per count, to keep the code instruction-cache resident)
template <int KA, int KB, bool MASK = false, int LAY = 0, bool TRI = false, bool RAG = false>
__device__ __forceinline__ void mma_ktile_bal(double (&acc)[MI][4][2], const double* As, const double* Bs, int nk,
                                          int act) {
    const bool tri = (act & 3) == 2;
    int wr, wc;
    if constexpr (TRI && WM == 32 && NWARP == 4) {   // the sub-tile origin travels in act (balanced diagonal tiles)
        wr = ((act >> 5) & 7) * 8;
        wc = ((act >> 8) & 7) * 8;
    } else {
        const int warp = threadIdx.x >> 5;
        wr = (warp / (64 / WN)) * WM;
        wc = (warp % (64 / WN)) * WN;
    }
    if constexpr (TRI && WM == 32 && NWARP == 4) {
        if ((act & 3) == 3) {
            mma_ktile_vb<KA, KB, MASK, LAY, false, MI, 2>(acc, As, Bs, nk, false, wr, wc);
            return;
        }
    }
    if constexpr (RAG) {
        if (2 * ((act >> 2) & 7) <= MI && !(TRI && (act & 3) >= 2)) {
            mma_ktile_vb<KA, KB, MASK, LAY, false, MI / 2>(acc, As, Bs, nk, false, wr, wc);
            return;
        }
    }
    mma_ktile_vb<KA, KB, MASK, LAY, TRI, MI>(acc, As, Bs, nk, tri, wr, wc);
}

// k-tile body: the balanced-diagonal one (sub-tile origin in act) for cta_gemm_impl_bal, the plain one otherwise
template <bool BALD, int KA, int KB, bool MASK, int LAY, bool TRI, bool RAG>
__device__ __forceinline__ void mma_ktile_sel(double (&acc)[MI][4][2], const double* As, const double* Bs, int nk,
                                              int act) {
    if constexpr (BALD) mma_ktile_bal<KA, KB, MASK, LAY, TRI, RAG>(acc, As, Bs, nk, act);
    else mma_ktile<KA, KB, MASK, LAY, TRI, RAG>(acc, As, Bs, nk, act);
}

// the ragged-row body where it pays: not in the merge-tile GEMMs (G^T G and -F F^T: their rows are whole tiles
// but for the one y row, and the extra body cost mtile 2 %)
template <int KA0, int KB0, int KA1, int KB1>
__host__ __device__ constexpr bool rag_of() { return !(KA0 == MEMT && KB0 == MEMT && KA1 == MEMN && KB1 == MEMN); }

// GEMM call descriptor: written to shared memory by the (inlined) caller, read by the single
// non-inlined implementation per operand-kind combination (keeps the kernels' SASS small enough
// to stay instruction-cache resident).
struct GemmDesc {
    Op A0, B0, A1, B1;
    CInit ci;
    CovP cp;
    double alpha;
    double* C;
    long long ldc;
    int Mr, Nc, lower, K0, K1;
    int amask;   // staging mode of the call (GEMM unit: 0 cp.async, 1 bulk copies, 3 TMA tensor loads)
    int ti[4], trow[4], tcol[4];   // TMA (MODE 3): registry entry and buffer coordinates of operand o
};
#ifdef MRA_BULK
constexpr int MISC_DBL = 256;                // misc smem (2 KB, so the main area is 1024-byte aligned for the swizzled
                                             // TMA stages): reductions, flags, work item, GemmDesc, BulkState, and
                                             // (from 128) the registry's buffer table (RegMeta[TMA_NREG])
#else
constexpr int MISC_DBL = 64;                 // misc smem: reductions, flags, work item, GemmDesc
#endif
__device__ __forceinline__ GemmDesc* gemm_desc(double* smem);

#ifdef MRA_BULK
// ------------------------------------------------------------ bulk-copy staging (GEMM unit)
// A transposed operand (MEMT: X[i][k] = p[k ld + i]) has each k-row of a tile contiguous in memory, so its
// 64 x TK k-tile is TK 1-D bulk copies (cp.async.bulk, the TMA unit, <= 512 B each) into the padded [k][LDT]
// layout, completing on an mbarrier transaction count -- no per-thread cp.async issue and, when every operand
// of a call is staged this way, no CTA barrier per k-tile (full / empty barriers per stage instead). No tensor
// map is involved. Row-major operands (MEMN, 128-byte k-rows: too small for the bulk engine, 46 % of the fp64
// peak in tools/bench_bulk2.cu) stay on cp.async. The per-CTA state persists across the GEMM calls of a kernel
// (engine_init).
struct BulkState {
    unsigned long long full[NSTAGE], empty[NSTAGE];   // all-bulk / all-TMA pipelines
    const TmaReg* reg;                                // the kernel's tensor-map registry (param space), or nullptr
    unsigned gs;                                      // k-tiles staged so far by the barrier pipelines
    unsigned pad;
};
__device__ __forceinline__ BulkState* bulk_state(double* smem);
__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n"
                 ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(double* dst, const double* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool bulk_ok(const Op& op) {
    return ((reinterpret_cast<uintptr_t>(op.p) & 15) == 0) && ((op.ld & 1) == 0) && op.ld > 0;
}
// bytes of one MEMT k-tile: nk k-rows of the rows [r0, r0 + nr) rounded up to an even count (16-byte multiple;
// the extra double is past the operand's last row: plan buffers carry slack, its value is never used)
__device__ __forceinline__ unsigned bulk_bytes(int nr, int nk) { return (unsigned)(nk * ((nr + 1) & ~1) * 8); }
// warp 0: copy the k-rows [k0, k0 + nk) of rows [r0, r0 + nr) of a MEMT operand into s ([k][LDT])
__device__ __forceinline__ void bulk_tile_t(double* s, const Op& op, int r0, int nr, int k0, int nk,
                                            unsigned long long* bar) {
    const int lane = threadIdx.x & 31;
    const unsigned rb = (unsigned)(((nr + 1) & ~1) * 8);
    for (int k = lane; k < nk; k += 32) bulk_g2s(s + k * LDT, op.p + (long long)(k0 + k) * op.ld + r0, rb, bar);
}
__device__ __forceinline__ void tma_load2(double* dst, const CUtensorMap* map, int c0, int c1, unsigned long long* bar) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
                 ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_load3(double* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                          unsigned long long* bar) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
                 ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)) : "memory");
}
// the registry's buffer table, copied to shared memory by engine_init (a lookup per GEMM call reads it there,
// not the kernel parameter: parameters beyond 4 KB are fetched through global memory)
struct RegMeta {
    unsigned long long base, end;
    long long ld;
    int kind, n;   // n: entries (valid in element 0)
};
__device__ __forceinline__ RegMeta* reg_meta(double* smem);
// registry entry of an operand (kind matching, inside the buffer, the buffer's row stride), its buffer row and
// column; a MEMT operand must start on a column octet. -1: not registered
template <int KIND>
__device__ __forceinline__ int tma_find(const RegMeta* rm, const Op& op, int* row, int* col) {
    if (KIND != MEMN && KIND != MEMT) return -1;
    const unsigned long long p = reinterpret_cast<unsigned long long>(op.p);
    const int kd = KIND == MEMT ? 1 : 0;
    const int n = rm[0].n;
    for (int i = 0; i < n; i++) {
        if (rm[i].kind != kd || rm[i].ld != op.ld || p < rm[i].base || p >= rm[i].end) continue;
        const unsigned long long off = p - rm[i].base;
        if (off & 7) return -1;
        const long long e = (long long)(off >> 3), r = e / op.ld, c = e % op.ld;
        if ((KIND == MEMT && (c & 7)) || r > 0x7fffffffLL) return -1;
        *row = (int)r;
        *col = (int)c;
        return i;
    }
    return -1;
}
// one operand k-tile by TMA (thread 0): MEMN box (16 k, 64 rows) at (col + k0, row + r0); MEMT box (8, 16, 8) at
// (0, row + k0, (col + r0) / 8)
template <int KIND>
__device__ __forceinline__ void tma_tile(double* dst, const TmaReg* reg, int ti, int trow, int tcol, int r0, int k0,
                                         unsigned long long* bar) {
    if (KIND == MEMN) tma_load2(dst, &reg->map[ti], tcol + k0, trow + r0, bar);
    else tma_load3(dst, &reg->map[ti], 0, trow + k0, (tcol + r0) >> 3, bar);
}
#endif

// accumulate both K-segments of one output tile through an NSTAGE-deep cp.async pipeline
template <int KA0, int KB0, int KA1, int KB1, bool TRI = false, bool BALD = false>
__device__ __forceinline__ void tile_pipeline(double (&acc)[MI][4][2], const GemmDesc& d, int r0, int nr, int c0,
                                              int nc, double* smem, int wact) {
    // only the current segment's two operand descriptors are held in registers (segment 1's are read
    // from the shared-memory GemmDesc when the loads reach it): the engine sits at the 128-register
    // budget of two 256-thread CTAs per SM
    const int K0 = d.K0, K1 = d.K1, T0 = (K0 + TK - 1) / TK, T = T0 + (K1 + TK - 1) / TK;
    Op a = d.A0, b = d.B0;
    bool aal = op_aligned16(a), bal = op_aligned16(b);
    __syncthreads();   // the stage buffers (and any smem view aliasing them) are free
    // single issue site: iterations kt < 0 only prefetch (pipeline prologue)
#pragma unroll 1
    for (int kt = -(NSTAGE - 1); kt < T; kt++) {
        if (kt >= 0) {
            cp_async_wait<NSTAGE - 2>();
            __syncthreads();
        }
        const int ki = kt + NSTAGE - 1;
        if (ki < T) {
            double* As = smem + (ki % NSTAGE) * STAGE_DBL;
            double* Bs = As + TILE_DBL;
            if (ki < T0) {
                const int k0 = ki * TK, nk = min(TK, K0 - k0);
                load_tile_async<KA0>(As, a, r0, nr, k0, nk, d.cp, aal);
                load_tile_async<KB0>(Bs, b, c0, nc, k0, nk, d.cp, bal);
            } else {
                if (ki == T0) {
                    a = d.A1; b = d.B1;
                    aal = op_aligned16(a); bal = op_aligned16(b);
                }
                const int k0 = (ki - T0) * TK, nk = min(TK, K1 - k0);
                load_tile_async<KA1>(As, a, r0, nr, k0, nk, d.cp, aal);
                load_tile_async<KB1>(Bs, b, c0, nc, k0, nk, d.cp, bal);
            }
        }
        cp_async_commit();
        if (kt < 0) continue;
        if (!(wact & 3)) continue;   // this warp's sub-tile holds no wanted output (it still loads)
        const double* As = smem + (kt % NSTAGE) * STAGE_DBL;
        const double* Bs = As + TILE_DBL;
        if (kt < T0) mma_ktile_sel<BALD, KA0, KB0, false, 0, TRI, rag_of<KA0, KB0, KA1, KB1>()>(acc, As, Bs, min(TK, K0 - kt * TK), wact);
        else mma_ktile_sel<BALD, KA1, KB1, false, 0, TRI, rag_of<KA0, KB0, KA1, KB1>()>(acc, As, Bs, min(TK, K1 - (kt - T0) * TK), wact);
    }
    cp_async_wait<0>();
}

#ifdef MRA_BULK
// every operand of the call is a bulk-staged MEMT: warp 0 keeps NSTAGE - 1 k-tiles in flight (lane 0 waits for a
// stage's empty barrier and posts the byte count, the lanes issue the k-row copies), every warp waits on the
// stage's full barrier, runs its DMMAs and arrives on the empty barrier
template <int KA0, int KB0, int KA1, int KB1, bool TRI = false, bool BALD = false>
__device__ __forceinline__ void tile_pipeline_bulk(double (&acc)[MI][4][2], const GemmDesc& d, int r0, int nr, int c0,
                                                   int nc, double* smem, int wact, unsigned gs) {
    BulkState* bs = bulk_state(smem);
    const int K0 = d.K0, K1 = d.K1, T0 = (K0 + TK - 1) / TK, T = T0 + (K1 + TK - 1) / TK;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    auto issue = [&](int ki) {
        const unsigned sidx = gs + ki, b = sidx % NSTAGE, n = sidx / NSTAGE;
        const bool s0 = ki < T0;
        const int k0 = (s0 ? ki : ki - T0) * TK, nk = min(TK, (s0 ? K0 : K1) - k0);
        if (lane == 0) {
            if (n > 0) mbar_wait(&bs->empty[b], (n - 1) & 1);
            mbar_expect_tx(&bs->full[b], bulk_bytes(nr, nk) + bulk_bytes(nc, nk));
        }
        __syncwarp();
        double* As = smem + b * STAGE_DBL;
        bulk_tile_t(As, s0 ? d.A0 : d.A1, r0, nr, k0, nk, &bs->full[b]);
        bulk_tile_t(As + TILE_DBL, s0 ? d.B0 : d.B1, c0, nc, k0, nk, &bs->full[b]);
    };
    if (warp == 0)
        for (int ki = 0; ki < NSTAGE - 1 && ki < T; ki++) issue(ki);
#pragma unroll 1
    for (int kt = 0; kt < T; kt++) {
        if (warp == 0 && kt + NSTAGE - 1 < T) issue(kt + NSTAGE - 1);
        const unsigned sidx = gs + kt, b = sidx % NSTAGE;
        mbar_wait(&bs->full[b], (sidx / NSTAGE) & 1);
        if (wact & 3) {
            const double* As = smem + b * STAGE_DBL;
            const double* Bs = As + TILE_DBL;
            if (kt < T0) mma_ktile_sel<BALD, KA0, KB0, true, 0, TRI, rag_of<KA0, KB0, KA1, KB1>()>(acc, As, Bs, min(TK, K0 - kt * TK), wact);
            else mma_ktile_sel<BALD, KA1, KB1, true, 0, TRI, rag_of<KA0, KB0, KA1, KB1>()>(acc, As, Bs, min(TK, K1 - (kt - T0) * TK), wact);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&bs->empty[b]);
    }
}

// every operand of the call lies in a registered buffer: thread 0 keeps NSTAGE - 1 k-tiles in flight, one TMA tensor
// load per operand k-tile (16 KB per stage); full / empty barriers as the bulk pipeline; ragged k-tiles masked (the
// boxes read the buffer's next columns / rows there)
template <int KA0, int KB0, int KA1, int KB1, bool TRI = false, bool BALD = false>
__device__ __forceinline__ void tile_pipeline_tma(double (&acc)[MI][4][2], const GemmDesc& d, int r0, int c0,
                                                  double* smem, int wact, unsigned gs) {
    BulkState* bs = bulk_state(smem);
    const TmaReg* reg = bs->reg;
    const int K0 = d.K0, K1 = d.K1, T0 = (K0 + TK - 1) / TK, T = T0 + (K1 + TK - 1) / TK;
    const int lane = threadIdx.x & 31;
    auto issue = [&](int ki) {
        const unsigned sidx = gs + ki, b = sidx % NSTAGE, n = sidx / NSTAGE;
        if (n > 0) mbar_wait(&bs->empty[b], (n - 1) & 1);
        mbar_expect_tx(&bs->full[b], 2u * 64 * 16 * 8);
        double* As = smem + b * STAGE_DBL;
        if (ki < T0) {
            tma_tile<KA0>(As, reg, d.ti[0], d.trow[0], d.tcol[0], r0, ki * TK, &bs->full[b]);
            tma_tile<KB0>(As + TILE_DBL, reg, d.ti[1], d.trow[1], d.tcol[1], c0, ki * TK, &bs->full[b]);
        } else {
            tma_tile<KA1>(As, reg, d.ti[2], d.trow[2], d.tcol[2], r0, (ki - T0) * TK, &bs->full[b]);
            tma_tile<KB1>(As + TILE_DBL, reg, d.ti[3], d.trow[3], d.tcol[3], c0, (ki - T0) * TK, &bs->full[b]);
        }
    };
    if (threadIdx.x == 0)
        for (int ki = 0; ki < NSTAGE - 1 && ki < T; ki++) issue(ki);
#pragma unroll 1
    for (int kt = 0; kt < T; kt++) {
        if (threadIdx.x == 0 && kt + NSTAGE - 1 < T) issue(kt + NSTAGE - 1);
        __syncwarp();
        const unsigned sidx = gs + kt, b = sidx % NSTAGE;
        mbar_wait(&bs->full[b], (sidx / NSTAGE) & 1);
        if (wact & 3) {
            const double* As = smem + b * STAGE_DBL;
            const double* Bs = As + TILE_DBL;
            if (kt < T0) mma_ktile_sel<BALD, KA0, KB0, true, 1, TRI, rag_of<KA0, KB0, KA1, KB1>()>(acc, As, Bs, min(TK, K0 - kt * TK), wact);
            else mma_ktile_sel<BALD, KA1, KB1, true, 1, TRI, rag_of<KA0, KB0, KA1, KB1>()>(acc, As, Bs, min(TK, K1 - (kt - T0) * TK), wact);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&bs->empty[b]);
    }
}
#endif

// EPI = 1: the epilogue can add a covariance initial value (ci_cov); only the instantiations that need it
// carry that code (it costs the other GEMMs registers: at 128 the MEMT x MEMT one would spill)
// MODE (GEMM unit): 0 cp.async only, 1 every operand a bulk-copied MEMT, 3 every operand in the TMA registry (a call
// mixing kinds stages everything by cp.async); separate
// non-inlined instantiations, so the paths do not share a register allocation
template <int KA0, int KB0, int KA1, int KB1, int EPI, int MODE>
__device__ __noinline__ void cta_gemm_impl(double* smem) {
    const GemmDesc& d = *gemm_desc(smem);
    const int Mr = d.Mr, Nc = d.Nc, lower = d.lower, K0 = d.K0, K1 = d.K1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int wr = (warp / (64 / WN)) * WM, wc = (warp % (64 / WN)) * WN;
    const int tiles_m = (Mr + TM - 1) / TM, tiles_n = (Nc + TN - 1) / TN;
#ifdef MRA_BULK
    BulkState* bs = bulk_state(smem);
    unsigned gs = bs->gs;
    if (MODE != 0) {
        __syncthreads();   // the stage area's previous users are done before the bulk engine writes it
        if (threadIdx.x < 32) {
            // order earlier generic writes of the operands (this CTA's, and through the caller's acquire other
            // CTAs') and of the stage area before the async-proxy copies
            asm volatile("fence.proxy.async.global;\n" ::: "memory");
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        }
    }
#endif
    for (int tm = 0; tm < tiles_m; tm++) {
        for (int tn = 0; tn < tiles_n; tn++) {
            if (lower && tn > tm) continue;
            const int r0 = tm * TM, c0 = tn * TN;
            const int nr = min(TM, Mr - r0), nc = min(TN, Nc - c0);
            double acc[MI][4][2];
#pragma unroll
            for (int mi = 0; mi < MI; mi++)
#pragma unroll
                for (int ni = 0; ni < 4; ni++) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
            // warps whose sub-tile lies outside a ragged tile (e.g. the 1-row y tile) or strictly above the
            // diagonal of a lower-triangular tile skip their DMMAs
            // 0: the warp's sub-tile holds no wanted output; 1: active; 2: active on the diagonal of a lower tile
            // (bits 2-4: how many of its 8-row blocks hold wanted rows, mma_ktile)
            const int wact = (wr < nr && wc < nc && !(lower && tm == tn && wc > wr + WM - 1))
                                 ? ((WM == WN && lower && tm == tn && wr == wc) ? 2 : 1) | (min(MI, (nr - wr + 7) >> 3) << 2)
                                 : 0;
#ifdef MRA_BULK
            if (MODE == 1) {
                tile_pipeline_bulk<KA0, KB0, KA1, KB1, EPI == 1>(acc, d, r0, nr, c0, nc, smem, wact, gs);
                gs += (K0 + TK - 1) / TK + (K1 + TK - 1) / TK;
            } else if (MODE == 3) {
                tile_pipeline_tma<KA0, KB0, KA1, KB1, EPI == 1>(acc, d, r0, c0, smem, wact, gs);
                gs += (K0 + TK - 1) / TK + (K1 + TK - 1) / TK;
            } else
#endif
            if (K0 + K1 > 0)
                tile_pipeline<KA0, KB0, KA1, KB1, EPI == 1>(acc, d, r0, nr, c0, nc, smem, wact);
            const CInit ci = d.ci;
            const double alpha = d.alpha;
            double* C = d.C;
            const long long ldc = d.ldc;
            // the (e = 0, 1) pair of a fragment is two adjacent columns: one 16-byte access when the
            // whole pair is in range and aligned
            const bool vec = ((reinterpret_cast<uintptr_t>(C) & 15) == 0) && ((ldc & 1) == 0) &&
                             (ci.kind != 1 || (((reinterpret_cast<uintptr_t>(ci.p) & 15) == 0) && ((ci.ld & 1) == 0)));
            if (EPI == 1 && ci.kind == 2) {
                // covariance initial value (Sigma tiles): C = alpha acc + (C(s_i, s_j) + diag), one store per element;
                // the covariance chains run unconditionally on clamped (valid) points and only the store is
                // predicated, so no branch splits the unrolled chains. A warp with nothing to store computes
                // nothing, and a warp on the diagonal of a diagonal tile only the 8 x 8 blocks on or below it (its
                // own straight-line body): the generation is a fifth of the Sigma tile's fp64-pipe time
                const CovP cpl = d.cp;
                auto cov_store = [&](auto diagc) {
                    constexpr bool DIAG = decltype(diagc)::value;
                    sfor<0, MI>([&](auto mic) {
                        constexpr int mi = decltype(mic)::value;
                        const int i = r0 + wr + mi * 8 + g;
                        const double2 pi = ldpt(ci.p, min(i, Mr - 1));
                        sfor<0, 8>([&](auto qc) {
                            constexpr int q = decltype(qc)::value, ni = q >> 1, e = q & 1;
                            if constexpr (!(DIAG && ni > mi)) {
                                const int j = c0 + wc + ni * 8 + 2 * t + e;
                                const double2 pj = ldpt(ci.q, min(j, Nc - 1));
                                const double w = covf(cpl, pi.x, pi.y, pj.x, pj.y) + (i == j ? ci.diag : 0.0);
                                if (i < Mr && j < Nc && (!lower || j <= i))
                                    C[(long long)i * ldc + j] = __dadd_rn(__dmul_rn(alpha, acc[mi][ni][e]), w);
                            }
                        });
                    });
                };
                if (wact & 3) {
                    if (WM == WN && lower && tm == tn && wr == wc) cov_store(std::true_type());
                    else cov_store(std::false_type());
                }
            } else
#pragma unroll
            for (int mi = 0; mi < MI; mi++)
#pragma unroll
                for (int ni = 0; ni < 4; ni++) {
                    const int i = r0 + wr + mi * 8 + g, j = c0 + wc + ni * 8 + 2 * t;
                    if (vec && i < Mr && j + 1 < Nc && (!lower || j + 1 <= i)) {
                        double2 v = make_double2(0.0, 0.0);
                        if (ci.kind == 1) v = *reinterpret_cast<const double2*>(ci.p + (long long)i * ci.ld + j);
                        *reinterpret_cast<double2*>(C + (long long)i * ldc + j) =
                            make_double2(v.x + alpha * acc[mi][ni][0], v.y + alpha * acc[mi][ni][1]);
                    } else {
#pragma unroll
                        for (int e = 0; e < 2; e++) {
                            const int jj = j + e;
                            if (i < Mr && jj < Nc && (!lower || jj <= i)) {
                                const double v = (ci.kind == 1) ? ci.p[(long long)i * ci.ld + jj] : 0.0;
                                C[(long long)i * ldc + jj] = v + alpha * acc[mi][ni][e];
                            }
                        }
                    }
                }
            if (EPI == 0 && ci.kind == 2) __trap();   // a covariance init needs the EPI = 1 instantiation
        }
    }
#ifdef MRA_BULK
    if (MODE != 0 && threadIdx.x == 0) bs->gs = gs;
#endif
    __syncthreads();
}

// EPI = 2 (the merge tiles' diagonal blocks): the TRI skip and the balanced diagonal tiles. A separate function, so
// that the other instantiations keep their register allocation (ptxas spilled the chain's TMA GEMM with the extra
// per-tile state compiled in). Measured on C3: merge tiles 576 -> 553 ms; on the Sigma tiles (EPI = 1) the extra
// bodies made the TMA k-loop spill and the balance did not pay (C2, all Sigma tiles diagonal: 3.2 -> 3.5 ms)
template <int KA0, int KB0, int KA1, int KB1, int EPI, int MODE>
__device__ __noinline__ void cta_gemm_impl_bal(double* smem) {
    const GemmDesc& d = *gemm_desc(smem);
    const int Mr = d.Mr, Nc = d.Nc, lower = d.lower, K0 = d.K0, K1 = d.K1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int tiles_m = (Mr + TM - 1) / TM, tiles_n = (Nc + TN - 1) / TN;
    constexpr bool TRI = EPI >= 1;   // the instantiations with the triangular DMMA skip
    constexpr bool BAL = TRI && WM == 32 && NWARP == 4;   // ... and the balanced diagonal tiles
    const int wr0 = (warp / (64 / WN)) * WM, wc0 = (warp % (64 / WN)) * WN;
#ifdef MRA_BULK
    BulkState* bs = bulk_state(smem);
    unsigned gs = bs->gs;
    if (MODE != 0) {
        __syncthreads();   // the stage area's previous users are done before the bulk engine writes it
        if (threadIdx.x < 32) {
            // order earlier generic writes of the operands (this CTA's, and through the caller's acquire other
            // CTAs') and of the stage area before the async-proxy copies
            asm volatile("fence.proxy.async.global;\n" ::: "memory");
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        }
    }
#endif
    for (int tm = 0; tm < tiles_m; tm++) {
        for (int tn = 0; tn < tiles_n; tn++) {
            if (lower && tn > tm) continue;
            const int r0 = tm * TM, c0 = tn * TN;
            const int nr = min(TM, Mr - r0), nc = min(TN, Nc - c0);
            // warp -> sub-tile. A diagonal tile of a lower output in the TRI instantiations (4 warps of 32 x 32) is
            // balanced: warps 0 / 3 take the two 32 x 32 diagonal sub-tiles (10 of 16 8 x 8 blocks each, the TRI skip),
            // warps 1 / 2 the two 32 x 16 halves of the sub-diagonal one (8 each) -- instead of one warp idle and one
            // at 16 blocks, which set the tile's time (each element is still accumulated in the same k order)
            const bool dtile = lower && tm == tn;
            const bool half = BAL && dtile && (warp == 1 || warp == 2);
            const int wr = half ? 32 : wr0, wc = half ? (warp == 1 ? 0 : 16) : wc0;
            const int nv = half ? 2 : 4;   // 8-column blocks of the warp's sub-tile
            double acc[MI][4][2];
#pragma unroll
            for (int mi = 0; mi < MI; mi++)
#pragma unroll
                for (int ni = 0; ni < 4; ni++) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
            // warps whose sub-tile lies outside a ragged tile (e.g. the 1-row y tile) or strictly above the
            // diagonal of a lower-triangular tile skip their DMMAs
            // 0: the warp's sub-tile holds no wanted output; 1: active; 2: active on the diagonal of a lower tile
            // (bits 2-4: how many of its 8-row blocks hold wanted rows, mma_ktile)
            const int wact = (wr < nr && wc < nc && !(dtile && wc > wr + WM - 1))
                                 ? (half ? 3 : (WM == WN && dtile && wr == wc) ? 2 : 1) |
                                       (min(MI, (nr - wr + 7) >> 3) << 2) | (BAL ? ((wr >> 3) << 5) | ((wc >> 3) << 8) : 0)
                                 : 0;
#ifdef MRA_BULK
            if (MODE == 1) {
                tile_pipeline_bulk<KA0, KB0, KA1, KB1, TRI, true>(acc, d, r0, nr, c0, nc, smem, wact, gs);
                gs += (K0 + TK - 1) / TK + (K1 + TK - 1) / TK;
            } else if (MODE == 3) {
                tile_pipeline_tma<KA0, KB0, KA1, KB1, TRI, true>(acc, d, r0, c0, smem, wact, gs);
                gs += (K0 + TK - 1) / TK + (K1 + TK - 1) / TK;
            } else
#endif
            if (K0 + K1 > 0)
                tile_pipeline<KA0, KB0, KA1, KB1, TRI, true>(acc, d, r0, nr, c0, nc, smem, wact);
            const CInit ci = d.ci;
            const double alpha = d.alpha;
            double* C = d.C;
            const long long ldc = d.ldc;
            // the (e = 0, 1) pair of a fragment is two adjacent columns: one 16-byte access when the
            // whole pair is in range and aligned
            const bool vec = ((reinterpret_cast<uintptr_t>(C) & 15) == 0) && ((ldc & 1) == 0) &&
                             (ci.kind != 1 || (((reinterpret_cast<uintptr_t>(ci.p) & 15) == 0) && ((ci.ld & 1) == 0)));
            static_assert(EPI == 2, "the balanced impl serves the EPI = 2 instantiations");
#pragma unroll
            for (int mi = 0; mi < MI; mi++)
#pragma unroll
                for (int ni = 0; ni < 4; ni++) {
                    const int i = r0 + wr + mi * 8 + g, j = c0 + wc + ni * 8 + 2 * t;
                    if (BAL && ni >= nv) continue;   // a half-width sub-tile: the next columns are another warp's
                    if (vec && i < Mr && j + 1 < Nc && (!lower || j + 1 <= i)) {
                        double2 v = make_double2(0.0, 0.0);
                        if (ci.kind == 1) v = *reinterpret_cast<const double2*>(ci.p + (long long)i * ci.ld + j);
                        *reinterpret_cast<double2*>(C + (long long)i * ldc + j) =
                            make_double2(v.x + alpha * acc[mi][ni][0], v.y + alpha * acc[mi][ni][1]);
                    } else {
#pragma unroll
                        for (int e = 0; e < 2; e++) {
                            const int jj = j + e;
                            if (i < Mr && jj < Nc && (!lower || jj <= i)) {
                                const double v = (ci.kind == 1) ? ci.p[(long long)i * ci.ld + jj] : 0.0;
                                C[(long long)i * ldc + jj] = v + alpha * acc[mi][ni][e];
                            }
                        }
                    }
                }
            if (EPI != 1 && ci.kind == 2) __trap();   // a covariance init needs the EPI = 1 instantiation
        }
    }
#ifdef MRA_BULK
    if (MODE != 0 && threadIdx.x == 0) bs->gs = gs;
#endif
    __syncthreads();
}

template <int KA0, int KB0, int KA1, int KB1, int EPI, int MODE>
__device__ __forceinline__ void cta_gemm_impl_sel(double* smem) {
    if constexpr (EPI == 2) cta_gemm_impl_bal<KA0, KB0, KA1, KB1, EPI, MODE>(smem);
    else cta_gemm_impl<KA0, KB0, KA1, KB1, EPI, MODE>(smem);
}

// C[Mr x Nc] = init + alpha * (A0 B0^T [K0] + A1 B1^T [K1]); lower != 0 -> only i >= j written.
// In-place use (C aliasing the operands / init) is safe when every output tile reads only its own
// rows (A side) / columns (B side) of the aliased region -- see DESIGN.md §5.
template <int KA0, int KB0, int KA1, int KB1, int EPI = 0>
__device__ __forceinline__ void cta_gemm(int Mr, int Nc, int lower, const Op& A0, const Op& B0, int K0,
                                         const Op& A1, const Op& B1, int K1, const CInit& ci, double alpha,
                                         double* C, long long ldc, const CovP& cp, double* smem) {
    GemmDesc* d = gemm_desc(smem);
    __syncthreads();   // the previous descriptor is no longer read
    if (threadIdx.x == 0) {
        d->A0 = A0; d->B0 = B0; d->A1 = A1; d->B1 = B1;
        d->ci = ci; d->cp = cp; d->alpha = alpha; d->C = C; d->ldc = ldc;
        d->Mr = Mr; d->Nc = Nc; d->lower = lower; d->K0 = K0; d->K1 = K1;
    }
#ifdef MRA_BULK
    // staging mode, decided by thread 0 (uniform through the descriptor): 3 when every operand lies in a buffer of
    // the kernel's TMA registry (tensor loads), 1 when every operand is a 16-byte-aligned MEMT with an even ld (1-D
    // bulk copies), else 0 (cp.async)
    constexpr bool any_t = KA0 == MEMT || KB0 == MEMT || KA1 == MEMT || KB1 == MEMT;
    constexpr bool tk_ok = (KA0 == MEMN || KA0 == MEMT) && (KB0 == MEMN || KB0 == MEMT) &&
                           (KA1 == MEMN || KA1 == MEMT) && (KB1 == MEMN || KB1 == MEMT);
    if (threadIdx.x == 0) {
        int mode = 0;
        if (tk_ok && K0 + K1 > 0) {
            const RegMeta* reg = reg_meta(smem);
            bool tma = bulk_state(smem)->reg != nullptr;
            if (tma && K0 > 0) {
                d->ti[0] = tma_find<KA0>(reg, A0, &d->trow[0], &d->tcol[0]);
                d->ti[1] = tma_find<KB0>(reg, B0, &d->trow[1], &d->tcol[1]);
                tma = d->ti[0] >= 0 && d->ti[1] >= 0;
            }
            if (tma && K1 > 0) {
                d->ti[2] = tma_find<KA1>(reg, A1, &d->trow[2], &d->tcol[2]);
                d->ti[3] = tma_find<KB1>(reg, B1, &d->trow[3], &d->tcol[3]);
                tma = d->ti[2] >= 0 && d->ti[3] >= 0;
            }
            if (tma) mode = 3;
        }
        if (mode == 0 && any_t && K0 + K1 > 0) {
            bool ok = true;
            if (K0 > 0) ok = KA0 == MEMT && KB0 == MEMT && bulk_ok(A0) && bulk_ok(B0);
            if (ok && K1 > 0) ok = KA1 == MEMT && KB1 == MEMT && bulk_ok(A1) && bulk_ok(B1);
            if (ok) mode = 1;
        }
        d->amask = mode;
    }
    __syncthreads();
    const int mode = d->amask;
    if (tk_ok && mode == 3)
        cta_gemm_impl_sel<KA0, KB0, KA1, KB1, EPI, tk_ok ? 3 : 0>(smem);
    else if (any_t && mode == 1)
        cta_gemm_impl_sel<KA0, KB0, KA1, KB1, EPI, any_t ? 1 : 0>(smem);
    else
        cta_gemm_impl_sel<KA0, KB0, KA1, KB1, EPI, 0>(smem);
#else
    __syncthreads();
    cta_gemm_impl_sel<KA0, KB0, KA1, KB1, EPI, 0>(smem);
#endif
}

// ---------------------------------------------------------------- small factor blocks
// In-smem Cholesky + triangular inverse of an n <= 64 block, blocked by 16 so that the CTA
// synchronises ~20 times instead of twice per column:
//   per 16-block: warp 0 factors and inverts the diagonal block (warp-synchronous), all threads
//   form the panel L_ib = A_ib D_bb^{-T} and the trailing update A -= L_ib L_kb^T;
//   then X = L^{-1} is assembled block-row by block-row: X_ij = -X_ii sum_k L_ik X_kj.
// a: n x n (ld LDB), lower, overwritten by L. x: n x n (ld LDB) receives L^{-1} (upper part 0).
// x == a: in place -- a receives L^{-1} (upper part 0) and L itself is not kept: each diagonal block
// is replaced by its inverse as soon as it is factored (the panels need only the inverse), and the
// block-row assembly of the off-diagonal blocks reads row i of L before overwriting it (through tmp).
// tmp: >= 3*256 doubles of smem scratch. Returns log|A| (all threads); *bad set if not PD.
#ifdef MRA_CHOL_DEBUG
__device__ long long g_chol_dbg[16];
// phase k accumulates the cycles since the previous CHK (thread 0 of CTA 0)
#define CHK(k) do { const long long _t = clock64(); if (threadIdx.x == 0 && blockIdx.x == 0) g_chol_dbg[k] += _t - chk_last; chk_last = _t; } while (0)
#define CHK_START long long chk_last = clock64()
#else
#define CHK(k)
#define CHK_START
#endif
__device__ __noinline__ double chol_inv_small(double* a, double* x, int n, double* diagv, int* bad, double* red,
                                              double* tmp) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    CHK_START;
    const int nbk = (n + 15) >> 4;
    const bool inplace = (x == a);
    for (int e = tid; e < 64 * 64; e += NT) {
        const int i = e >> 6, j = e & 63;
        if (i < n && j < n && (!inplace || j > i)) x[i * LDB + j] = 0.0;
    }
    CHK(1);
    for (int b = 0; b < nbk; b++) {
        const int j0 = b * 16, nb = min(16, n - j0);
        if (warp == 0) {
            // 16 x 16 diagonal block: lane i keeps row i in registers (rows >= nb padded with the
            // identity); the pivot column is broadcast through shared memory (independent LDS, no
            // shuffle chains).
            const int i = lane & 15;
            double* d = a + j0 * LDB + j0;
            double r[16];
#pragma unroll
            for (int k = 0; k < 16; k++)
                r[k] = (i < nb && k < nb && k <= i) ? d[i * LDB + k] : (i == k ? 1.0 : 0.0);
            double dv[16];
            bool ok = true;
            // the lane's own running diagonal a_ii - sum_{j<i} l_ij^2, kept apart from r[] so that
            // the serial pivot chain is shuffle -> rsqrt -> scale -> fma per column (no smem trip);
            // the off-diagonal columns travel through a double-buffered smem column one step ahead.
            double dg = 1.0;
#pragma unroll
            for (int k = 0; k < 16; k++)
                if (i == k) dg = r[k];
#pragma unroll
            for (int j = 0; j < 16; j++) {
                const double piv = __shfl_sync(0xffffffffu, dg, j);
                ok = ok && (piv > 0.0);
                // one rsqrt on the serial pivot chain: 1/l_jj, then l_jj = piv / l_jj
                const double pv = piv > 0.0 ? piv : 1.0;
                const double il = rsqrt(pv);
                const double ljj = pv * il;
                dv[j] = il;
                const double lij = r[j] * il;
                r[j] = (i == j) ? ljj : ((i > j) ? lij : r[j]);
                if (i > j) dg -= lij * lij;
                double* col = tmp + 16 + 16 * (j & 1);
                if (lane < 16) col[i] = r[j];   // column j of L (l_ij for i > j)
                __syncwarp();
#pragma unroll
                for (int k = j + 1; k < 16; k++) {
                    const double lk = col[k];
                    if (i >= k) r[k] -= r[j] * lk;
                }
            }
            __syncwarp();
            CHK(6);
            if (!ok && lane == 0) *bad = 1;
            // publish L_bb rows to smem (lower part) for the inverse and the panel
            if (lane < nb) {
#pragma unroll
                for (int k = 0; k < 16; k++)
                    if (k <= i && k < nb) d[i * LDB + k] = r[k];
            }
            __syncwarp();
            // column `lane` of X_bb = L_bb^{-1}: x_i = (delta_ic - sum_{k<i} L_ik x_k) / L_ii
            const int c = lane & 15;
            double xc[16];
#pragma unroll
            for (int ii = 0; ii < 16; ii++) {
                double s0 = (ii == c) ? 1.0 : 0.0, s1 = 0.0;
                if (ii < nb) {
#pragma unroll
                    for (int k = 0; k + 1 < ii; k += 2) {
                        s0 -= d[ii * LDB + k] * xc[k];
                        s1 -= d[ii * LDB + k + 1] * xc[k + 1];
                    }
                    if (ii & 1) s0 -= d[ii * LDB + ii - 1] * xc[ii - 1];
                }
                xc[ii] = (s0 + s1) * dv[ii];
            }
            double* xd = x + j0 * LDB + j0;
            if (inplace) __syncwarp();   // every lane has read L_bb before X_bb replaces it
            if (lane < nb) {
#pragma unroll
                for (int k = 0; k < 16; k++)
                    if (k < nb) xd[k * LDB + c] = xc[k];
            }
        }
        CHK(2);
        __syncthreads();
        CHK(3);
        const int r0 = j0 + nb, nr = n - r0;
        if (nr > 0) {
#ifndef MRA_CHOL_SCALAR
            // panel L_ib = A_ib X_bb^T (rows r0..n-1, <= 48; the nb columns of block b) and trailing update
            // A_rc -= L_rb L_cb^T (lower part) as 8 x 8 DMMA tiles (m8n8k4, K = 16 masked to nb), warp-strided
            {
                const int g = lane >> 2, t = lane & 3, nw = NT / 32;
                const int rb = (nr + 7) >> 3, cbn = (nb + 7) >> 3;
                // the panel tiles go to the scratch first (every operand is read before A_ib is overwritten)
                for (int tsk = warp; tsk < rb * cbn; tsk += nw) {
                    const int m = tsk / cbn, cc = tsk % cbn;
                    double d0 = 0.0, d1 = 0.0;
#pragma unroll
                    for (int k0 = 0; k0 < 16; k0 += 4) {
                        const int k = k0 + t;
                        const double av = k < nb ? a[(r0 + 8 * m + g) * LDB + j0 + k] : 0.0;
                        const double bv = (k < nb && 8 * cc + g < nb) ? x[(j0 + 8 * cc + g) * LDB + j0 + k] : 0.0;
                        dmma(d0, d1, av, bv);
                    }
                    double* pt = tmp + (8 * m + g) * 16 + 8 * cc + 2 * t;
                    pt[0] = d0;
                    pt[1] = d1;
                }
                __syncthreads();
                for (int e = tid; e < nr * 16; e += NT) {
                    const int rr = e >> 4, c = e & 15;
                    if (c < nb) a[(r0 + rr) * LDB + j0 + c] = tmp[e];
                }
                __syncthreads();
                CHK(7);
                for (int tsk = warp; tsk < rb * (rb + 1) / 2; tsk += nw) {
                    int m = 0;
                    while ((m + 1) * (m + 2) / 2 <= tsk) m++;
                    const int cc = tsk - m * (m + 1) / 2;
                    double d0 = 0.0, d1 = 0.0;
#pragma unroll
                    for (int k0 = 0; k0 < 16; k0 += 4) {
                        const int k = k0 + t;
                        const double av = k < nb ? a[(r0 + 8 * m + g) * LDB + j0 + k] : 0.0;
                        const double bv = k < nb ? a[(r0 + 8 * cc + g) * LDB + j0 + k] : 0.0;
                        dmma(d0, d1, av, bv);
                    }
                    const int row = r0 + 8 * m + g, col = r0 + 8 * cc + 2 * t;
                    if (row < n) {
                        if (col <= row) a[row * LDB + col] -= d0;
                        if (col + 1 <= row) a[row * LDB + col + 1] -= d1;
                    }
                }
            }
#else
            // panel: L_ib = A_ib X_bb^T for rows r0..n-1 (<= 48), cols j0..j0+nb-1; thread = (row group, col)
            constexpr int RG = NT / 16, NQ = (48 + RG - 1) / RG;   // row groups per pass, passes over <= 48 rows
            const int jj = tid & 15, rg = tid >> 4;
            const double* xr = x + (j0 + jj) * LDB + j0;
            double v[NQ];
#pragma unroll
            for (int q = 0; q < NQ; q++) {
                const int row = r0 + rg + RG * q;
                double s0 = 0.0, s1 = 0.0;
                if (row < n && jj < nb) {
                    const double* ar = a + row * LDB + j0;
#pragma unroll
                    for (int kk = 0; kk < 16; kk += 2) {   // X_bb upper part is 0
                        s0 += ar[kk] * xr[kk];
                        s1 += ar[kk + 1] * xr[kk + 1];
                    }
                }
                v[q] = s0 + s1;
            }
            __syncthreads();
#pragma unroll
            for (int q = 0; q < NQ; q++) {
                const int row = r0 + rg + RG * q;
                if (row < n && jj < nb) a[row * LDB + j0 + jj] = v[q];
            }
            __syncthreads();
            CHK(7);
            // trailing update A_rc -= sum_k L_rk L_ck (lower part), thread = (row offset, col offset) 16 x 16
            const int tx = tid & 15, ty = tid >> 4;
#pragma unroll
            for (int qi = 0; qi < NQ; qi++) {
                const int row = r0 + ty + RG * qi;
                if (row >= n) continue;
                const double* lr = a + row * LDB + j0;
                double lrv[16];
#pragma unroll
                for (int kk = 0; kk < 16; kk++) lrv[kk] = kk < nb ? lr[kk] : 0.0;
#pragma unroll
                for (int qj = 0; qj < 3; qj++) {
                    const int col = r0 + tx + 16 * qj;
                    if (col > row) continue;
                    const double* lc = a + col * LDB + j0;
                    double s0 = 0.0, s1 = 0.0;
#pragma unroll
                    for (int kk = 0; kk < 16; kk += 2) {
                        s0 += lrv[kk] * (kk < nb ? lc[kk] : 0.0);
                        s1 += lrv[kk + 1] * (kk + 1 < nb ? lc[kk + 1] : 0.0);
                    }
                    a[row * LDB + col] -= s0 + s1;
                }
            }
#endif
            __syncthreads();
            CHK(8);
        }
    }
    // off-diagonal blocks of X = L^{-1}, block row by block row: X_ij = -X_ii sum_{k=j}^{i-1} L_ik X_kj, as 8 x 8
    // DMMA tiles: Y_j = L_{i,j..i-1} X_{j..i-1,j} (K = 16 (i - j)) into the scratch, then X_ij = -X_ii Y_j (K = 16)
#ifndef MRA_CHOL_SCALAR
    {
        const int g = lane >> 2, t = lane & 3, nw = NT / 32;
        for (int bi = 1; bi < nbk; bi++) {
            const int i0 = bi * 16, ni = min(16, n - i0);
            for (int tsk = warp; tsk < 4 * bi; tsk += nw) {
                const int bj = tsk >> 2, mr = (tsk >> 1) & 1, mc = tsk & 1;
                double d0 = 0.0, d1 = 0.0;
                const double* lr = a + (i0 + 8 * mr + g) * LDB;
                const double* xc = x + 16 * bj + 8 * mc + g;
                for (int k0 = 16 * bj; k0 < i0; k0 += 4) dmma(d0, d1, lr[k0 + t], xc[(k0 + t) * LDB]);
                double* y = tmp + (bj << 8) + (8 * mr + g) * 16 + 8 * mc + 2 * t;
                y[0] = d0;
                y[1] = d1;
            }
            __syncthreads();
            for (int tsk = warp; tsk < 4 * bi; tsk += nw) {
                const int bj = tsk >> 2, mr = (tsk >> 1) & 1, mc = tsk & 1;
                double d0 = 0.0, d1 = 0.0;
                const double* xr = x + (i0 + 8 * mr + g) * LDB + i0;
                const double* yc = tmp + (bj << 8) + 8 * mc + g;
#pragma unroll
                for (int k0 = 0; k0 < 16; k0 += 4) {
                    const int k = k0 + t;
                    dmma(d0, d1, k < ni ? xr[k] : 0.0, k < ni ? yc[k * 16] : 0.0);
                }
                const int rr = 8 * mr + g, c = 16 * bj + 8 * mc + 2 * t;
                if (rr < ni) {
                    x[(i0 + rr) * LDB + c] = -d0;
                    x[(i0 + rr) * LDB + c + 1] = -d1;
                }
            }
            __syncthreads();
        }
    }
#else
    // off-diagonal blocks of X = L^{-1}, block row by block row: X_ij = -X_ii sum_{k=j}^{i-1} L_ik X_kj
    for (int bi = 1; bi < nbk; bi++) {
        const int i0 = bi * 16, ni = min(16, n - i0);
        for (int e = tid; e < bi * 256; e += NT) {
            const int bj = e >> 8, rr = (e >> 4) & 15, c = e & 15;
            double s0 = 0.0, s1 = 0.0;
            if (rr < ni) {
                const double* lr = a + (i0 + rr) * LDB;
                const double* xcol = x + bj * 16 + c;
                int k = bj * 16 + c;
                for (; k + 1 < i0; k += 2) {
                    s0 += lr[k] * xcol[k * LDB];
                    s1 += lr[k + 1] * xcol[(k + 1) * LDB];
                }
                if (k < i0) s0 += lr[k] * xcol[k * LDB];
            }
            tmp[e] = s0 + s1;
        }
        __syncthreads();
        for (int e = tid; e < bi * 256; e += NT) {
            const int bj = e >> 8, rr = (e >> 4) & 15, c = e & 15;
            if (rr < ni) {
                const double* xr = x + (i0 + rr) * LDB + i0;
                double sacc = 0.0;
                for (int k = 0; k <= rr; k++) sacc += xr[k] * tmp[(bj << 8) + (k << 4) + c];
                x[(i0 + rr) * LDB + bj * 16 + c] = -sacc;
            }
        }
        __syncthreads();
    }
#endif
    CHK(4);
    // log-determinant: the n diagonal logs in parallel (warp 0), then a shuffle reduction
    if (tid < 32) {
        double sl = 0.0;
        for (int j = tid; j < n; j += 32) sl += inplace ? -log(a[j * LDB + j]) : log(a[j * LDB + j]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sl += __shfl_xor_sync(0xffffffffu, sl, o);
        if (tid == 0) *red = 2.0 * sl;
    }
    __syncthreads();
    CHK(5);
    const double ld = *red;
    __syncthreads();
    return ld;
}

// smem layout (doubles): [ misc: MISC_DBL doubles ] [ main: GEMM tiles | factor blocks ]
//   kernels address the main area (`smem` = dyn_smem()); misc sits just below it, so a kernel that only
//   runs GEMMs needs GEMM_SMEM_DBL, one that also factors needs SMEM_DBL
//   factor view of main: blk[64*LDB] | inv[64*LDB] | diag[64]
//   misc: red[0..15] (reductions) | bad flag (int) at misc+16 | work item at misc+18 | GemmDesc at misc+24
constexpr int FAC_DBL = 2 * 64 * LDB + 64 + 768;
constexpr int MAIN_DBL = (FAC_DBL > NSTAGE * STAGE_DBL) ? FAC_DBL : NSTAGE * STAGE_DBL;
constexpr int SMEM_DBL = MAIN_DBL + MISC_DBL;
constexpr int GEMM_SMEM_DBL = NSTAGE * STAGE_DBL + MISC_DBL;
__device__ __forceinline__ double* dyn_smem() {
#ifdef MRA_BULK
    extern __shared__ __align__(1024) double smem_raw[];
#else
    extern __shared__ double smem_raw[];
#endif
    return smem_raw + MISC_DBL;
}
__device__ __forceinline__ GemmDesc* gemm_desc(double* smem) {
    return reinterpret_cast<GemmDesc*>(smem - MISC_DBL + 24);
}
#ifdef MRA_BULK
__device__ __forceinline__ BulkState* bulk_state(double* smem) {
    return reinterpret_cast<BulkState*>(smem - MISC_DBL + 64);
}
static_assert(sizeof(BulkState) <= 8 * sizeof(double), "BulkState must fit the misc smem");
// once per kernel, before its first GEMM: the bulk engine's barriers and counters
__device__ __forceinline__ RegMeta* reg_meta(double* smem) {
    return reinterpret_cast<RegMeta*>(smem - MISC_DBL + 128);
}
static_assert(sizeof(RegMeta) * TMA_NREG <= 128 * sizeof(double), "RegMeta table must fit the misc smem");
__device__ __forceinline__ void engine_init(double* smem, const TmaReg* reg) {
    BulkState* bs = bulk_state(smem);
    RegMeta* rm = reg_meta(smem);
    const int nreg = reg ? reg->n : 0;
    if (threadIdx.x < TMA_NREG) {
        RegMeta e{0, 0, 0, -1, nreg};
        if ((int)threadIdx.x < nreg) {
            e.base = reg->base[threadIdx.x];
            e.end = e.base + reg->bytes[threadIdx.x];
            e.ld = reg->ld[threadIdx.x];
            e.kind = reg->kind[threadIdx.x];
        }
        rm[threadIdx.x] = e;
    }
    if (threadIdx.x == 0) {
        bs->reg = nreg > 0 ? reg : nullptr;
        for (int b = 0; b < NSTAGE; b++) {
            mbar_init(&bs->full[b], 1);
            mbar_init(&bs->empty[b], NT / 32);
        }
        bs->gs = 0;
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
}
#endif
static_assert(sizeof(GemmDesc) <= 40 * sizeof(double), "GemmDesc must fit the misc smem");
struct FacSmem {
    double* blk;
    double* inv;
    double* diagv;
    double* tmp;
    double* red;
    int* bad;
};
__device__ __forceinline__ double* misc_smem(double* smem) { return smem - MISC_DBL; }
__device__ __forceinline__ FacSmem fac_smem(double* smem) {
    FacSmem f;
    f.blk = smem;
    f.inv = smem + 64 * LDB;
    f.diagv = smem + 2 * 64 * LDB;
    f.tmp = f.diagv + 64;
    f.red = misc_smem(smem);
    f.bad = reinterpret_cast<int*>(misc_smem(smem) + 16);
    return f;
}

// in-place factor view (chol_inv_small with x == blk): blk[64*LDB] | diag[64] | tmp[768]
constexpr int FAC_IN_DBL = 64 * LDB + 64 + 768;
__device__ __forceinline__ FacSmem fac_smem_inplace(double* smem) {
    FacSmem f = fac_smem(smem);
    f.inv = f.blk;
    f.diagv = smem + 64 * LDB;
    f.tmp = f.diagv + 64;
    return f;
}

// load lower n x n block of global A (ld) into blk; add `shift` to the diagonal
// every element copied by cp.async (all of a thread's copies in flight at once: the block usually comes from L2 or
// HBM, and a load-then-store loop exposes one memory latency per element), then the diagonal shift
__device__ __forceinline__ void load_block_lower(double* blk, const double* A, long long ld, int n, double shift) {
    for (int e = threadIdx.x; e < 64 * 64; e += NT) {
        const int i = e >> 6, j = e & 63;
        if (i < n && j <= i) cp_async8(blk + i * LDB + j, A + (long long)i * ld + j, 8);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    if (shift != 0.0) {
        for (int i = threadIdx.x; i < n; i += NT) blk[i * LDB + i] += shift;
        __syncthreads();
    }
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
// optional phase timing (build with -DMRA_PHASE_TIMING): CTA-cycles per phase of the bottom kernel
static __device__ unsigned long long g_phase_cycles[32];   // per translation unit (debug counters)
#ifdef MRA_PHASE_TIMING
#define CPHASE_MARK(var) long long var = clock64()
#define CPHASE_ADD(idx, from) do { if (threadIdx.x == 0) atomicAdd(&g_phase_cycles[idx], (unsigned long long)(clock64() - (from))); } while (0)
#else
#define CPHASE_MARK(var)
#define CPHASE_ADD(idx, from)
#endif
__device__ double chol_blocked(double* S, int n, long long ld, double* Dinv, const CovP& cp, double* smem) {
    FacSmem f = fac_smem(smem);
    double total = 0.0;
    for (int j0 = 0; j0 < n; j0 += 64) {
        const int nb = min(64, n - j0);
        CPHASE_MARK(q0);
        load_block_lower(f.blk, S + (long long)j0 * ld + j0, ld, nb, 0.0);
        CPHASE_ADD(9, q0);
        CPHASE_MARK(q3);
        total += chol_inv_small(f.blk, f.inv, nb, f.diagv, f.bad, f.red, f.tmp);
        CPHASE_ADD(10, q3);
        CPHASE_ADD(6, q0);
#ifdef MRA_PHASE_TIMING
        if (threadIdx.x == 0) atomicAdd(&g_phase_cycles[11], 1ULL);
#endif
        double* Di = Dinv + (long long)(j0 / 64) * 4096;
        store_block_lower(f.blk, S + (long long)j0 * ld + j0, ld, nb);
        store_block_full(f.inv, Di, 64, nb);
        __syncthreads();
        const int r = n - j0 - nb;
        if (r > 0) {
            double* P = S + (long long)(j0 + nb) * ld + j0;
            CPHASE_MARK(q1);
            // panel: L_ij = A_ij L_jj^{-T}  (in place, single column tile)
            cta_gemm<MEMN, MEMN, MEMN, MEMN>(r, nb, 0, op_mem(P, ld), op_mem(Di, 64), nb, op_mem(P, ld),
                                             op_mem(P, ld), 0, ci_zero(), 1.0, P, ld, cp, smem);
            CPHASE_ADD(7, q1);
            CPHASE_MARK(q2);
            // trailing: A_ik -= L_ij L_kj^T (lower tiles, in place)
            double* T = S + (long long)(j0 + nb) * ld + j0 + nb;
            cta_gemm<MEMN, MEMN, MEMN, MEMN>(r, r, 1, op_mem(P, ld), op_mem(P, ld), nb, op_mem(P, ld),
                                             op_mem(P, ld), 0, ci_mem(T, ld), -1.0, T, ld, cp, smem);
            CPHASE_ADD(8, q2);
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

}  // inline namespace MRA_ENG_NS
}  // namespace mra
