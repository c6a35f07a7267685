/*
 * mra_oracle.c -- TEST INFRASTRUCTURE ONLY (not part of the product).
 *
 * Plain, slow, obviously-correct CPU implementation of the multi-resolution
 * approximation (MRA) log-likelihood and posterior state, written from the paper
 * (arXiv:1905.00141, reference/PAPER.md) and the north_star formulas
 * (BASELINE.json) in the paper's W / K notation. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load this file's library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_1905_00141_b200/); neither includes the other.
 *
 * Followed passages (PAPER.md line numbers):
 *   plan   : 99-103 (J in {2,4}; J=4 halves both axes; J=2 halves the longer axis),
 *            101 (root = data domain with top/right pushed out 1%, half-open regions),
 *            112-125 (knot grid ceil(sqrt r) x floor(r / ceil(sqrt r)), offset margin),
 *            134-135 (eliminate observations located at pre-finest knots; offset e/100),
 *            60, 113 (finest-level knots = the observations of the leaf).
 *   prior  : 84-97 (C_m recursion; tau_m(s) = C_m(s,Q)^T eta, eta ~ N(0, C_m(Q,Q)^{-1})),
 *            north_star: W^l = C(Q_R, Q_{a_l}) - sum_{k<l} W^k_R K_{a_k} (W^k_{a_l})^T,
 *            K = (W^m)^{-1} via Cholesky.
 *   post   : 486, 929-936 (ATilde: M(M-1)/2 r x r blocks per leaf, conditional
 *            (co)variances of ancestor pairs), north_star: leaf A^{k,l} = B^{kT} Sigma^{-1} B^l,
 *            omega^k, merges Ktilde^{-1} = K^{-1} + sum A^{m,m}, A <- sum A - A Ktilde A,
 *            log-determinant and quadratic-form accumulation.
 *   result : log L = -1/2 (N log 2 pi + log|Sigma_MRA + tau2 I| + y^T (Sigma_MRA + tau2 I)^{-1} y).
 * Readings where the paper is silent are DESIGN.md §3 (R1..R12).
 *
 * Pins (tests/test_oracle_pins.py): M=1 equals the exact dense GP (scipy), tiny
 * inputs equal the dense Sigma_MRA assembled from PAPER.md:62-92 (oracle/dense.py),
 * paper-printed plan facts, invariances. Every function below is covered by one.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Arithmetic type of the recursion. The oracle proper is fp64 (the paper's precision);
 * -DORACLE_LONG_DOUBLE builds the SAME loops in x87 extended precision (64-bit significand) as a referee
 * for cases where fp64 rounding itself is in question (R12). The plan (boxes, knots, leaf
 * assignment) stays fp64 in both builds, so both evaluate the identical partition. tgmath.h makes
 * sqrt / exp / log follow the argument type. */
#ifdef ORACLE_LONG_DOUBLE
typedef long double real;
#else
typedef double real;
#endif
#include <tgmath.h>

/* ------------------------------------------------------------------ types */
typedef struct {
    const double *x, *y, *z;
    int64_t n;
    int M, J, r;
    double offset, xs, ys;
    int cov;
    double s2, rho, tau2;
    /* plan */
    int nx, ny, rh;
    int64_t nreg, nint, nleaf;
    double *box;          /* nreg*4: x0 x1 y0 y1 */
    double *kx, *ky;      /* nint*rh */
    int64_t *leaf;        /* n: leaf index or -1 (eliminated) */
    int64_t *lstart, *lcnt, *lidx; /* retained observations per leaf, original order */
    int64_t nret;
    /* prior */
    char *need;
    real **W;           /* interior region R at level m: m blocks rh x rh, W^1_R..W^m_R */
    real **LW;          /* chol(W^m_R), rh x rh lower */
    real *ldW;          /* log|W^m_R| */
    /* posterior state */
    int want_post;
    real **Arow;        /* rh x (m rh): Atilde^{m,1..m} */
    real **wm;          /* rh: omegatilde^m */
    real **LP;          /* chol(W^m + Atilde^{mm}) */
    double *region_d, *region_u;
    /* fan-out cache */
    int fan;
    real **cA, **cw, *cd, *cu;
} O;

static int64_t ipow(int64_t b, int e) { int64_t v = 1; while (e-- > 0) v *= b; return v; }
/* first region id of level m (1-based), level-major numbering */
static int64_t lvl_first(const O *o, int m) { return (ipow(o->J, m - 1) - 1) / (o->J - 1); }
static int64_t rid(const O *o, int m, int64_t t) { return lvl_first(o, m) + t; }

/* covariance: exponential ("exponential covariance function") or
   Matern nu=3/2 (BASELINE C2; reading R3), planar Euclidean distance (reading R4) */
static real covf(const O *o, real x1, real y1, real x2, real y2) {
    real dx = (x1 - x2) * o->xs, dy = (y1 - y2) * o->ys;
    real d = sqrt(dx * dx + dy * dy);
    if (o->cov == 0) return o->s2 * exp(-d / o->rho);
    real a = sqrt((real)3) * d / o->rho;
    return o->s2 * (1.0 + a) * exp(-a);
}

/* ------------------------------------------------------ dense helpers (plain) */
/* in-place lower Cholesky of n x n row-major A; returns 0 on success */
static int chol(int n, real *A) {
    for (int j = 0; j < n; j++) {
        real s = A[(int64_t)j * n + j];
        for (int k = 0; k < j; k++) s -= A[(int64_t)j * n + k] * A[(int64_t)j * n + k];
        if (!(s > 0.0)) return -1;
        real L = sqrt(s);
        A[(int64_t)j * n + j] = L;
        for (int i = j + 1; i < n; i++) {
            real t = A[(int64_t)i * n + j];
            for (int k = 0; k < j; k++) t -= A[(int64_t)i * n + k] * A[(int64_t)j * n + k];
            A[(int64_t)i * n + j] = t / L;
        }
        for (int k = j + 1; k < n; k++) A[(int64_t)j * n + k] = 0.0;
    }
    return 0;
}
static real logdet_chol(int n, const real *L) {
    real s = 0;
    for (int i = 0; i < n; i++) s += log(L[(int64_t)i * n + i]);
    return 2.0 * s;
}
/* B (n x k, ld k) <- A^{-1} B with A = L L^T */
static void cholsolve(int n, const real *L, int k, real *B) {
    for (int c = 0; c < k; c++) {
        for (int i = 0; i < n; i++) {
            real t = B[(int64_t)i * k + c];
            for (int j = 0; j < i; j++) t -= L[(int64_t)i * n + j] * B[(int64_t)j * k + c];
            B[(int64_t)i * k + c] = t / L[(int64_t)i * n + i];
        }
        for (int i = n - 1; i >= 0; i--) {
            real t = B[(int64_t)i * k + c];
            for (int j = i + 1; j < n; j++) t -= L[(int64_t)j * n + i] * B[(int64_t)j * k + c];
            B[(int64_t)i * k + c] = t / L[(int64_t)i * n + i];
        }
    }
}
/* C (m x n) -= A (m x k) B (k x n), all row-major with the given leading dims */
static void gemm_sub(int m, int n, int k, const real *A, int lda, const real *B, int ldb,
                     real *C, int ldc) {
    for (int i = 0; i < m; i++)
        for (int p = 0; p < k; p++) {
            real a = A[(int64_t)i * lda + p];
            for (int j = 0; j < n; j++) C[(int64_t)i * ldc + j] -= a * B[(int64_t)p * ldb + j];
        }
}

/* ---------------------------------------------------------------- the plan */
/* knot bars along one axis (reading R6: spacing = ext*(1-2 offset)/(n-1);
   R7: a single bar sits at the midpoint) */
static double bar(double lo, double hi, int nb, int i, double off) {
    if (nb == 1) return 0.5 * (lo + hi);
    double ext = hi - lo;
    return lo + off * ext + (double)i * (ext * (1.0 - 2.0 * off) / (double)(nb - 1));
}

/* J=2 splits the longer axis; equal extents split x (reading R8) */
static int splits_x(const double *b) { return (b[1] - b[0]) >= (b[3] - b[2]); }

static int build_plan(O *o) {
    int M = o->M, J = o->J;
    /* knot grid: nx = ceil(sqrt r), ny = floor(r / nx) */
    int nx = 1;
    while (nx * nx < o->r) nx++;
    o->nx = nx;
    o->ny = o->r / nx;
    o->rh = o->nx * o->ny;
    o->nreg = (ipow(J, M) - 1) / (J - 1);
    o->nint = (ipow(J, M - 1) - 1) / (J - 1);
    o->nleaf = ipow(J, M - 1);
    /* root: data bounding box, top and right pushed out by 1% */
    double x0 = o->x[0], x1 = o->x[0], y0 = o->y[0], y1 = o->y[0];
    for (int64_t i = 1; i < o->n; i++) {
        if (o->x[i] < x0) x0 = o->x[i];
        if (o->x[i] > x1) x1 = o->x[i];
        if (o->y[i] < y0) y0 = o->y[i];
        if (o->y[i] > y1) y1 = o->y[i];
    }
    if (!(x1 > x0) || !(y1 > y0)) return -2;
    o->box = malloc(sizeof(double) * 4 * o->nreg);
    o->box[0] = x0; o->box[1] = x1 + 0.01 * (x1 - x0);
    o->box[2] = y0; o->box[3] = y1 + 0.01 * (y1 - y0);
    /* recursive split */
    for (int m = 1; m < M; m++) {
        int64_t cnt = ipow(J, m - 1);
        for (int64_t t = 0; t < cnt; t++) {
            const double *b = o->box + 4 * rid(o, m, t);
            for (int c = 0; c < J; c++) {
                double *cb = o->box + 4 * rid(o, m + 1, t * J + c);
                memcpy(cb, b, 4 * sizeof(double));
                if (J == 4) {
                    double mx = 0.5 * (b[0] + b[1]), my = 0.5 * (b[2] + b[3]);
                    if (c & 1) cb[0] = mx; else cb[1] = mx;
                    if (c & 2) cb[2] = my; else cb[3] = my;
                } else if (splits_x(b)) {
                    double mx = 0.5 * (b[0] + b[1]);
                    if (c) cb[0] = mx; else cb[1] = mx;
                } else {
                    double my = 0.5 * (b[2] + b[3]);
                    if (c) cb[2] = my; else cb[3] = my;
                }
            }
        }
    }
    /* knots of levels 1..M-1, row-major by (y, x) (reading R9) */
    o->kx = malloc(sizeof(double) * (o->nint * o->rh + 1));
    o->ky = malloc(sizeof(double) * (o->nint * o->rh + 1));
    for (int64_t id = 0; id < o->nint; id++) {
        const double *b = o->box + 4 * id;
        for (int iy = 0; iy < o->ny; iy++)
            for (int ix = 0; ix < o->nx; ix++) {
                o->kx[id * o->rh + iy * o->nx + ix] = bar(b[0], b[1], o->nx, ix, o->offset);
                o->ky[id * o->rh + iy * o->nx + ix] = bar(b[2], b[3], o->ny, iy, o->offset);
            }
    }
    /* leaf of each observation by descending the tree, half-open [lo, hi);
       eliminate an observation equal to a knot of any pre-finest region */
    o->leaf = malloc(sizeof(int64_t) * o->n);
    int64_t nleaf = o->nleaf;
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < o->n; i++) {
        double px = o->x[i], py = o->y[i];
        int64_t t = 0;
        int elim = 0;
        for (int m = 1; m < M; m++) {
            int64_t id = rid(o, m, t);
            const double *b = o->box + 4 * id;
            for (int iy = 0; iy < o->ny && !elim; iy++)
                for (int ix = 0; ix < o->nx; ix++)
                    if (px == o->kx[id * o->rh + iy * o->nx + ix] &&
                        py == o->ky[id * o->rh + iy * o->nx + ix]) { elim = 1; break; }
            int c;
            if (J == 4) c = (px >= 0.5 * (b[0] + b[1]) ? 1 : 0) + (py >= 0.5 * (b[2] + b[3]) ? 2 : 0);
            else if (splits_x(b)) c = px >= 0.5 * (b[0] + b[1]) ? 1 : 0;
            else c = py >= 0.5 * (b[2] + b[3]) ? 1 : 0;
            t = t * J + c;
        }
        o->leaf[i] = elim ? -1 : t;
    }
    o->lcnt = calloc(nleaf, sizeof(int64_t));
    o->lstart = malloc(sizeof(int64_t) * (nleaf + 1));
    for (int64_t i = 0; i < o->n; i++) if (o->leaf[i] >= 0) o->lcnt[o->leaf[i]]++;
    o->lstart[0] = 0;
    for (int64_t t = 0; t < nleaf; t++) o->lstart[t + 1] = o->lstart[t] + o->lcnt[t];
    o->nret = o->lstart[nleaf];
    if (o->nret == 0) return -3;
    o->lidx = malloc(sizeof(int64_t) * (o->nret + 1));
    int64_t *fill = calloc(nleaf, sizeof(int64_t));
    for (int64_t i = 0; i < o->n; i++) {
        int64_t t = o->leaf[i];
        if (t >= 0) o->lidx[o->lstart[t] + fill[t]++] = i;
    }
    free(fill);
    return 0;
}

/* ------------------------------------------------------------------ prior */
/* W^l(Q, Q_{a_l}) for l = 1..L for a point set Q of np points inside region (lev, t):
 *   W^l = C(Q, Q_{a_l}) - sum_{k<l} W^k(Q) K_{a_k} (W^k_{a_l})^T,   K_{a_k} = (W^k_{a_k})^{-1}
 * (north_star; PAPER.md:84-92 evaluated at the knots). When L == lev the ancestor at
 * level L is the region itself and W^k_{a_L} = Wout[k-1] (np == rh). */
static void w_chain(O *o, const real *px, const real *py, int np, int lev, int64_t t,
                    int L, real **Wout) {
    int rh = o->rh;
    real *T = malloc(sizeof(real) * rh * (np > rh ? np : rh));
    for (int l = 1; l <= L; l++) {
        int64_t al = t / ipow(o->J, lev - l);
        int64_t idl = rid(o, l, al);
        real *Wl = Wout[l - 1];
        for (int i = 0; i < np; i++)
            for (int j = 0; j < rh; j++)
                Wl[(int64_t)i * rh + j] = covf(o, px[i], py[i], o->kx[idl * rh + j], o->ky[idl * rh + j]);
        for (int k = 1; k < l; k++) {
            int64_t ak = t / ipow(o->J, lev - k);
            int64_t idk = rid(o, k, ak);
            const real *Wk_al = (l == lev) ? Wout[k - 1] : o->W[idl] + (int64_t)(k - 1) * rh * rh;
            int nal = (l == lev) ? np : rh;
            /* T = K_{a_k} (W^k_{a_l})^T : rh x nal */
            for (int p = 0; p < rh; p++)
                for (int q = 0; q < nal; q++) T[(int64_t)p * nal + q] = Wk_al[(int64_t)q * rh + p];
            cholsolve(rh, o->LW[idk], nal, T);
            gemm_sub(np, nal, rh, Wout[k - 1], rh, T, nal, Wl, rh);
        }
    }
    free(T);
}

static int prior_region(O *o, int m, int64_t t) {
    int rh = o->rh;
    int64_t id = rid(o, m, t);
    real *px = malloc(sizeof(real) * rh), *py = malloc(sizeof(real) * rh);
    for (int i = 0; i < rh; i++) { px[i] = o->kx[id * rh + i]; py[i] = o->ky[id * rh + i]; }
    o->W[id] = malloc(sizeof(real) * m * rh * rh);
    real **Wout = malloc(sizeof(real *) * m);
    for (int l = 0; l < m; l++) Wout[l] = o->W[id] + (int64_t)l * rh * rh;
    w_chain(o, px, py, rh, m, t, m, Wout);
    o->LW[id] = malloc(sizeof(real) * rh * rh);
    memcpy(o->LW[id], Wout[m - 1], sizeof(real) * rh * rh);
    int rc = chol(rh, o->LW[id]);
    o->ldW[id] = rc ? NAN : logdet_chol(rh, o->LW[id]);
    free(Wout); free(px); free(py);
    return rc;
}

/* ------------------------------------------------------------- posterior */
/* leaf j: B^l = W^l(S_j, Q_{a_l}), Sigma_j = W^M(S_j,S_j) + tau2 I,
   A^{k,l} = B^{kT} Sigma^{-1} B^l, omega^k = B^{kT} Sigma^{-1} y, d = log|Sigma|, u = y^T Sigma^{-1} y */
static int leaf_factor(O *o, int64_t j, int np, real *B, real *S, real **Bl) {
    int rh = o->rh, P = o->M - 1;
    const int64_t *idx = o->lidx + o->lstart[j];
    real *px = malloc(sizeof(real) * (np + 1)), *py = malloc(sizeof(real) * (np + 1));
    for (int i = 0; i < np; i++) { px[i] = o->x[idx[i]]; py[i] = o->y[idx[i]]; }
    for (int l = 0; l < P; l++) Bl[l] = B + (int64_t)l * np * rh;
    if (P > 0) w_chain(o, px, py, np, o->M, j, P, Bl);
    /* W^M = C(S,S) - sum_k B^k K_{a_k} B^{kT} */
    for (int i = 0; i < np; i++)
        for (int q = 0; q < np; q++) S[(int64_t)i * np + q] = covf(o, px[i], py[i], px[q], py[q]);
    real *T = malloc(sizeof(real) * rh * (np + 1));
    for (int k = 1; k <= P; k++) {
        int64_t idk = rid(o, k, j / ipow(o->J, o->M - k));
        for (int p = 0; p < rh; p++)
            for (int q = 0; q < np; q++) T[(int64_t)p * np + q] = Bl[k - 1][(int64_t)q * rh + p];
        cholsolve(rh, o->LW[idk], np, T);
        gemm_sub(np, np, rh, Bl[k - 1], rh, T, np, S, np);
    }
    for (int i = 0; i < np; i++) S[(int64_t)i * np + i] += o->tau2;   /* nugget (reading R2) */
    free(T); free(px); free(py);
    return chol(np, S);
}

static int leaf_terms(O *o, int64_t j, real *A, real *w, real *d, real *u) {
    int rh = o->rh, P = o->M - 1, PP = P * rh;
    int np = (int)o->lcnt[j];
    memset(A, 0, sizeof(real) * PP * PP);
    memset(w, 0, sizeof(real) * (PP + 1));
    *d = 0; *u = 0;
    if (np == 0) return 0;   /* empty leaf: zero contribution (reading R10) */
    real *B = malloc(sizeof(real) * ((int64_t)np * PP + 1));
    real *S = malloc(sizeof(real) * (int64_t)np * np);
    real **Bl = malloc(sizeof(real *) * (P + 1));
    int rc = leaf_factor(o, j, np, B, S, Bl);
    if (rc) { free(B); free(S); free(Bl); return -4; }
    /* X = Sigma^{-1} [B^1 .. B^P | y] */
    int nc = PP + 1;
    real *X = malloc(sizeof(real) * (int64_t)np * nc);
    const int64_t *idx = o->lidx + o->lstart[j];
    for (int i = 0; i < np; i++) {
        for (int l = 0; l < P; l++)
            for (int c = 0; c < rh; c++) X[(int64_t)i * nc + l * rh + c] = Bl[l][(int64_t)i * rh + c];
        X[(int64_t)i * nc + PP] = o->z[idx[i]];
    }
    cholsolve(np, S, nc, X);
    for (int k = 0; k < P; k++)
        for (int a = 0; a < rh; a++)
            for (int c = 0; c < nc; c++) {
                real s = 0;
                for (int i = 0; i < np; i++) s += Bl[k][(int64_t)i * rh + a] * X[(int64_t)i * nc + c];
                if (c < PP) A[(int64_t)(k * rh + a) * PP + c] = s; else w[k * rh + a] = s;
            }
    real uu = 0;
    for (int i = 0; i < np; i++) uu += o->z[idx[i]] * X[(int64_t)i * nc + PP];
    *u = uu;
    *d = logdet_chol(np, S);
    free(X); free(B); free(S); free(Bl);
    return 0;
}

/* region (lev, t): output A (P x P, P = (lev-1) rh), omega (P), d, u for its parent */
static int post_region(O *o, int lev, int64_t t, real *A, real *w, real *d, real *u) {
    int64_t id = rid(o, lev, t);
    int rc = 0;
    if (o->cA && lev == o->fan && o->cA[t]) {
        int P = (lev - 1) * o->rh;
        memcpy(A, o->cA[t], sizeof(real) * P * P);
        memcpy(w, o->cw[t], sizeof(real) * (P + 1));
        *d = o->cd[t]; *u = o->cu[t];
        return 0;
    }
    if (lev == o->M) {
        rc = leaf_terms(o, t, A, w, d, u);
        if (o->region_d) { o->region_d[id] = *d; o->region_u[id] = *u; }
        return rc;
    }
    int rh = o->rh, m = lev, Pm = m * rh, Pp = (m - 1) * rh;
    real *At = calloc((int64_t)Pm * Pm, sizeof(real)), *wt = calloc(Pm + 1, sizeof(real));
    real *Ac = malloc(sizeof(real) * ((int64_t)Pm * Pm + 1)), *wc = malloc(sizeof(real) * (Pm + 1));
    real dt = 0, ut = 0, dc, uc;
    /* Atilde = sum over children (fixed child order), PAPER.md:462 supervisor gather */
    for (int c = 0; c < o->J && !rc; c++) {
        rc = post_region(o, m + 1, t * o->J + c, Ac, wc, &dc, &uc);
        for (int64_t e = 0; e < (int64_t)Pm * Pm; e++) At[e] += Ac[e];
        for (int e = 0; e < Pm; e++) wt[e] += wc[e];
        dt += dc; ut += uc;
    }
    if (rc) { free(At); free(wt); free(Ac); free(wc); return rc; }
    /* Ktilde^{-1} = K^{-1} + Atilde^{m,m} = W^m + Atilde^{m,m} (north_star; reading R1) */
    real *LPm = malloc(sizeof(real) * rh * rh);
    for (int a = 0; a < rh; a++)
        for (int b = 0; b < rh; b++)
            LPm[a * rh + b] = o->W[id][(int64_t)(m - 1) * rh * rh + a * rh + b] +
                              At[(int64_t)(Pp + a) * Pm + Pp + b];
    if (chol(rh, LPm)) { free(At); free(wt); free(Ac); free(wc); free(LPm); return -4; }
    /* X = Ktilde [Atilde^{m,1..m-1} | omegatilde^m] : rh x (Pp+1) */
    int nc = Pp + 1;
    real *X = malloc(sizeof(real) * rh * nc);
    for (int a = 0; a < rh; a++) {
        for (int c = 0; c < Pp; c++) X[a * nc + c] = At[(int64_t)(Pp + a) * Pm + c];
        X[a * nc + Pp] = wt[Pp + a];
    }
    cholsolve(rh, LPm, nc, X);
    /* A^{k,l} = Atilde^{k,l} - Atilde^{k,m} Ktilde Atilde^{m,l}; omega^k likewise */
    for (int a = 0; a < Pp; a++) {
        for (int b = 0; b < Pp; b++) {
            real s = At[(int64_t)a * Pm + b];
            for (int q = 0; q < rh; q++) s -= At[(int64_t)a * Pm + Pp + q] * X[q * nc + b];
            A[(int64_t)a * Pp + b] = s;
        }
        real s = wt[a];
        for (int q = 0; q < rh; q++) s -= At[(int64_t)a * Pm + Pp + q] * X[q * nc + Pp];
        w[a] = s;
    }
    real qf = 0;
    for (int q = 0; q < rh; q++) qf += wt[Pp + q] * X[q * nc + Pp];
    /* d = sum d_c + log|Ktilde^{-1}| - log|W^m| ;  u = sum u_c - omegatilde^mT Ktilde omegatilde^m */
    *d = dt + logdet_chol(rh, LPm) - o->ldW[id];
    *u = ut - qf;
    if (o->region_d) { o->region_d[id] = *d; o->region_u[id] = *u; }
    if (o->want_post) {
        o->Arow[id] = malloc(sizeof(real) * rh * Pm);
        for (int a = 0; a < rh; a++)
            for (int c = 0; c < Pm; c++) o->Arow[id][(int64_t)a * Pm + c] = At[(int64_t)(Pp + a) * Pm + c];
        o->wm[id] = malloc(sizeof(real) * rh);
        memcpy(o->wm[id], wt + Pp, sizeof(real) * rh);
        o->LP[id] = LPm;
    } else {
        free(LPm);
    }
    free(X); free(At); free(wt); free(Ac); free(wc);
    return 0;
}

/* -------------------------------------------------------------- prediction */
/* Posterior mean and variance of X(p) at query points (the paper's "prediction" calculation mode,
 * PAPER.md:228, 494), in the W / K notation used above. For p in leaf j with
 * ancestors a_1..a_P (P = M-1):
 *   b^l(p)   = W^l(p, Q_{a_l})  by the same recursion as the observations (w_chain)
 *   c        = C_M(S_j, p) = C(S_j, p) - sum_k B^k_j K_{a_k} b^k(p)^T
 *   C_M(p,p) = C(p, p) - sum_k b^k(p) K_{a_k} b^k(p)^T
 *   mean     = sum_l b^l(p) nu_{a_l} + c^T Sigma_j^{-1} (y_j - sum_l B^l_j nu_{a_l})
 *   bt_l     = b^l(p) - B^{lT}_j Sigma_j^{-1} c
 *   var      = C_M(p,p) - c^T Sigma_j^{-1} c + sum_{l,l'} bt_l^T Cov(eta_{a_l}, eta_{a_l'} | y) bt_l'
 * where nu = E[eta | y] (the mu recursion above) and the posterior covariances of the ancestor
 * chain (the paper's BTilde) follow top-down from
 *   eta_R | eta_anc, y ~ N(Ktilde_R (omegatilde^m - sum_k Atilde^{m,k} eta_{a_k}), Ktilde_R):
 *   Cov(eta_m, eta_l) = -Ktilde_m sum_{k<m} Atilde^{m,k} Cov(eta_k, eta_l)          (l < m)
 *   Cov(eta_m, eta_m) = Ktilde_m + Ktilde_m (sum_{k,k'} Atilde^{m,k} Cov(eta_k, eta_k') Atilde^{m,k'T}) Ktilde_m
 * Queries outside the root domain get NaN. Pinned against the dense definition (oracle/dense.py). */
static int predict_all(O *o, const real *MU, const double *qx, const double *qy, int64_t nq,
                       double *pmean, double *pvar) {
    const int M = o->M, J = o->J, rh = o->rh, P = M - 1, PP = P * rh;
    int64_t *ql = malloc(sizeof(int64_t) * (nq + 1));
    for (int64_t i = 0; i < nq; i++) {
        const double *b = o->box;
        double px = qx[i], py = qy[i];
        if (!(px >= b[0] && px < b[1] && py >= b[2] && py < b[3])) { ql[i] = -1; continue; }
        int64_t t = 0;
        for (int m = 1; m < M; m++) {
            const double *bb = o->box + 4 * rid(o, m, t);
            int c;
            if (J == 4) c = (px >= 0.5 * (bb[0] + bb[1]) ? 1 : 0) + (py >= 0.5 * (bb[2] + bb[3]) ? 2 : 0);
            else if (splits_x(bb)) c = px >= 0.5 * (bb[0] + bb[1]) ? 1 : 0;
            else c = py >= 0.5 * (bb[2] + bb[3]) ? 1 : 0;
            t = t * J + c;
        }
        ql[i] = t;
    }
    int bad = 0;
    #pragma omp parallel for schedule(dynamic, 1) reduction(|:bad)
    for (int64_t j = 0; j < o->nleaf; j++) {
        int64_t nqj = 0;
        for (int64_t i = 0; i < nq; i++) nqj += (ql[i] == j);
        if (nqj == 0) continue;
        int np = (int)o->lcnt[j];
        const int64_t *idx = o->lidx + o->lstart[j];
        real *B = malloc(sizeof(real) * ((int64_t)np * PP + 1));
        real *S = malloc(sizeof(real) * ((int64_t)np * np + 1));
        real **Bl = malloc(sizeof(real *) * (P + 1));
        if (np > 0 && leaf_factor(o, j, np, B, S, Bl)) { bad |= 1; free(B); free(S); free(Bl); continue; }
        /* rr = Sigma_j^{-1} (y_j - sum_l B^l nu_{a_l}) */
        real *rr = malloc(sizeof(real) * (np + 1));
        for (int i = 0; i < np; i++) {
            real s = o->z[idx[i]];
            for (int k = 1; k <= P; k++) {
                int64_t ak = rid(o, k, j / ipow(J, M - k));
                for (int q = 0; q < rh; q++) s -= Bl[k - 1][(int64_t)i * rh + q] * MU[ak * rh + q];
            }
            rr[i] = s;
        }
        if (np > 0) cholsolve(np, S, 1, rr);
        /* posterior covariance of the ancestor chain eta_{a_1..a_P} (PP x PP), top-down */
        real *CC = calloc((int64_t)PP * PP + 1, sizeof(real));
        for (int m = 1; m <= P; m++) {
            int64_t id = rid(o, m, j / ipow(J, M - m));
            int Pp = (m - 1) * rh, Pm = m * rh;
            const real *Ar = o->Arow[id];   /* rh x Pm: Atilde^{m,1..m} */
            /* Gm = Atilde^{m,<m} CC[<m, <m]   (rh x Pp) */
            real *Gm = calloc((int64_t)rh * Pp + 1, sizeof(real));
            for (int a = 0; a < rh; a++)
                for (int l = 0; l < Pp; l++) {
                    real s = 0;
                    for (int k = 0; k < Pp; k++) s += Ar[(int64_t)a * Pm + k] * CC[(int64_t)k * PP + l];
                    Gm[(int64_t)a * Pp + l] = s;
                }
            /* Cov(eta_m, eta_l) = -Ktilde_m Gm */
            real *X = malloc(sizeof(real) * ((int64_t)rh * Pp + 1));
            for (int64_t e = 0; e < (int64_t)rh * Pp; e++) X[e] = Gm[e];
            if (Pp) cholsolve(rh, o->LP[id], Pp, X);
            for (int a = 0; a < rh; a++)
                for (int l = 0; l < Pp; l++) {
                    CC[(int64_t)(Pp + a) * PP + l] = -X[(int64_t)a * Pp + l];
                    CC[(int64_t)l * PP + Pp + a] = -X[(int64_t)a * Pp + l];
                }
            /* Cov(eta_m, eta_m) = Ktilde_m + Ktilde_m (Gm Atilde^{m,<m T}) Ktilde_m */
            /* Y = I + (Gm Atilde^T) Ktilde_m, then Ktilde_m Y = Ktilde_m + Ktilde_m Gm A^T Ktilde_m */
            real *Y = calloc((int64_t)rh * rh, sizeof(real));
            for (int a = 0; a < rh; a++) Y[a * rh + a] = 1.0;
            real *Z = calloc((int64_t)rh * rh, sizeof(real));
            for (int a = 0; a < rh; a++)
                for (int b = 0; b < rh; b++) {
                    real s = 0;
                    for (int l = 0; l < Pp; l++) s += Gm[(int64_t)a * Pp + l] * Ar[(int64_t)b * Pm + l];
                    Z[a * rh + b] = s;   /* Gm Atilde^{m,<m T}, symmetric */
                }
            cholsolve(rh, o->LP[id], rh, Z);          /* Ktilde Z */
            for (int a = 0; a < rh; a++)               /* (Ktilde Z)^T = Z Ktilde */
                for (int b = 0; b < rh; b++) Y[a * rh + b] += Z[b * rh + a];
            cholsolve(rh, o->LP[id], rh, Y);           /* Ktilde (I + Z Ktilde) */
            for (int a = 0; a < rh; a++)
                for (int b = 0; b < rh; b++) CC[(int64_t)(Pp + a) * PP + Pp + b] = Y[a * rh + b];
            free(Gm); free(X); free(Y); free(Z);
        }
        /* per query */
        real *bq = malloc(sizeof(real) * (PP + 1)), *c = malloc(sizeof(real) * (np + 1));
        real *w = malloc(sizeof(real) * (np + 1)), *bt = malloc(sizeof(real) * (PP + 1));
        real *t = malloc(sizeof(real) * (rh + 1));
        real **Bq = malloc(sizeof(real *) * (P + 1));
        for (int l = 0; l < P; l++) Bq[l] = bq + (int64_t)l * rh;
        for (int64_t iq = 0; iq < nq; iq++) {
            if (ql[iq] != j) continue;
            real px = qx[iq], py = qy[iq];
            if (P > 0) w_chain(o, &px, &py, 1, M, j, P, Bq);
            real cpp = covf(o, px, py, px, py);
            for (int i = 0; i < np; i++) c[i] = covf(o, o->x[idx[i]], o->y[idx[i]], px, py);
            for (int k = 1; k <= P; k++) {
                int64_t idk = rid(o, k, j / ipow(J, M - k));
                for (int a = 0; a < rh; a++) t[a] = Bq[k - 1][a];
                cholsolve(rh, o->LW[idk], 1, t);                 /* K_{a_k} b^k(p)^T */
                for (int a = 0; a < rh; a++) cpp -= Bq[k - 1][a] * t[a];
                for (int i = 0; i < np; i++)
                    for (int a = 0; a < rh; a++) c[i] -= Bl[k - 1][(int64_t)i * rh + a] * t[a];
            }
            real mean = 0.0;
            for (int k = 1; k <= P; k++) {
                int64_t ak = rid(o, k, j / ipow(J, M - k));
                for (int a = 0; a < rh; a++) mean += Bq[k - 1][a] * MU[ak * rh + a];
            }
            for (int i = 0; i < np; i++) { mean += c[i] * rr[i]; w[i] = c[i]; }
            if (np > 0) cholsolve(np, S, 1, w);
            real var = cpp;
            for (int i = 0; i < np; i++) var -= c[i] * w[i];
            for (int l = 0; l < P; l++)
                for (int a = 0; a < rh; a++) {
                    real s = Bq[l][a];
                    for (int i = 0; i < np; i++) s -= Bl[l][(int64_t)i * rh + a] * w[i];
                    bt[l * rh + a] = s;
                }
            for (int e = 0; e < PP; e++) {
                real s = 0;
                for (int f = 0; f < PP; f++) s += CC[(int64_t)e * PP + f] * bt[f];
                var += bt[e] * s;
            }
            pmean[iq] = mean;
            pvar[iq] = var;
        }
        free(bq); free(c); free(w); free(bt); free(t); free(Bq);
        free(CC); free(rr); free(B); free(S); free(Bl);
    }
    for (int64_t i = 0; i < nq; i++)
        if (ql[i] < 0) { pmean[i] = NAN; pvar[i] = NAN; }
    free(ql);
    return bad ? -4 : 0;
}

/* ----------------------------------------------------------------- driver */
static void free_all(O *o) {
    if (o->W) for (int64_t i = 0; i < o->nint; i++) { free(o->W[i]); free(o->LW[i]); }
    if (o->Arow) for (int64_t i = 0; i < o->nint; i++) { free(o->Arow[i]); free(o->wm[i]); free(o->LP[i]); }
    if (o->cA) for (int64_t i = 0; i < ipow(o->J, o->fan - 1); i++) { free(o->cA[i]); free(o->cw[i]); }
    free(o->W); free(o->LW); free(o->ldW); free(o->Arow); free(o->wm); free(o->LP);
    free(o->cA); free(o->cw); free(o->cd); free(o->cu);
    free(o->box); free(o->kx); free(o->ky); free(o->leaf); free(o->lstart); free(o->lcnt); free(o->lidx);
    free(o->need);
}

static int is_in_subtree(const O *o, int m, int64_t t, int tm, int64_t tt) {
    /* region (m,t) is target (tm,tt), an ancestor of it, or a descendant of it */
    if (m <= tm) return (tt / ipow(o->J, tm - m)) == t;
    return (t / ipow(o->J, m - tm)) == tt;
}

/* Plan only (for plan tests). Outputs are optional (NULL to skip).
   leaf_of[n]: leaf index or -1; boxes[nreg*4]; knots_x/y[nint*rh]. */
int oracle_plan(const double *x, const double *y, int64_t n, int M, int J, int r, double offset,
                int *rhat, int64_t *nreg, int64_t *leaf_of, double *boxes, double *knx, double *kny) {
    if (M < 1 || (J != 2 && J != 4) || r < 1 || n < 1) return -1;
    O o; memset(&o, 0, sizeof o);
    o.x = x; o.y = y; o.n = n; o.M = M; o.J = J; o.r = r; o.offset = offset;
    int rc = build_plan(&o);
    if (rc == 0 || rc == -3) {
        if (rhat) *rhat = o.rh;
        if (nreg) *nreg = o.nreg;
        if (leaf_of) memcpy(leaf_of, o.leaf, sizeof(int64_t) * n);
        if (boxes) memcpy(boxes, o.box, sizeof(double) * 4 * o.nreg);
        if (knx && o.nint) memcpy(knx, o.kx, sizeof(double) * o.nint * o.rh);
        if (kny && o.nint) memcpy(kny, o.ky, sizeof(double) * o.nint * o.rh);
    }
    free_all(&o);
    return rc;
}

/* Full evaluation (target_level = 0) or one subtree (target_level >= 1, target index
   target_t): prior of the target's ancestors + its subtree, posterior of its subtree.
   Returns 0 or a negative error: -1 config, -2 degenerate domain, -3 all eliminated,
   -4 Cholesky failure. out_d / out_u are d, u of the root (or target); loglik only for
   the full evaluation. region_d/u [nreg] (NaN where not computed), mu [nint*rh] =
   E[eta_R | y] in the paper's parametrization, xq [nint*rh] = E[X(q)|y]
   at every pre-finest knot, smooth [n] = E[X(s_i)|y] at the observations (NaN for
   eliminated). */
static int run_impl(const double *x, const double *y, const double *z, int64_t n, int M, int J, int r,
                    double offset, double xscale, double yscale, int cov, double sigma2, double rho,
                    double tau2, int target_level, int64_t target_t, double *loglik, double *out_d,
                    double *out_u, double *region_d, double *region_u, double *mu, double *xq,
                    double *smooth, int64_t *n_retained, int nthreads, double *out_A, double *out_w,
                    int given_level, const double *gA, const double *gw, const double *gd,
                    const double *gu, const double *qx, const double *qy, int64_t nq, double *pmean,
                    double *pvar) {
    if (M < 1 || (J != 2 && J != 4) || r < 1 || n < 1) return -1;
    if (!(sigma2 > 0) || !(rho > 0) || !(tau2 > 0)) return -1;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
    O o; memset(&o, 0, sizeof o);
    o.x = x; o.y = y; o.z = z; o.n = n; o.M = M; o.J = J; o.r = r; o.offset = offset;
    o.xs = xscale; o.ys = yscale; o.cov = cov; o.s2 = sigma2; o.rho = rho; o.tau2 = tau2;
    int rc = build_plan(&o);
    if (rc) { free_all(&o); return rc; }
    if (n_retained) *n_retained = o.nret;
    int tl = target_level > 0 ? target_level : 1;
    int64_t tt = target_level > 0 ? target_t : 0;
    if (tl > M || tt < 0 || tt >= ipow(J, tl - 1)) { free_all(&o); return -1; }
    o.want_post = (mu || xq || smooth || nq > 0) && target_level <= 0;
    o.region_d = region_d; o.region_u = region_u;
    if (region_d) for (int64_t i = 0; i < o.nreg; i++) { region_d[i] = NAN; region_u[i] = NAN; }
    int64_t nint = o.nint;
    o.W = calloc(nint + 1, sizeof(real *));
    o.LW = calloc(nint + 1, sizeof(real *));
    o.ldW = calloc(nint + 1, sizeof(real));
    o.Arow = calloc(nint + 1, sizeof(real *));
    o.wm = calloc(nint + 1, sizeof(real *));
    o.LP = calloc(nint + 1, sizeof(real *));
    /* prior, top-down, levels 1..M-1 (regions of a level are independent) */
    int bad = 0;
    for (int m = 1; m < M && !bad; m++) {
        int64_t cnt = ipow(J, m - 1);
        #pragma omp parallel for schedule(dynamic, 1) reduction(|:bad)
        for (int64_t t = 0; t < cnt; t++)
            if (is_in_subtree(&o, m, t, tl, tt))
                if (prior_region(&o, m, t)) bad |= 1;
    }
    if (bad) { free_all(&o); return -4; }
    /* posterior, bottom-up. Regions of the fan-out level are computed in parallel (each
       depth-first), then the levels above serially; per-region arithmetic is unchanged. */
    int rh = o.rh;
    int fan = tl;
    while (fan < M && (ipow(J, fan - tl)) < 64) fan++;
    if (given_level > 0) {
        /* finish from given level-s outputs (the exchange step of subtree sharding):
           the level-s regions' (A, omega, d, u) are supplied, the levels above are merged here */
        fan = given_level;
        o.fan = fan;
        int64_t cnt = ipow(J, fan - 1);
        int P = (fan - 1) * rh;
        o.cA = calloc(cnt, sizeof(real *));
        o.cw = calloc(cnt, sizeof(real *));
        o.cd = calloc(cnt, sizeof(real));
        o.cu = calloc(cnt, sizeof(real));
        for (int64_t t = 0; t < cnt; t++) {
            o.cA[t] = malloc(sizeof(real) * ((int64_t)P * P + 1));
            o.cw[t] = malloc(sizeof(real) * (P + 1));
            for (int64_t e = 0; e < (int64_t)P * P; e++) o.cA[t][e] = gA[t * (int64_t)P * P + e];
            for (int e = 0; e < P; e++) o.cw[t][e] = gw[t * (int64_t)P + e];
            o.cd[t] = gd[t];
            o.cu[t] = gu[t];
        }
    } else if (fan > tl) {
        o.fan = fan;
        int64_t cnt = ipow(J, fan - 1);
        o.cA = calloc(cnt, sizeof(real *));
        o.cw = calloc(cnt, sizeof(real *));
        o.cd = calloc(cnt, sizeof(real));
        o.cu = calloc(cnt, sizeof(real));
        int P = (fan - 1) * rh;
        int64_t lo = tt * ipow(J, fan - tl), hi = (tt + 1) * ipow(J, fan - tl);
        #pragma omp parallel for schedule(dynamic, 1) reduction(|:bad)
        for (int64_t t = lo; t < hi; t++) {
            real *A = malloc(sizeof(real) * ((int64_t)P * P + 1));
            real *w = malloc(sizeof(real) * (P + 1));
            real d, u;
            int e = post_region(&o, fan, t, A, w, &d, &u);
            if (e) bad |= 1;
            o.cd[t] = d; o.cu[t] = u;
            o.cw[t] = w;
            o.cA[t] = A;   /* publish last: post_region() checks cA[t] */
        }
        if (bad) { free_all(&o); return -4; }
    }
    {
        int P = (tl - 1) * rh;
        real *A = malloc(sizeof(real) * ((int64_t)P * P + 1)), *w = malloc(sizeof(real) * (P + 1));
        real d, u;
        rc = post_region(&o, tl, tt, A, w, &d, &u);
        if (!rc && out_A) for (int64_t e = 0; e < (int64_t)P * P; e++) out_A[e] = A[e];
        if (!rc && out_w) for (int e = 0; e < P; e++) out_w[e] = w[e];
        free(A); free(w);
        if (rc) { free_all(&o); return rc; }
        if (out_d) *out_d = d;
        if (out_u) *out_u = u;
        if (loglik) *loglik = target_level > 0 ? NAN
                                  : -0.5 * ((real)o.nret * log(2 * acos((real)-1)) + d + u);
    }
    if (o.want_post) {
        /* mu_R = Ktilde_R (omegatilde^m - sum_{k<m} Atilde^{m,k} mu_{a_k}), top-down */
        real *MU = calloc(nint * rh + 1, sizeof(real));
        for (int m = 1; m < M; m++) {
            int64_t cnt = ipow(J, m - 1);
            #pragma omp parallel for schedule(static)
            for (int64_t t = 0; t < cnt; t++) {
                int64_t id = rid(&o, m, t);
                int Pm = m * rh;
                real *v = malloc(sizeof(real) * rh);
                for (int a = 0; a < rh; a++) {
                    real s = o.wm[id][a];
                    for (int k = 1; k < m; k++) {
                        int64_t ak = rid(&o, k, t / ipow(J, m - k));
                        for (int q = 0; q < rh; q++)
                            s -= o.Arow[id][(int64_t)a * Pm + (k - 1) * rh + q] * MU[ak * rh + q];
                    }
                    v[a] = s;
                }
                cholsolve(rh, o.LP[id], 1, v);
                memcpy(MU + id * rh, v, sizeof(real) * rh);
                /* E[X(q)|y] at the knots of R: sum_{k<=m} W^k_R mu_{a_k} (the
                   finer levels vanish at a level-m knot since C_{m+1}(q, .) = 0) */
                if (xq)
                    for (int a = 0; a < rh; a++) {
                        real s = 0;
                        for (int k = 1; k <= m; k++) {
                            int64_t ak = rid(&o, k, t / ipow(J, m - k));
                            for (int q = 0; q < rh; q++)
                                s += o.W[id][(int64_t)(k - 1) * rh * rh + a * rh + q] * MU[ak * rh + q];
                        }
                        xq[id * rh + a] = s;
                    }
                free(v);
            }
        }
        if (mu) for (int64_t e = 0; e < nint * rh; e++) mu[e] = MU[e];
        if (nq > 0 && predict_all(&o, MU, qx, qy, nq, pmean, pvar)) bad |= 1;
        if (smooth) {
            /* E[X(S_j)|y] = y_j - tau2 Sigma_j^{-1} (y_j - sum_k B^k mu_{a_k}) */
            for (int64_t i = 0; i < n; i++) smooth[i] = NAN;
            int P = M - 1;
            #pragma omp parallel for schedule(dynamic, 1) reduction(|:bad)
            for (int64_t j = 0; j < o.nleaf; j++) {
                int np = (int)o.lcnt[j];
                if (np == 0) continue;
                real *B = malloc(sizeof(real) * ((int64_t)np * P * rh + 1));
                real *S = malloc(sizeof(real) * (int64_t)np * np);
                real **Bl = malloc(sizeof(real *) * (P + 1));
                real *v = malloc(sizeof(real) * np);
                if (leaf_factor(&o, j, np, B, S, Bl)) { bad |= 1; }
                else {
                    const int64_t *idx = o.lidx + o.lstart[j];
                    for (int i = 0; i < np; i++) {
                        real s = o.z[idx[i]];
                        for (int k = 1; k <= P; k++) {
                            int64_t ak = rid(&o, k, j / ipow(J, M - k));
                            for (int q = 0; q < rh; q++) s -= Bl[k - 1][(int64_t)i * rh + q] * MU[ak * rh + q];
                        }
                        v[i] = s;
                    }
                    cholsolve(np, S, 1, v);
                    for (int i = 0; i < np; i++) smooth[idx[i]] = o.z[idx[i]] - o.tau2 * v[i];
                }
                free(B); free(S); free(Bl); free(v);
            }
        }
        free(MU);
    }
    free_all(&o);
    return bad ? -4 : 0;
}

int oracle_run(const double *x, const double *y, const double *z, int64_t n, int M, int J, int r,
               double offset, double xscale, double yscale, int cov, double sigma2, double rho,
               double tau2, int target_level, int64_t target_t, double *loglik, double *out_d,
               double *out_u, double *region_d, double *region_u, double *mu, double *xq,
               double *smooth, int64_t *n_retained, int nthreads, double *out_A, double *out_w) {
    return run_impl(x, y, z, n, M, J, r, offset, xscale, yscale, cov, sigma2, rho, tau2, target_level,
                    target_t, loglik, out_d, out_u, region_d, region_u, mu, xq, smooth, n_retained,
                    nthreads, out_A, out_w, 0, NULL, NULL, NULL, NULL, NULL, NULL, 0, NULL, NULL);
}

/* log L from the outputs (A, omega, d, u) of every level-s region (s >= 2), merging levels
   s-1..1 with the recursion above (the rank-0 side of the exchange step). gA: [J^{s-1}][P][P],
   gw: [J^{s-1}][P], gd/gu: [J^{s-1}], P = (s-1) r_hat. */
int oracle_finish(const double *x, const double *y, const double *z, int64_t n, int M, int J, int r,
                  double offset, double xscale, double yscale, int cov, double sigma2, double rho,
                  double tau2, int s, const double *gA, const double *gw, const double *gd,
                  const double *gu, double *loglik) {
    if (s < 2 || s > M) return -1;
    return run_impl(x, y, z, n, M, J, r, offset, xscale, yscale, cov, sigma2, rho, tau2, 0, 0, loglik,
                    NULL, NULL, NULL, NULL, NULL, NULL, NULL, NULL, 0, NULL, NULL, s, gA, gw, gd, gu, NULL, NULL,
                    0, NULL, NULL);
}

/* Posterior mean / variance (noise-free X, no nugget: SPEC.md:271) at nq query locations after a
   full evaluation; NaN for queries outside the root domain. Returns as oracle_run. */
int oracle_predict(const double *x, const double *y, const double *z, int64_t n, int M, int J, int r,
                   double offset, double xscale, double yscale, int cov, double sigma2, double rho,
                   double tau2, const double *qx, const double *qy, int64_t nq, double *pmean, double *pvar,
                   int nthreads) {
    if (nq < 1) return -1;
    return run_impl(x, y, z, n, M, J, r, offset, xscale, yscale, cov, sigma2, rho, tau2, 0, 0, NULL, NULL,
                    NULL, NULL, NULL, NULL, NULL, NULL, NULL, nthreads, NULL, NULL, 0, NULL, NULL, NULL, NULL,
                    qx, qy, nq, pmean, pvar);
}

int oracle_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
