// mra_plan.cu -- S0 on the device: bounding box, leaf key of every
// observation (descent through the half-open boxes; elimination of observations at
// pre-finest knots), stable sort by leaf (LSD radix sort over the base-J digits of the
// leaf path, one pass per level, so the within-leaf order is the input order exactly as in the host
// build), CSR offsets, and the leaf-ordered coordinate pairs. The arithmetic of the descent is the
// host build's, operation for operation, so both builds give bitwise-identical plans.
#include <cuda_runtime.h>

#include <cmath>

#include "mra_internal.h"

namespace mra {

constexpr int PB_NT = 256;              // threads per block
constexpr int PB_IT = 8;                // elements per thread per block
constexpr int PB_CHUNK = PB_NT * PB_IT; // elements per block

// per-block min/max of x and y, and a non-finite flag
__global__ void k_plan_bbox(const double* x, const double* y, long long n, double* part, int* bad) {
    __shared__ double s[4][PB_NT];
    double x0 = INFINITY, x1 = -INFINITY, y0 = INFINITY, y1 = -INFINITY;
    for (long long i = blockIdx.x * (long long)PB_NT + threadIdx.x; i < n; i += (long long)gridDim.x * PB_NT) {
        const double a = x[i], b = y[i];
        if (!isfinite(a) || !isfinite(b)) *bad = 1;
        x0 = fmin(x0, a); x1 = fmax(x1, a); y0 = fmin(y0, b); y1 = fmax(y1, b);
    }
    s[0][threadIdx.x] = x0; s[1][threadIdx.x] = x1; s[2][threadIdx.x] = y0; s[3][threadIdx.x] = y1;
    __syncthreads();
    for (int o = PB_NT / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            s[0][threadIdx.x] = fmin(s[0][threadIdx.x], s[0][threadIdx.x + o]);
            s[1][threadIdx.x] = fmax(s[1][threadIdx.x], s[1][threadIdx.x + o]);
            s[2][threadIdx.x] = fmin(s[2][threadIdx.x], s[2][threadIdx.x + o]);
            s[3][threadIdx.x] = fmax(s[3][threadIdx.x], s[3][threadIdx.x + o]);
        }
        __syncthreads();
    }
    if (threadIdx.x < 4) part[blockIdx.x * 4 + threadIdx.x] = s[threadIdx.x][0];
}

// leaf key by descent (host build_host arithmetic); eliminated observations get key n_leaves
__global__ void k_plan_keys(const double* x, const double* y, long long n, PlanGeom pg, int* key, int* idx,
                            unsigned int* cnt) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double px = x[i], py = y[i];
        long long t = 0;
        bool elim = false;
        long long first = 0, pw = 1;   // first region id of level m: (J^{m-1} - 1) / (J - 1)
        for (int m = 1; m < pg.M; m++) {
            const long long id = first + t;
            const double* b = pg.box + 4 * id;
            if (!elim) {
                bool inx = false, iny = false;
                for (int ix = 0; ix < pg.nx && !inx; ix++) inx = (px == pg.xbar[id * pg.nx + ix]);
                if (inx)
                    for (int iy = 0; iy < pg.ny && !iny; iy++) iny = (py == pg.ybar[id * pg.ny + iy]);
                elim = inx && iny;
            }
            const double mx = 0.5 * (b[0] + b[1]), my = 0.5 * (b[2] + b[3]);
            int c;
            if (pg.J == 4) c = (px >= mx ? 1 : 0) | (py >= my ? 2 : 0);
            else if ((b[1] - b[0]) >= (b[3] - b[2])) c = px >= mx ? 1 : 0;
            else c = py >= my ? 1 : 0;
            t = t * pg.J + c;
            first += pw;
            pw *= pg.J;
        }
        const int k = elim ? (int)pg.nleaf : (int)t;
        key[i] = k;
        idx[i] = (int)i;
        atomicAdd(cnt + k, 1u);
    }
}

// one stable radix pass over digit `d` (base J = 1 << lj): per-block digit counts
__global__ void k_plan_radix_count(const int* key, long long n, int lj, int d, unsigned int* bcnt, int nblk) {
    __shared__ unsigned int c[8];
    if (threadIdx.x < 8) c[threadIdx.x] = 0;
    __syncthreads();
    const int R = 1 << lj, mask = R - 1;
    const long long b0 = (long long)blockIdx.x * PB_CHUNK;
    for (int u = 0; u < PB_IT; u++) {
        const long long e = b0 + u * PB_NT + threadIdx.x;
        if (e < n) atomicAdd(&c[(key[e] >> (lj * d)) & mask], 1u);
    }
    __syncthreads();
    if (threadIdx.x < R) bcnt[threadIdx.x * nblk + blockIdx.x] = c[threadIdx.x];
}

// stable scatter: element order inside a block is (u, thread), i.e. the input order
__global__ void k_plan_radix_scatter(const int* key, const int* idx, long long n, int lj, int d,
                                     const unsigned int* boff, int nblk, int* key2, int* idx2) {
    __shared__ unsigned int wc[PB_NT / 32][8];
    __shared__ unsigned int run[8];
    const int R = 1 << lj, mask = R - 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x < 8) run[threadIdx.x] = 0;
    __syncthreads();
    const long long b0 = (long long)blockIdx.x * PB_CHUNK;
    for (int u = 0; u < PB_IT; u++) {
        const long long e = b0 + u * PB_NT + threadIdx.x;
        const bool ok = e < n;
        const int k = ok ? key[e] : 0, v = ok ? idx[e] : 0;
        const int dg = ok ? (k >> (lj * d)) & mask : -1;
        unsigned int myrank = 0;
        for (int r = 0; r < R; r++) {
            const unsigned int bal = __ballot_sync(0xffffffffu, dg == r);
            if (dg == r) myrank = __popc(bal & ((1u << lane) - 1u));
            if (lane == 0) wc[warp][r] = __popc(bal);
        }
        __syncthreads();
        if (ok) {
            unsigned int before = run[dg];
            for (int w = 0; w < warp; w++) before += wc[w][dg];
            const unsigned int pos = boff[dg * nblk + blockIdx.x] + before + myrank;
            key2[pos] = k;
            idx2[pos] = v;
        }
        __syncthreads();
        if (threadIdx.x < R) {
            unsigned int tot = 0;
            for (int w = 0; w < PB_NT / 32; w++) tot += wc[w][threadIdx.x];
            run[threadIdx.x] += tot;
        }
        __syncthreads();
    }
}

__global__ void k_plan_gather(const double* x, const double* y, const int* idx, long long N, double* pxy,
                              long long* perm) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
        const int j = idx[i];
        pxy[2 * i] = x[j];
        pxy[2 * i + 1] = y[j];
        perm[i] = j;
    }
}

static int grid_for(long long n) {
    long long b = (n + 255) / 256;
    return (int)(b < 1 ? 1 : (b > 8192 ? 8192 : b));
}

cudaError_t plan_bbox(const double* x, const double* y, long long n, double* part, int nblk, int* bad,
                      cudaStream_t st) {
    ++g_kernel_launches;
    k_plan_bbox<<<nblk, PB_NT, 0, st>>>(x, y, n, part, bad);
    return cudaGetLastError();
}

cudaError_t plan_keys(const double* x, const double* y, long long n, const PlanGeom& pg, int* key, int* idx,
                      unsigned int* cnt, cudaStream_t st) {
    ++g_kernel_launches;
    k_plan_keys<<<grid_for(n), 256, 0, st>>>(x, y, n, pg, key, idx, cnt);
    return cudaGetLastError();
}

int plan_radix_blocks(long long n) { return (int)((n + PB_CHUNK - 1) / PB_CHUNK); }

cudaError_t plan_radix_count(const int* key, long long n, int lj, int d, unsigned int* bcnt, cudaStream_t st) {
    const int nblk = plan_radix_blocks(n);
    ++g_kernel_launches;
    k_plan_radix_count<<<nblk, PB_NT, 0, st>>>(key, n, lj, d, bcnt, nblk);
    return cudaGetLastError();
}

cudaError_t plan_radix_scatter(const int* key, const int* idx, long long n, int lj, int d, const unsigned int* boff,
                               int* key2, int* idx2, cudaStream_t st) {
    const int nblk = plan_radix_blocks(n);
    ++g_kernel_launches;
    k_plan_radix_scatter<<<nblk, PB_NT, 0, st>>>(key, idx, n, lj, d, boff, nblk, key2, idx2);
    return cudaGetLastError();
}

cudaError_t plan_gather(const double* x, const double* y, const int* idx, long long N, double* pxy, long long* perm,
                        cudaStream_t st) {
    ++g_kernel_launches;
    k_plan_gather<<<grid_for(N), 256, 0, st>>>(x, y, idx, N, pxy, perm);
    return cudaGetLastError();
}

}  // namespace mra
