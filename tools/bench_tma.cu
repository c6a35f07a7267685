// bench_tma.cu -- prototype of the GEMM unit's TMA engine: 64x64 fp64 output tiles on DMMA (4 warps of
// 32x32), operand k-tiles (64 x TK) staged by cp.async.bulk.tensor from per-CTA tensor maps that are
// re-targeted per GEMM call with tensormap.replace (address, extents, row stride), completion on
// full/empty mbarriers (no CTA barrier per k-tile). Layouts chosen for conflict-free DMMA fragment loads:
//   MEMN  X[i][k] = p[i ld + k]: 2-D box (16 k, 64 i), SWIZZLE_128B (16-byte chunk ^= row & 7)
//   MEMT  X[i][k] = p[k ld + i]: 3-D box (8 i_lo, TK k, 8 i_hi) -> smem [i_hi][k][i_lo]
// Reports TFLOP/s vs the measured DMMA peak (37.15) for MEMN x MEMN and MEMT x MEMT at several K, and
// checks the product against a reference computed with plain loads.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o bench_tma bench_tma.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cmath>

#ifndef NST
#define NST 3
#endif
#ifndef TKD
#define TKD 16
#endif
#ifndef MINB
#define MINB 4
#endif
constexpr int TK = TKD;
constexpr int NT = 128;
constexpr int TILE_DBL = 64 * TK;            // one operand k-tile
constexpr int STAGE_DBL = 2 * TILE_DBL;
enum { MEMN = 0, MEMT = 1 };

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n"
                 ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma2(void* dst, const void* map, int c0, int c1, uint64_t* bar) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
                 ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma3(void* dst, const void* map, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
                 ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)) : "memory");
}
// re-target a tensor map in global memory: address, one extent, one stride
__device__ __forceinline__ void tm_addr(void* map, const void* p) {
    asm volatile("tensormap.replace.tile.global_address.global.b1024.b64 [%0], %1;\n" ::"l"(map), "l"(p) : "memory");
}
template <int ORD>
__device__ __forceinline__ void tm_dim(void* map, int v) {
    asm volatile("tensormap.replace.tile.global_dim.global.b1024.b32 [%0], %1, %2;\n" ::"l"(map), "n"(ORD), "r"(v) : "memory");
}
template <int ORD>
__device__ __forceinline__ void tm_stride(void* map, long long v) {
    asm volatile("tensormap.replace.tile.global_stride.global.b1024.b64 [%0], %1, %2;\n" ::"l"(map), "n"(ORD), "l"(v) : "memory");
}
__device__ __forceinline__ void tm_publish(void* map) {
    asm volatile("fence.proxy.tensormap::generic.release.gpu;\n" ::: "memory");
    asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;\n" ::"l"(map) : "memory");
}
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
// fragment (row i, k) of a staged k-tile
template <int KIND>
__device__ __forceinline__ double frag(const double* s, int i, int k) {
    if (KIND == MEMN) return s[(k >> 4) * 1024 + i * 16 + (((((k & 15) >> 1) ^ (i & 7)) << 1) | (k & 1))];
    return s[(i >> 3) * (TK * 8) + k * 8 + (i & 7)];
}

// operand descriptor re-targeting: MEMN 2-D (K, rows), MEMT 3-D (8, K, rows/8)
template <int KIND>
__device__ __forceinline__ void retarget(void* map, const double* p, long long ld, int rows, int K) {
    tm_addr(map, p);
    if (KIND == MEMN) {
        tm_dim<0>(map, K);
        tm_dim<1>(map, rows);
        tm_stride<0>(map, ld * 8);
    } else {
        tm_dim<1>(map, K);
        tm_dim<2>(map, (rows + 7) / 8);
        tm_stride<0>(map, ld * 8);
    }
    tm_publish(map);
}
template <int KIND>
__device__ __forceinline__ void load_tile(double* dst, const void* map, int r0, int k0, uint64_t* bar) {
    if (KIND == MEMN) {
#pragma unroll
        for (int h = 0; h < TK / 16; h++) tma2(dst + h * 64 * 16, map, k0 + 16 * h, r0, bar);
    } else {
        tma3(dst, map, 0, k0, r0 / 8, bar);
    }
}

struct Pipe {   // in smem
    uint64_t full[NST], empty[NST];
    unsigned gs;   // stages issued so far (uniform)
};

template <int KA, int KB>
__global__ void __launch_bounds__(NT, MINB)
ktma(const double* A, const double* B, double* C, int K, long long ntiles, char* maps, int per_call) {
    extern __shared__ __align__(1024) unsigned char smraw[];
    double* st = reinterpret_cast<double*>(smraw);
    Pipe* pp = reinterpret_cast<Pipe*>(smraw + NST * STAGE_DBL * 8);
    char* mapA = maps + (size_t)blockIdx.x * 256;
    char* mapB = mapA + 128;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int wr = (warp >> 1) * 32, wc = (warp & 1) * 32;
    if (threadIdx.x == 0) {
        for (int b = 0; b < NST; b++) { mbar_init(&pp->full[b], 1); mbar_init(&pp->empty[b], NT / 32); }
        pp->gs = 0;
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    unsigned gs = 0;
    const int T = (K + TK - 1) / TK;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int pa = (int)(tile % 64), pb = (int)((tile / 64) % 64);
        const double *Ap, *Bp;
        long long lda, ldb;
        if (KA == MEMN) { Ap = A + (long long)pa * 64 * K; lda = K; } else { Ap = A + 64 * pa; lda = 64 * 64; }
        if (KB == MEMN) { Bp = B + (long long)pb * 64 * K; ldb = K; } else { Bp = B + 64 * pb; ldb = 64 * 64; }
        if (threadIdx.x == 0 && (per_call || tile == blockIdx.x)) {
            asm volatile("fence.proxy.async.global;\n" ::: "memory");
            retarget<KA>(mapA, Ap, lda, 64, K);
            retarget<KB>(mapB, Bp, ldb, 64, K);
        }
        double acc[4][4][2];
#pragma unroll
        for (int a = 0; a < 4; a++)
#pragma unroll
            for (int b = 0; b < 4; b++) acc[a][b][0] = acc[a][b][1] = 0.0;
        // producer: thread 0 keeps NST-1 k-tiles in flight
        auto issue = [&](int ki) {
            const unsigned s = gs + ki, b = s % NST, n = s / NST;
            if (n > 0) mbar_wait(&pp->empty[b], (n - 1) & 1);
            mbar_expect(&pp->full[b], STAGE_DBL * 8);
            double* As = st + b * STAGE_DBL;
            load_tile<KA>(As, mapA, 0, ki * TK, &pp->full[b]);
            load_tile<KB>(As + TILE_DBL, mapB, 0, ki * TK, &pp->full[b]);
        };
        if (threadIdx.x == 0)
            for (int ki = 0; ki < NST - 1 && ki < T; ki++) issue(ki);
        for (int kt = 0; kt < T; kt++) {
            if (threadIdx.x == 0 && kt + NST - 1 < T) issue(kt + NST - 1);
            __syncwarp();
            const unsigned s = gs + kt, b = s % NST;
            mbar_wait(&pp->full[b], (s / NST) & 1);
            const double* As = st + b * STAGE_DBL;
            const double* Bs = As + TILE_DBL;
            const int nk = min(TK, K - kt * TK);
#pragma unroll
            for (int kk = 0; kk < TK; kk += 4) {
                if (kk < nk) {
                    double a[4], bb[4];
#pragma unroll
                    for (int mi = 0; mi < 4; mi++) a[mi] = frag<KA>(As, wr + mi * 8 + g, kk + t);
#pragma unroll
                    for (int ni = 0; ni < 4; ni++) bb[ni] = frag<KB>(Bs, wc + ni * 8 + g, kk + t);
#pragma unroll
                    for (int mi = 0; mi < 4; mi++)
#pragma unroll
                        for (int ni = 0; ni < 4; ni++) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi], bb[ni]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&pp->empty[b]);
        }
        gs += T;
        double* Cp = C + (tile % 1024) * 4096;
#pragma unroll
        for (int mi = 0; mi < 4; mi++)
#pragma unroll
            for (int ni = 0; ni < 4; ni++) {
                const int i = wr + mi * 8 + g, j = wc + ni * 8 + 2 * t;
                *reinterpret_cast<double2*>(Cp + i * 64 + j) = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
            }
    }
}

static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;

static void make_template(CUtensorMap* m, int kind, void* base) {
    CUresult r;
    if (kind == MEMN) {
        cuuint64_t dims[2] = {64, 64};
        cuuint64_t strides[1] = {64 * 8};
        cuuint32_t box[2] = {16, 64};
        cuuint32_t es[2] = {1, 1};
        r = encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
        cuuint64_t dims[3] = {8, 64, 8};
        cuuint64_t strides[2] = {64 * 64 * 8, 64};
        cuuint32_t box[3] = {8, TK, 8};
        cuuint32_t es[3] = {1, 1, 1};
        r = encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_64B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r != CUDA_SUCCESS) { printf("encode kind %d failed: %d\n", kind, (int)r); exit(1); }
}

template <int KA, int KB>
void run(const char* name, double* A, double* B, double* C, int K, char* maps, int per_call,
         const std::vector<double>& hA, const std::vector<double>& hB) {
    const int bytes = NST * STAGE_DBL * 8 + 1024;
    cudaFuncSetAttribute(ktma<KA, KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, ktma<KA, KB>, NT, bytes);
    const int grid = per * 148;
    // templates for every CTA slot
    std::vector<CUtensorMap> h(2 * grid);
    for (int c = 0; c < grid; c++) { make_template(&h[2 * c], KA, A); make_template(&h[2 * c + 1], KB, B); }
    cudaMemcpy(maps, h.data(), sizeof(CUtensorMap) * 2 * grid, cudaMemcpyHostToDevice);
    const long long ntiles = (long long)grid * 40;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    ktma<KA, KB><<<grid, NT, bytes>>>(A, B, C, K, ntiles, maps, per_call);
    cudaEventRecord(e0);
    ktma<KA, KB><<<grid, NT, bytes>>>(A, B, C, K, ntiles, maps, per_call);
    cudaEventRecord(e1);
    cudaError_t err = cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ktma<KA, KB><<<grid, NT, bytes>>>(A, B, C, K, 128, maps, per_call);   // every C slot written once
    cudaDeviceSynchronize();
    const double tf = 2.0 * 64 * 64 * K * (double)ntiles / (ms * 1e-3) / 1e12;
    // check tile 0 (pa = pb = 0) and tile 65 (pa = 1, pb = 1) against host loops
    std::vector<double> hc(2 * 4096);
    cudaMemcpy(hc.data(), C, 8 * 4096, cudaMemcpyDeviceToHost);
    cudaMemcpy(hc.data() + 4096, C + 65 * 4096, 8 * 4096, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int which = 0; which < 2; which++) {
        const int pa = which ? 1 : 0, pb = which ? 1 : 0;
        for (int i = 0; i < 64; i++)
            for (int j = 0; j < 64; j++) {
                double s = 0;
                for (int k = 0; k < K; k++) {
                    const double a = KA == MEMN ? hA[(size_t)pa * 64 * K + (size_t)i * K + k] : hA[(size_t)k * 4096 + 64 * pa + i];
                    const double b = KB == MEMN ? hB[(size_t)pb * 64 * K + (size_t)j * K + k] : hB[(size_t)k * 4096 + 64 * pb + j];
                    s += a * b;
                }
                maxerr = fmax(maxerr, fabs(s - hc[which * 4096 + i * 64 + j]) / (1 + fabs(s)));
            }
    }
    printf("%-10s K=%5d NST=%d TK=%d %d CTA/SM per_call=%d  %.3f ms  %.2f TFLOP/s  (%.1f%% of 37.15)  maxrel %.1e  %s\n",
           name, K, NST, TK, per, per_call, ms, tf, 100 * tf / 37.15, maxerr, cudaGetErrorString(err));
}

int main() {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q);
    if (!encode) { printf("no cuTensorMapEncodeTiled\n"); return 1; }
    const int KMAX = 1024;
    const size_t nel = (size_t)64 * 64 * KMAX;
    std::vector<double> hA(nel), hB(nel);
    srand(1);
    for (size_t i = 0; i < nel; i++) { hA[i] = rand() / (double)RAND_MAX - 0.5; hB[i] = rand() / (double)RAND_MAX - 0.5; }
    double *A, *B, *C;
    char* maps;
    cudaMalloc(&A, 8 * nel);
    cudaMalloc(&B, 8 * nel);
    cudaMalloc(&C, 8LL * 1024 * 4096);
    cudaMalloc(&maps, 256 * 148 * 8);
    for (int K : {64, 192, 576, 1024}) {
        // MEMN operands: 64 panels of [64 rows][K]; MEMT: [K][64 * 64]
        cudaMemcpy(A, hA.data(), 8 * (size_t)64 * 64 * K, cudaMemcpyHostToDevice);
        cudaMemcpy(B, hB.data(), 8 * (size_t)64 * 64 * K, cudaMemcpyHostToDevice);
        std::vector<double> a2(hA.begin(), hA.begin() + (size_t)64 * 64 * K), b2(hB.begin(), hB.begin() + (size_t)64 * 64 * K);
        run<MEMN, MEMN>("MEMNxMEMN", A, B, C, K, maps, 1, a2, b2);
        run<MEMT, MEMT>("MEMTxMEMT", A, B, C, K, maps, 1, a2, b2);
        run<MEMN, MEMN>("MEMNxMEMN", A, B, C, K, maps, 0, a2, b2);
    }
    return 0;
}
