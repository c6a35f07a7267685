// bench_gemm.cu -- microbenchmark of the CTA GEMM engine (cta_gemm in mra_device.cuh) in isolation:
// persistent grid, every CTA computes 64x64 output tiles with K-deep operands resident in L2, for the
// operand kinds the hot path uses (MEMN x MEMN: Sigma/panels, MEMT x MEMT: stacked SYRK, COVK x MEMN:
// chain with fused covariance). Reports fp64 TFLOP/s against the measured DMMA peak (37.15).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o bench_gemm bench_gemm.cu
#include <cstdio>
#include <cuda_runtime.h>
#ifdef WITH_CUBLAS
#include <cublas_v2.h>
#endif
#ifndef MRA_MINB
#define MRA_MINB 2
#endif
#include "../paper_1905_00141_b200/csrc/mra_device.cuh"
using namespace mra;

template <int KA, int KB>
__global__ void __launch_bounds__(NT, MRA_MINB) kbench(const double* A, const double* B, const double* pts,
                                                       double* C, int K, long long ntiles) {
    double* smem = dyn_smem();
    CovP cp;
    cp.kind = 0; cp.s2 = 1.0; cp.rho = 2.0; cp.xs = 1.0; cp.ys = 1.0;
#ifdef MRA_HAS_IR
    cp.ir = 0.5;
#endif
    for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
#ifdef HOT
        const int pa = (int)(blockIdx.x % 64), pb = (int)(blockIdx.x % 64);   // same panels every tile (L1/L2-hot)
#else
        const int pa = (int)(t % 64), pb = (int)((t / 64) % 64);
#endif
        Op a, b;
        if (KA == COVK) a = op_cov(pts + 128 * pa, pts + 128 * ((pa + 7) % 64));
        else if (KA == MEMN) a = op_mem(A + (long long)pa * 64 * K, K);
        else a = op_mem(A + 64 * pa, 64 * 64);     // MEMT: [k][64 * 64 rows]
        if (KB == MEMN) b = op_mem(B + (long long)pb * 64 * K, K);
        else b = op_mem(B + 64 * pb, 64 * 64);
        const int K0 = (KA == COVK) ? 64 : K;
        if (KA == COVK)
            cta_gemm<COVK, KB, MEMN, KB>(64, 64, 0, a, b, K0, op_mem(A + (long long)pa * 64 * K, K),
                                         op_mem(B + (long long)pb * 64 * K + 64, K), K - 64, ci_zero(), 1.0,
                                         C + (t % 1024) * 4096, 64, cp, smem);
        else
            cta_gemm<KA, KB, MEMN, MEMN>(64, 64, 0, a, b, K0, a, b, 0, ci_zero(), 1.0, C + (t % 1024) * 4096, 64,
                                         cp, smem);
    }
}

template <int KA, int KB>
void run(const char* name, double* A, double* B, double* P, double* C, int K) {
    const int bytes = GEMM_SMEM_DBL * 8;
    cudaFuncSetAttribute(kbench<KA, KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kbench<KA, KB>, NT, bytes);
    const int grid = per * 148;
    const long long ntiles = (long long)grid * 40;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    kbench<KA, KB><<<grid, NT, bytes>>>(A, B, P, C, K, ntiles);
    cudaEventRecord(e0);
    kbench<KA, KB><<<grid, NT, bytes>>>(A, B, P, C, K, ntiles);
    cudaEventRecord(e1);
    cudaError_t err = cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double tf = 2.0 * 64 * 64 * K * (double)ntiles / (ms * 1e-3) / 1e12;
    printf("%-10s K=%5d  %d CTA/SM  %.3f ms  %.2f TFLOP/s  (%.1f%% of 37.15)  %s\n", name, K, per, ms, tf,
           100 * tf / 37.15, cudaGetErrorString(err));
}

int main() {
    const int KMAX = 1024;
    double *A, *B, *P, *C;
    cudaMalloc(&A, 8LL * 64 * 64 * KMAX);
    cudaMalloc(&B, 8LL * 64 * 64 * KMAX);
    cudaMalloc(&P, 8LL * 2 * 64 * 64 * 2);
    cudaMalloc(&C, 8LL * 1024 * 4096);
    cudaMemset(A, 0, 8LL * 64 * 64 * KMAX);
    cudaMemset(B, 0, 8LL * 64 * 64 * KMAX);
    cudaMemset(P, 0, 8LL * 2 * 64 * 64 * 2);
#ifdef WITH_CUBLAS
    {   // yardstick: cuBLAS DGEMM 8192^3 (library; not on the product path)
        const int n = 8192;
        double *X, *Y, *Z;
        cudaMalloc(&X, 8LL * n * n); cudaMalloc(&Y, 8LL * n * n); cudaMalloc(&Z, 8LL * n * n);
        cudaMemset(X, 0, 8LL * n * n); cudaMemset(Y, 0, 8LL * n * n);
        cublasHandle_t h; cublasCreate(&h);
        const double one = 1.0, zero = 0.0;
        cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, X, n, Y, n, &zero, Z, n);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        for (int r = 0; r < 3; r++) cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, X, n, Y, n, &zero, Z, n);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("cuBLAS DGEMM 8192^3: %.2f TFLOP/s\n", 3 * 2.0 * n * (double)n * n / (ms * 1e-3) / 1e12);
        cudaFree(X); cudaFree(Y); cudaFree(Z);
    }
#endif
    for (int K : {64, 128, 192, 576}) {
        run<MEMN, MEMN>("MEMNxMEMN", A, B, P, C, K);
        run<MEMT, MEMT>("MEMTxMEMT", A, B, P, C, K);
        run<COVK, MEMN>("COVKxMEMN", A, B, P, C, K);
    }
    return 0;
}
