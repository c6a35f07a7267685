// Throughput of the in-place 64x64 Cholesky + inverse (chol_inv_small with x == a) as the wide path's
// diagonal-factor kernel runs it: every resident CTA factors its own block repeatedly.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 [-DMRA_NT=128 -DMRA_TK=16 -DMRA_NSTAGE=2]
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1905_00141_b200/csrc/mra_device.cuh"
using namespace mra;
#ifndef MINB
#define MINB 4
#endif
#ifndef INPLACE
#define INPLACE 1
#endif

__global__ void __launch_bounds__(NT, MINB) kbench(int n, int reps, double* out) {
    double* smem = dyn_smem();
    FacSmem f = INPLACE ? fac_smem_inplace(smem) : fac_smem(smem);
    double acc = 0;
    for (int r = 0; r < reps; r++) {
        for (int e = threadIdx.x; e < 64 * 64; e += NT) {
            int i = e >> 6, j = e & 63;
            if (i < n && j <= i) f.blk[i * LDB + j] = exp(-fabs((double)(i - j)) / 8.0) + (i == j ? 0.5 + 1e-3 * r : 0.0);
        }
        if (threadIdx.x == 0) *f.bad = 0;
        __syncthreads();
        acc += chol_inv_small(f.blk, f.inv, n, f.diagv, f.bad, f.red, f.tmp);
    }
    if (threadIdx.x == 0) out[blockIdx.x] = acc + f.inv[0];
}

int main() {
    double* o;
    cudaMalloc(&o, 8 * 8192);
    const int dbl = (INPLACE ? FAC_IN_DBL : FAC_DBL) + MISC_DBL;
    const int bytes = dbl * 8;
    cudaFuncSetAttribute(kbench, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kbench, NT, bytes);
    const int grid = per * 148, reps = 50;
    for (int n : {64, 51}) {
        kbench<<<grid, NT, bytes>>>(n, 2, o);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        kbench<<<grid, NT, bytes>>>(n, reps, o);
        cudaEventRecord(e1);
        cudaError_t err = cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double calls = (double)grid * reps;
        printf("NT=%d inplace=%d n=%d: %d CTA/SM, %.1f ns per factor (GPU throughput), %.0f ns per call per CTA (%s)\n",
               NT, INPLACE, n, per, ms * 1e6 / calls, ms * 1e6 / reps, cudaGetErrorString(err));
    }
    return 0;
}
