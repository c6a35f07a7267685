// Microbenchmark of the in-place 64x64 Cholesky + inverse (chol_inv_small, x == a) in the GEMM unit's shape
// (128 threads), alone on one SM and with every SM loaded at 5 CTAs (as k_wide_diag runs it).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DMRA_NT=128 -DMRA_TK=16 -DMRA_NSTAGE=2 -DMRA_MINB=5 tools/bench_chol_unit.cu
#include <cstdio>
#include <cuda_runtime.h>
#define MRA_CHOL_DEBUG
#include "../paper_1905_00141_b200/csrc/mra_device.cuh"
using namespace mra;

__global__ void __launch_bounds__(NT, 5) kbench(int n, int reps, unsigned long long* cycles, double* out) {
    double* smem = dyn_smem();
    FacSmem f = fac_smem_inplace(smem);
    long long total = 0;
    double acc = 0;
    for (int r = 0; r < reps; r++) {
        for (int e = threadIdx.x; e < 64 * 64; e += NT) {
            int i = e >> 6, j = e & 63;
            if (i < n && j <= i) f.blk[i * LDB + j] = exp(-fabs((double)(i - j)) / 8.0) + (i == j ? 0.5 : 0.0);
        }
        if (threadIdx.x == 0) *f.bad = 0;
        __syncthreads();
        long long t0 = clock64();
        acc += chol_inv_small(f.blk, f.blk, n, f.diagv, f.bad, f.red, f.tmp);
        total += clock64() - t0;
    }
    if (threadIdx.x == 0) { atomicAdd(cycles, (unsigned long long)total); out[blockIdx.x] = acc + f.blk[0]; }
}

int main() {
    unsigned long long* c; double* o;
    cudaMalloc(&c, 8); cudaMalloc(&o, 8 * 4096);
    int bytes = (FAC_IN_DBL + MISC_DBL) * 8 + 1024;
    cudaFuncSetAttribute(kbench, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    int nsm = 0; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    int per = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kbench, NT, bytes);
    printf("NT %d smem %d B, %d CTAs/SM\n", NT, bytes, per);
    for (int grid : {1, nsm * per}) {
        for (int n : {52, 64}) {
            cudaMemset(c, 0, 8);
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a);
            kbench<<<grid, NT, bytes>>>(n, 20, c, o);
            cudaEventRecord(b);
            cudaError_t e = cudaDeviceSynchronize();
            float ms = 0; cudaEventElapsedTime(&ms, a, b);
            unsigned long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
            printf("grid %d n %d: %.0f cycles/call, %.3f us per call per SM-throughput (%s)\n", grid, n,
                   (double)h / grid / 20, 1e3 * ms / (20.0 * grid / nsm), cudaGetErrorString(e));
            long long dbg[16];
            cudaMemcpyFromSymbol(dbg, g_chol_dbg, sizeof dbg);
            printf("   per call (CTA 0): zero %.0f | w0 factor %.0f | w0 inverse %.0f | barrier %.0f | panel %.0f | trailing %.0f | X blocks %.0f | logdet %.0f\n",
                   dbg[1] / 20.0, dbg[6] / 20.0, dbg[2] / 20.0, dbg[3] / 20.0, dbg[7] / 20.0, dbg[8] / 20.0, dbg[4] / 20.0, dbg[5] / 20.0);
            long long z[16] = {0}; cudaMemcpyToSymbol(g_chol_dbg, z, sizeof z);
        }
    }
    return 0;
}
