// Microbenchmark of the in-smem 64x64 Cholesky + inverse (chol_inv_small) in isolation.
#include <cstdio>
#include <cuda_runtime.h>
#define MRA_CHOL_DEBUG
#include "../paper_1905_00141_b200/csrc/mra_device.cuh"
using namespace mra;

__global__ void __launch_bounds__(NT, 2) kbench(int n, int reps, unsigned long long* cycles, double* out) {
    double* smem = dyn_smem();
    FacSmem f = fac_smem(smem);
    long long total = 0;
    double acc = 0;
    for (int r = 0; r < reps; r++) {
        // SPD matrix: A = 0.5 I + exp(-|i-j|/8)
        for (int e = threadIdx.x; e < 64 * 64; e += NT) {
            int i = e >> 6, j = e & 63;
            if (i < n && j <= i) f.blk[i * LDB + j] = exp(-fabs((double)(i - j)) / 8.0) + (i == j ? 0.5 : 0.0);
        }
        if (threadIdx.x == 0) *f.bad = 0;
        __syncthreads();
        long long t0 = clock64();
        acc += chol_inv_small(f.blk, f.inv, n, f.diagv, f.bad, f.red, f.tmp);
        total += clock64() - t0;
    }
    if (threadIdx.x == 0) { atomicAdd(cycles, (unsigned long long)total); out[blockIdx.x] = acc + f.inv[0]; }
}

int main() {
    unsigned long long* c; double* o;
    cudaMalloc(&c, 8); cudaMalloc(&o, 8 * 4096);
    int bytes = SMEM_DBL * 8;
    cudaFuncSetAttribute(kbench, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    for (int grid : {1}) {
        for (int n : {16, 64}) {
            cudaMemset(c, 0, 8);
            kbench<<<grid, NT, bytes>>>(n, 20, c, o);
            cudaError_t e = cudaDeviceSynchronize();
            unsigned long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
            printf("grid %d n %d: %.0f cycles/call (%s)\n", grid, n, (double)h / grid / 20, cudaGetErrorString(e));
            long long dbg[16];
            cudaMemcpyFromSymbol(dbg, g_chol_dbg, sizeof dbg);
            printf("   zero %.0f | warp0-block %.0f | sync %.0f | rest %.0f | final %.0f  (per call, summed over blocks)\n",
                   (dbg[1] - dbg[0]) / 20.0, (dbg[2] - dbg[1]) / 20.0, (dbg[3] - dbg[2]) / 20.0, (dbg[4] - dbg[3]) / 20.0, (dbg[5] - dbg[4]) / 20.0);
            long long z[16] = {0}; cudaMemcpyToSymbol(g_chol_dbg, z, sizeof z);
        }
    }
    return 0;
}
