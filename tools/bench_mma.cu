// bench_mma.cu -- ceiling of the CTA GEMM engine's inner loop (mma_ktile on smem-resident tiles) with
// and without the per-k-tile barrier, vs the register-only DMMA peak. Diagnostic only.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1905_00141_b200/csrc/mra_device.cuh"
using namespace mra;

template <int KA, int KB, bool SYNC, int LOADS = 0>
__global__ void __launch_bounds__(NT, 2) kloop(double* out, int iters, const double* src) {
    extern __shared__ double smem[];
    for (int e = threadIdx.x; e < STAGE_DBL; e += NT) smem[e] = 1e-6 * (e & 63);
    __syncthreads();
    double acc[2][4][2] = {};
    double* scratch = smem + STAGE_DBL;   // cp.async targets (not read by the MMAs)
    const double* g = src + (blockIdx.x % 64) * 4096;
    for (int it = 0; it < iters; it++) {
        if (LOADS) {
#pragma unroll
            for (int i = 0; i < LOADS; i++) {
                const int e = threadIdx.x + NT * i;
                cp_async16(scratch + 2 * (e % 1024), g + 2 * ((e + it * 8) % 2048), 16);
            }
            cp_async_commit();
            cp_async_wait<1>();
        }
        mma_ktile<KA, KB>(acc, smem, smem + TILE_DBL, TK);
        if (SYNC) __syncthreads();
    }
    double s = 0;
    for (int mi = 0; mi < 2; mi++) for (int ni = 0; ni < 4; ni++) s += acc[mi][ni][0] + acc[mi][ni][1];
    if (s == 1234.5) out[0] = s;
}

template <int KA, int KB, bool SYNC, int LOADS = 0>
void run(const char* name, double* o) {
    const int bytes = SMEM_DBL * 8, iters = 4000;
    cudaFuncSetAttribute(kloop<KA, KB, SYNC, LOADS>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    for (int per : {1, 2}) {
        const int grid = 148 * per;
        kloop<KA, KB, SYNC, LOADS><<<grid, NT, bytes>>>(o, 10, o + 64);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        kloop<KA, KB, SYNC, LOADS><<<grid, NT, bytes>>>(o, iters, o + 64);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double tf = 2.0 * 64 * 64 * TK * (double)iters * grid / (ms * 1e-3) / 1e12;
        printf("%-22s %d CTA/SM: %.2f TFLOP/s (%.1f%% of 37.15)\n", name, per, tf, 100 * tf / 37.15);
    }
}

int main() {
    double* o; cudaMalloc(&o, 8 * (64 + 64 * 4096 + 4096));
    cudaMemset(o, 0, 8 * (64 + 64 * 4096 + 4096));
    run<MEMN, MEMN, false>("MEMNxMEMN no-sync", o);
    run<MEMN, MEMN, true>("MEMNxMEMN sync", o);
    run<MEMT, MEMT, false>("MEMTxMEMT no-sync", o);
    run<MEMT, MEMT, true>("MEMTxMEMT sync", o);
    run<MEMN, MEMN, true, 4>("MEMN sync +4 LDGSTS", o);
    run<MEMN, MEMN, true, 8>("MEMN sync +8 LDGSTS", o);
    run<MEMN, MEMN, false, 8>("MEMN nosync +8 LDGSTS", o);
    return 0;
}
