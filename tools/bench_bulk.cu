// bench_bulk.cu -- prototype: the CTA GEMM engine's stage loads as TMA bulk copies (one
// cp.async.bulk per 256-byte tile row, issued by one warp, completion through mbarrier transaction
// counts) instead of 8 cp.async per thread, with full/empty mbarriers per stage. Diagnostic only:
// MEMN x MEMN, 64x64 tiles, K a multiple of 32, 16-byte aligned operands.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1905_00141_b200/csrc/mra_device.cuh"
using namespace mra;

__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, int parity) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n"
                 ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

template <bool BULK>
__global__ void __launch_bounds__(NT, 2) kbulk(const double* A, const double* B, double* C, int K, long long ntiles) {
    extern __shared__ double smem[];
    unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + NSTAGE * STAGE_DBL);
    unsigned long long* empty = full + NSTAGE;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int wr = (warp >> 1) * 16, wc = (warp & 1) * 32;
    if (threadIdx.x == 0) {
        for (int b = 0; b < NSTAGE; b++) { mbar_init(&full[b], 1); mbar_init(&empty[b], NT / 32); }
    }
    __syncthreads();
    long long it = 0;   // stages issued so far
    const int T = K / TK;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int pa = (int)(tile % 64), pb = (int)((tile / 64) % 64);
        const double* Ap = A + (long long)pa * 64 * K;
        const double* Bp = B + (long long)pb * 64 * K;
        double acc[2][4][2] = {};
        auto produce = [&](int ki) {
            const long long gs = it + ki;
            const int buf = (int)(gs % NSTAGE);
            double* As = smem + buf * STAGE_DBL;
            double* Bs = As + TILE_DBL;
            if (BULK) {
                if (warp == 0) {
                    if (gs >= NSTAGE) mbar_wait(&empty[buf], (int)(((gs / NSTAGE) - 1) & 1));
                    if (lane == 0) mbar_expect(&full[buf], 2u * 64 * TK * 8);
                    __syncwarp();
#pragma unroll
                    for (int r = lane; r < 64; r += 32) {
                        bulk_g2s(As + r * LDN, Ap + (long long)r * K + ki * TK, TK * 8, &full[buf]);
                        bulk_g2s(Bs + r * LDN, Bp + (long long)r * K + ki * TK, TK * 8, &full[buf]);
                    }
                }
            }
        };
        if (BULK) {
            for (int ki = 0; ki < NSTAGE - 1 && ki < T; ki++) produce(ki);
            for (int kt = 0; kt < T; kt++) {
                if (kt + NSTAGE - 1 < T) produce(kt + NSTAGE - 1);
                const long long gs = it + kt;
                const int buf = (int)(gs % NSTAGE);
                mbar_wait(&full[buf], (int)((gs / NSTAGE) & 1));
                const double* As = smem + buf * STAGE_DBL;
                mma_ktile<MEMN, MEMN>(acc, As, As + TILE_DBL, TK);
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[buf]);
            }
            it += T;
        }
        double* Ct = C + (tile % 1024) * 4096;
#pragma unroll
        for (int mi = 0; mi < 2; mi++)
#pragma unroll
            for (int ni = 0; ni < 4; ni++) {
                const int i = wr + mi * 8 + g, j = wc + ni * 8 + 2 * t;
                *reinterpret_cast<double2*>(Ct + i * 64 + j) = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
            }
    }
}

int main() {
    const int KMAX = 1024;
    double *A, *B, *C;
    cudaMalloc(&A, 8LL * 64 * 64 * KMAX);
    cudaMalloc(&B, 8LL * 64 * 64 * KMAX);
    cudaMalloc(&C, 8LL * 1024 * 4096);
    cudaMemset(A, 0, 8LL * 64 * 64 * KMAX);
    cudaMemset(B, 0, 8LL * 64 * 64 * KMAX);
    const int bytes = (NSTAGE * STAGE_DBL + 2 * NSTAGE) * 8;
    cudaFuncSetAttribute(kbulk<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kbulk<true>, NT, bytes);
    for (int K : {128, 576, 1024}) {
        const int grid = per * 148;
        const long long ntiles = (long long)grid * 40;
        kbulk<true><<<grid, NT, bytes>>>(A, B, C, K, ntiles);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        kbulk<true><<<grid, NT, bytes>>>(A, B, C, K, ntiles);
        cudaEventRecord(e1);
        cudaError_t err = cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double tf = 2.0 * 64 * 64 * K * (double)ntiles / (ms * 1e-3) / 1e12;
        printf("bulk MEMNxMEMN K=%5d %d CTA/SM %.2f TFLOP/s (%.1f%% of 37.15) %s\n", K, per, tf, 100 * tf / 37.15,
               cudaGetErrorString(err));
    }
    return 0;
}
