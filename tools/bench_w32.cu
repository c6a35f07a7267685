// bench_w32.cu -- engine variant study: 128-thread CTAs, 64x64 CTA tile, four 32x32 warp tiles
// (16 DMMAs per 8 fragment loads per k-step), 2-stage cp.async pipeline, up to 3 CTAs per SM.
// MEMN x MEMN only, operands L2-resident as in bench_gemm.cu. Diagnostic only.
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>
constexpr int NTW = 128, TKW = 32, LDNW = TKW + 4, NSTW = 2, TILEW = 64 * LDNW;
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cpa16(double* s, const double* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(su32(s)), "l"(g));
}
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int MINB>
__global__ void __launch_bounds__(NTW, MINB) kw(const double* A, const double* B, double* C, int K, long long ntiles) {
    extern __shared__ double sm[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int wr = (warp >> 1) * 32, wc = (warp & 1) * 32;
    const int T = K / TKW;
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int pa = (int)(tile % 64), pb = (int)((tile / 64) % 64);
        const double* Ap = A + (long long)pa * 64 * K;
        const double* Bp = B + (long long)pb * 64 * K;
        double acc[4][4][2];
#pragma unroll
        for (int i = 0; i < 4; i++)
#pragma unroll
            for (int j = 0; j < 4; j++) acc[i][j][0] = acc[i][j][1] = 0.0;
        auto load = [&](int ki) {
            double* As = sm + (ki % NSTW) * 2 * TILEW;
            double* Bs = As + TILEW;
#pragma unroll
            for (int i = 0; i < 8; i++) {   // 64 rows x 16 copies of 16 B per operand over 128 threads
                const int e = tid + NTW * i, row = e >> 4, kk = (e & 15) * 2;
                cpa16(As + row * LDNW + kk, Ap + (long long)row * K + ki * TKW + kk);
                cpa16(Bs + row * LDNW + kk, Bp + (long long)row * K + ki * TKW + kk);
            }
            asm volatile("cp.async.commit_group;\n" ::);
        };
        __syncthreads();
        load(0);
        for (int kt = 0; kt < T; kt++) {
            if (kt + 1 < T) load(kt + 1); else asm volatile("cp.async.commit_group;\n" ::);
            asm volatile("cp.async.wait_group 1;\n" ::);
            __syncthreads();
            const double* As = sm + (kt % NSTW) * 2 * TILEW;
            const double* Bs = As + TILEW;
#pragma unroll
            for (int kk = 0; kk < TKW; kk += 4) {
                double a[4], b[4];
#pragma unroll
                for (int i = 0; i < 4; i++) a[i] = As[(wr + i * 8 + g) * LDNW + kk + t];
#pragma unroll
                for (int j = 0; j < 4; j++) b[j] = Bs[(wc + j * 8 + g) * LDNW + kk + t];
#pragma unroll
                for (int i = 0; i < 4; i++)
#pragma unroll
                    for (int j = 0; j < 4; j++) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
            }
            __syncthreads();
        }
        double* Ct = C + (tile % 1024) * 4096;
#pragma unroll
        for (int i = 0; i < 4; i++)
#pragma unroll
            for (int j = 0; j < 4; j++)
                *reinterpret_cast<double2*>(Ct + (wr + i * 8 + g) * 64 + wc + j * 8 + 2 * t) =
                    make_double2(acc[i][j][0], acc[i][j][1]);
    }
}
template <int MINB>
void run(double* A, double* B, double* C) {
    const int bytes = NSTW * 2 * TILEW * 8;
    cudaFuncSetAttribute(kw<MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kw<MINB>, NTW, bytes);
    for (int K : {128, 576, 1024}) {
        const int grid = per * 148;
        const long long ntiles = (long long)grid * 40;
        kw<MINB><<<grid, NTW, bytes>>>(A, B, C, K, ntiles);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        kw<MINB><<<grid, NTW, bytes>>>(A, B, C, K, ntiles);
        cudaEventRecord(e1);
        cudaError_t err = cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double tf = 2.0 * 64 * 64 * K * (double)ntiles / (ms * 1e-3) / 1e12;
        printf("w32 MINB=%d K=%5d %d CTA/SM %.2f TFLOP/s (%.1f%% of 37.15) %s\n", MINB, K, per, tf, 100 * tf / 37.15,
               cudaGetErrorString(err));
    }
}
int main() {
    const int KMAX = 1024;
    double *A, *B, *C;
    cudaMalloc(&A, 8LL * 64 * 64 * KMAX); cudaMalloc(&B, 8LL * 64 * 64 * KMAX); cudaMalloc(&C, 8LL * 1024 * 4096);
    cudaMemset(A, 0, 8LL * 64 * 64 * KMAX); cudaMemset(B, 0, 8LL * 64 * 64 * KMAX);
    run<3>(A, B, C);
    run<4>(A, B, C);
    return 0;
}
