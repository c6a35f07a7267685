// fp64_peak.cu -- N8 microbenchmark: measured fp64 peak of a B200 (DMMA m8n8k4 tensor path and
// DFMA), all SMs, CUDA events. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
    double acc[8][2];
    for (int i = 0; i < 8; i++) acc[i][0] = acc[i][1] = 0.0;
    double a = 1e-9 * threadIdx.x, b = 1e-9 * blockIdx.x;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
    for (int i = 0; i < 8; i++) s += acc[i][0] + acc[i][1];
    if (s == 12345.0) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
    double acc[8];
    for (int i = 0; i < 8; i++) acc[i] = threadIdx.x * 1e-3 + i;
    const double a = 0.999999, b = 1e-7;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) acc[i] = fma(acc[i], a, b);
    }
    double s = 0;
    for (int i = 0; i < 8; i++) s += acc[i];
    if (s == 12345.0) out[0] = s;
}

int main() {
    int dev = 0, nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    double* out;
    cudaMalloc(&out, 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int warps = 4; warps <= 16; warps *= 2) {
        const int threads = 32 * warps, iters = 20000;
        for (int blocksPerSm = 1; blocksPerSm <= 2; blocksPerSm++) {
            int grid = nsm * blocksPerSm;
            dmma_loop<<<grid, threads>>>(out, 100);
            cudaEventRecord(a);
            dmma_loop<<<grid, threads>>>(out, iters);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            double flops = 2.0 * 256 * 8 * (double)iters * warps * grid;
            printf("DMMA m8n8k4: %2d warps/CTA x %d CTA/SM: %.2f TFLOP/s\n", warps, blocksPerSm, flops / ms / 1e9);
            dfma_loop<<<grid, threads>>>(out, 100);
            cudaEventRecord(a);
            dfma_loop<<<grid, threads>>>(out, iters);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            flops = 2.0 * 8 * (double)iters * threads * grid;
            printf("DFMA       : %2d warps/CTA x %d CTA/SM: %.2f TFLOP/s\n", warps, blocksPerSm, flops / ms / 1e9);
        }
    }
    return 0;
}
