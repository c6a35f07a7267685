// Accuracy of the kernels' exp_neg / sqrt_fast / covf against libm (exp, sqrt) on the GPU
// (tests/test_gpu_devmath.py builds and runs it).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o check_exp check_exp.cu
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
#include "../paper_1905_00141_b200/csrc/mra_device.cuh"
using namespace mra;

__device__ double ulp_err(double got, double ref) {
    if (ref == 0.0) return got == 0.0 ? 0.0 : 1e30;
    const double u = ldexp(1.0, ilogb(ref) - 52);
    return fabs(got - ref) / u;
}
__global__ void k(long long n, double xmax, double* maxu, unsigned long long* seed_out) {
    double m = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double x = xmax * ((double)i + 0.5) / (double)n;   // dense grid over [0, xmax)
        const double e = exp_neg(x), r = exp(-x);
        if (r > 1e-300) m = fmax(m, ulp_err(e, r));
    }
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax((unsigned long long*)maxu, __double_as_longlong(m));
}
__global__ void ksqrt(long long n, double* maxu) {
    double m = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        // log-uniform q over [1e-30, 1e6]
        const double q = exp(-69.0776 + 82.8931 * ((double)i + 0.5) / (double)n);
        m = fmax(m, ulp_err(sqrt_fast(q), sqrt(q)));
    }
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax((unsigned long long*)maxu, __double_as_longlong(m));
}
// the scaled branch of sqrt_fast (q < 2^-120): log-uniform q over [1e-100, 1e-30]; plus the exact special cases
__global__ void ksqrt_tiny(long long n, double* maxu, int* bad) {
    double m = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double q = exp(-230.2585 + 161.1810 * ((double)i + 0.5) / (double)n);
        m = fmax(m, ulp_err(sqrt_fast(q), sqrt(q)));
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (sqrt_fast(0.0) != 0.0) atomicAdd(bad, 1);
        if (exp_neg(708.0) != 0.0 || exp_neg(1e300) != 0.0 || exp_neg(nan("")) != 0.0) atomicAdd(bad, 1);
        if (exp_neg(0.0) != 1.0) atomicAdd(bad, 1);
    }
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax((unsigned long long*)maxu, __double_as_longlong(m));
}
__global__ void kcov(long long n, int kind, double* maxrel) {
    CovP c;
    c.kind = kind; c.s2 = 1.7; c.rho = 0.3; c.xs = 1.0; c.ys = 1.0;
    c.ir = (kind == 0 ? 1.0 : 1.7320508075688772935) / c.rho;
    double m = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double x1 = (double)(i % 9973) / 9973.0 * 10.0, y1 = (double)(i % 7919) / 7919.0 * 10.0;
        const double x2 = (double)(i % 104729) / 104729.0 * 10.0, y2 = (double)(i % 1299709) / 1299709.0 * 10.0;
        const double d = sqrt((x1 - x2) * (x1 - x2) + (y1 - y2) * (y1 - y2)) * c.ir;
        const double ref = kind == 0 ? c.s2 * exp(-d) : c.s2 * (1.0 + d) * exp(-d);
        if (ref > 1e-290) m = fmax(m, fabs(covf(c, x1, y1, x2, y2) - ref) / ref);
    }
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax((unsigned long long*)maxrel, __double_as_longlong(m));
}

int main() {
    double* d; cudaMalloc(&d, 8);
    for (double xmax : {1.0, 20.0, 700.0}) {
        cudaMemset(d, 0, 8);
        k<<<1184, 256>>>(200000000LL, xmax, d, nullptr);
        double h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("exp_neg vs libm exp(-x), x in [0, %g) on 2e8 points: max %.2f ulp\n", xmax, h);
    }
    cudaMemset(d, 0, 8);
    ksqrt<<<1184, 256>>>(200000000LL, d);
    double h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("sqrt_fast vs sqrt, q in [1e-30, 1e6] on 2e8 points: max %.2f ulp\n", h);
    {
        int* bad; cudaMalloc(&bad, 4); cudaMemset(bad, 0, 4); cudaMemset(d, 0, 8);
        ksqrt_tiny<<<1184, 256>>>(20000000LL, d, bad);
        int hb; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
        printf("sqrt_fast tiny q in [1e-100, 1e-30] on 2e7 points: max %.2f ulp; special cases failed: %d\n", h, hb);
    }
    for (int kind = 0; kind < 2; kind++) {
        cudaMemset(d, 0, 8);
        kcov<<<1184, 256>>>(100000000LL, kind, d);
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("covf kind %d vs libm formula on 1e8 pairs: max relative %.3e\n", kind, h);
    }
    return 0;
}
