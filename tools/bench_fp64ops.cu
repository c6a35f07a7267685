#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, int which) {
    double v = 1.0 + threadIdx.x * 1e-3, acc = 0;
    long long t0 = clock64();
    for (int j = 0; j < 16; j++) {
        double r;
        if (which == 0) r = sqrt(v);
        else if (which == 1) r = __dsqrt_rn(v);
        else if (which == 2) r = __drcp_rn(v);
        else if (which == 3) r = 1.0 / v;
        else if (which == 4) r = log(v);
        else if (which == 5) r = exp(-v);
        else r = v * 1.0000001;
        acc += r;
        v = r + 1.0;   // dependent chain
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[which] = (t1 - t0) / 16; out[0] = acc; }
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 8 * 8);
    const char* nm[] = {"sqrt", "__dsqrt_rn", "__drcp_rn", "1.0/x", "log", "exp", "dmul"};
    for (int w = 0; w < 7; w++) { k<<<1, 32>>>(o, c, w); cudaDeviceSynchronize(); }
    for (int w = 0; w < 7; w++) { k<<<1, 32>>>(o, c, w); }
    long long h[8]; cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
    for (int w = 0; w < 7; w++) printf("%-12s %lld cycles per dependent op\n", nm[w], h[w]);
}
