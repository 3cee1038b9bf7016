// FP64 dependent-chain latency on the GPU: DADD, DFMA, division (div.rn.f64).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *out, long long *cyc, double a, double b, int n) {
    double x = a, y = b;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = x + y;            // DADD chain
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, y, 1e-3);  // DFMA chain
    long long t2 = clock64();
    for (int i = 0; i < n; ++i) x = y / x;            // division chain
    long long t3 = clock64();
    float f = (float)x;
    for (int i = 0; i < n; ++i) f = f * 1.0001f + 1e-6f;  // FFMA chain
    long long t4 = clock64();
    out[threadIdx.x] = x + f;
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
__global__ void tput(double *out, long long *cyc, double a, int n) {
    double x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { x0 = 1.5 / x0; x1 = 1.5 / x1; x2 = 1.5 / x2; x3 = 1.5 / x3; }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[4] = t1 - t0;
}
int main() {
    double *o; long long *c, h[8];
    cudaMalloc(&o, 1 << 24); cudaMalloc(&c, 64);
    int n = 4096;
    k<<<1, 32>>>(o, c, 1.0, 1e-9, n);
    k<<<1, 32>>>(o, c, 1.0, 1e-9, n);
    cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
    printf("latency cycles: DADD %.1f  DFMA %.1f  DDIV %.1f  FFMA %.1f\n", h[0] / (double)n,
           h[1] / (double)n, h[2] / (double)n, h[3] / (double)n);
    for (int w : {1, 4, 8, 16, 32}) {
        tput<<<148, 32 * w>>>(o, c, 1.0, n);
        cudaMemcpy(h + 4, c + 4, 8, cudaMemcpyDeviceToHost);
        printf("div throughput, %2d warps/SM x4 indep chains: %.1f cycles per 4 divs/warp\n", w,
               h[4] / (double)n);
    }
    return 0;
}
