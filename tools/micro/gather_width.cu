// Random L2-resident gathers: does the load width matter?  n node records, every lane of
// every warp gathers a random record per step (indices from a coalesced u32 stream, like
// scol).  Variants: 32-byte records with one 256-bit load; 16-byte records with one
// 128-bit load; 16-byte records gathered as the enclosing 32-byte sector (256-bit load +
// select).  Prints gathers/ns.   nvcc -O3 -arch=sm_100a gather_width.cu -o gather_width
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>
#include <random>

template <int MODE>
__global__ void gk(const uint32_t *idx, int64_t m, const double *rec, double *out) {
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += 4 * nt) {
        uint32_t j[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) j[u] = i + u * nt < m ? idx[i + u * nt] : 0u;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            double a, b, c, d;
            if (MODE == 0) {  // 32-byte record, 256-bit load
                asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(rec + 4 * (int64_t)j[u]));
                acc += a + c;
            } else if (MODE == 1) {  // 16-byte record, 128-bit load
                asm volatile("ld.global.cg.v2.f64 {%0,%1}, [%2];" : "=d"(a), "=d"(b) : "l"(rec + 2 * (int64_t)j[u]));
                acc += a + b;
            } else if (MODE == 2) {  // 16-byte record, 256-bit load of its sector + select
                asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(rec + 4 * (int64_t)(j[u] >> 1)));
                acc += (j[u] & 1) ? c + d : a + b;
            } else {  // 32-byte stride, 128-bit load
                asm volatile("ld.global.cg.v2.f64 {%0,%1}, [%2];" : "=d"(a), "=d"(b) : "l"(rec + 4 * (int64_t)j[u]));
                acc += a + b;
            }
        }
    }
    if (acc == 1.2345) out[0] = acc;
}

int main() {
    const int64_t n = 1 << 20, m = 1 << 26;
    std::vector<uint32_t> h(m);
    std::mt19937 g(1);
    for (auto &v : h) v = g() & (n - 1);
    uint32_t *idx; double *rec, *out;
    cudaMalloc(&idx, m * 4); cudaMalloc(&rec, n * 32); cudaMalloc(&out, 8);
    cudaMemcpy(idx, h.data(), m * 4, cudaMemcpyHostToDevice);
    cudaMemset(rec, 0, n * 32);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const char *names[4] = {"rec32/ld256", "rec16/ld128", "rec16/ld256+sel", "rec32/ld128"};
    for (int rep = 0; rep < 2; ++rep)
        for (int mode = 0; mode < 4; ++mode) {
            for (int it = 0; it < 3; ++it) {
                if (it == 1) cudaEventRecord(e0);
                const int gsz = 148 * 4, bsz = 512;
                if (mode == 0) gk<0><<<gsz, bsz>>>(idx, m, rec, out);
                if (mode == 1) gk<1><<<gsz, bsz>>>(idx, m, rec, out);
                if (mode == 2) gk<2><<<gsz, bsz>>>(idx, m, rec, out);
                if (mode == 3) gk<3><<<gsz, bsz>>>(idx, m, rec, out);
            }
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("%-18s %.3f ms per %ld gathers = %.1f gathers/ns\n", names[mode], ms / 2, (long)m, m / (ms / 2 * 1e6));
        }
    // DRAM-resident random gathers: 16-byte records over 512 MB (the message array of config 1)
    {
        const int64_t nb = 1 << 25;  // 32 Mi records x 16 B
        double *big; cudaMalloc(&big, nb * 16); cudaMemset(big, 0, nb * 16);
        for (auto &v : h) v = g() & (nb - 1);
        cudaMemcpy(idx, h.data(), m * 4, cudaMemcpyHostToDevice);
        for (int it = 0; it < 3; ++it) {
            if (it == 1) cudaEventRecord(e0);
            gk<1><<<148 * 4, 512>>>(idx, m, big, out);
        }
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("dram rec16/ld128 over 512 MB: %.3f ms per %ld gathers = %.1f gathers/ns\n", ms / 2, (long)m, m / (ms / 2 * 1e6));
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
