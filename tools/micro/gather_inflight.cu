// Random 16-byte gathers over a 512 MB array (DRAM resident): achieved gathers/ns against
// the number of gathers in flight per SM, for register loads (ld.global.cg) and cp.async
// into shared memory.   nvcc -O3 -arch=sm_100a gather_inflight.cu -o gather_inflight
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>
#include <random>

template <int U, bool ASYNC>
__global__ void gk(const uint32_t *idx, int64_t m, const double2 *rec, double *out) {
    extern __shared__ double2 sm[];
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i + (U - 1) * nt < m; i += U * nt) {
        uint32_t j[U];
#pragma unroll
        for (int u = 0; u < U; ++u) j[u] = idx[i + u * nt];
        if (ASYNC) {
#pragma unroll
            for (int u = 0; u < U; ++u)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(sm + u * blockDim.x + threadIdx.x)), "l"(rec + j[u]) : "memory");
            asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
#pragma unroll
            for (int u = 0; u < U; ++u) acc += sm[u * blockDim.x + threadIdx.x].x;
        } else {
            double2 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                asm volatile("ld.global.cg.v2.f64 {%0,%1}, [%2];" : "=d"(v[u].x), "=d"(v[u].y) : "l"(rec + j[u]));
#pragma unroll
            for (int u = 0; u < U; ++u) acc += v[u].x;
        }
    }
    if (acc == 1.2345) out[0] = acc;
}

// the parallel sweep's traffic mix per gather: 16 B edge record + 16 B own old message
// streamed in, one random 16-byte gather, 16 B streamed out
template <int U>
__global__ void mixk(const int4 *er, int64_t m, const double2 *rec, const double2 *oldm, double2 *outm) {
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i + (U - 1) * nt < m; i += U * nt) {
        int4 e[U];
        double2 v[U], o[U];
#pragma unroll
        for (int u = 0; u < U; ++u) e[u] = __ldcs(er + i + u * nt);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            asm volatile("ld.global.cg.v2.f64 {%0,%1}, [%2];" : "=d"(v[u].x), "=d"(v[u].y) : "l"(rec + (uint32_t)e[u].x));
            o[u] = __ldcs(oldm + i + u * nt);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) __stcs(outm + i + u * nt, make_double2(v[u].x + o[u].x, v[u].y + o[u].y));
    }
}

template <int U, bool ASYNC>
float run(int ctas_per_sm, int threads, const uint32_t *idx, int64_t m, const double2 *rec, double *out) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const size_t smem = ASYNC ? (size_t)U * threads * 16 : 0;
    cudaFuncSetAttribute(gk<U, ASYNC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int it = 0; it < 3; ++it) {
        if (it == 1) cudaEventRecord(e0);
        gk<U, ASYNC><<<148 * ctas_per_sm, threads, smem>>>(idx, m, rec, out);
    }
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    return ms / 2;
}

int main() {
    const int64_t nb = 1 << 25, m = 1 << 25;  // 32 Mi records x 16 B; 32 Mi gathers per launch
    std::vector<uint32_t> h(m);
    std::mt19937 g(1);
    for (auto &v : h) v = g() & (nb - 1);
    uint32_t *idx; double2 *rec; double *out;
    cudaMalloc(&idx, m * 4); cudaMalloc(&rec, nb * 16); cudaMalloc(&out, 8);
    cudaMemcpy(idx, h.data(), m * 4, cudaMemcpyHostToDevice);
    cudaMemset(rec, 0, nb * 16);
    struct { int ctas, threads; } cfg[] = {{1, 128}, {1, 256}, {1, 512}, {2, 512}, {2, 1024}};
    for (auto c : cfg) {
        const int thr = c.ctas * c.threads;
        float a1 = run<1, false>(c.ctas, c.threads, idx, m, rec, out);
        float a4 = run<4, false>(c.ctas, c.threads, idx, m, rec, out);
        float a8 = run<8, false>(c.ctas, c.threads, idx, m, rec, out);
        float b4 = run<4, true>(c.ctas, c.threads, idx, m, rec, out);
        float b8 = run<8, true>(c.ctas, c.threads, idx, m, rec, out);
        printf("threads/SM %4d | ldg x1 %5.1f  x4 %5.1f  x8 %5.1f | cp.async x4 %5.1f  x8 %5.1f   (gathers/ns; in flight/SM = threads x U)\n",
               thr, m / (a1 * 1e6), m / (a4 * 1e6), m / (a8 * 1e6), m / (b4 * 1e6), m / (b8 * 1e6));
    }
    {
        int4 *er; double2 *oldm, *outm;
        cudaMalloc(&er, m * 16); cudaMalloc(&oldm, m * 16); cudaMalloc(&outm, m * 16);
        std::vector<int4> he(m);
        for (int64_t i = 0; i < m; ++i) he[i] = make_int4((int)h[i], 0, 0, 0);
        cudaMemcpy(er, he.data(), m * 16, cudaMemcpyHostToDevice);
        cudaMemset(oldm, 0, m * 16);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        for (int thr : {256, 512, 1024}) {
            for (int it = 0; it < 3; ++it) {
                if (it == 1) cudaEventRecord(e0);
                mixk<4><<<148 * 2, thr>>>(er, m, rec, oldm, outm);
            }
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 2;
            printf("mix (16 B record + 16 B old in, random 16 B gather, 16 B out) threads/SM %4d x4: %.3f ms = %.1f gathers/ns, %.2f TB/s at 176 B per gather\n",
                   2 * thr, ms, m / (ms * 1e6), m * 176.0 / (ms * 1e9));
        }
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
