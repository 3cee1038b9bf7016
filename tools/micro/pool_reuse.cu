// Probe: cost of cudaMallocAsync reuse across streams with a retained default pool.
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
static double now() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
int main() {
    cudaFree(0);
    cudaMemPool_t pool;
    cudaDeviceGetDefaultMemPool(&pool, 0);
    uint64_t keep = UINT64_MAX;
    printf("set threshold: %d\n", (int)cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    for (int it = 0; it < 6; ++it) {
        cudaStream_t s;
        cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
        void *a = nullptr, *b = nullptr;
        double t0 = now();
        cudaMallocAsync(&a, 420u << 20, s);
        double t1 = now();
        cudaMallocAsync(&b, (size_t)1800 << 20, s);
        double t2 = now();
        cudaMemsetAsync(b, 0, 1 << 20, s);
        cudaFreeAsync(a, s);
        cudaStreamSynchronize(s);
        uint64_t res = 0;
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &res);
        cudaFreeAsync(b, s);
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
        printf("it %d: alloc420 %.3f ms alloc1800 %.3f ms reserved %.2f GB\n", it, t1 - t0, t2 - t1, res / 1e9);
    }
    // same stream reuse
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    for (int it = 0; it < 3; ++it) {
        void *b = nullptr;
        double t0 = now();
        cudaMallocAsync(&b, (size_t)1800 << 20, s);
        double t1 = now();
        cudaFreeAsync(b, s);
        cudaStreamSynchronize(s);
        printf("same stream it %d: alloc1800 %.3f ms\n", it, t1 - t0);
    }
    return 0;
}
