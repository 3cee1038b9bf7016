// CDP2 tail launch from a kernel captured in a CUDA graph: the child runs after the parent
// grid, before the next node; launched only when the parent decides so.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void child(int *x) { if (threadIdx.x == 0) atomicAdd(&x[1], 1); }
__global__ void parent(int *x, int v) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        x[0] += 1;
        if (v) child<<<148, 256, 0, cudaStreamTailLaunch>>>(x);
    }
}
__global__ void after(int *x) { if (threadIdx.x == 0 && blockIdx.x == 0) x[2] = x[1]; }
#define T(c) do { cudaError_t e = (c); if (e != cudaSuccess) { printf("FAIL %s: %s\n", #c, cudaGetErrorString(e)); return 1; } } while (0)
int main() {
    int *x; T(cudaMalloc(&x, 12)); T(cudaMemset(x, 0, 12));
    cudaStream_t st; T(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    cudaGraph_t g; T(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    for (int k = 0; k < 4; ++k) { parent<<<148, 256, 0, st>>>(x, k == 2); after<<<1, 32, 0, st>>>(x); }
    T(cudaStreamEndCapture(st, &g));
    cudaGraphExec_t ex; T(cudaGraphInstantiate(&ex, g, 0));
    T(cudaGraphLaunch(ex, st)); T(cudaStreamSynchronize(st));
    int h[3]; T(cudaMemcpy(h, x, 12, cudaMemcpyDeviceToHost));
    printf("graph: parent %d child-blocks %d seen-by-next %d (expect 4, 148, 148)\n", h[0], h[1], h[2]);
    // timing: 200 parents without child launches, graph vs plain
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a, st);
    for (int k = 0; k < 200; ++k) parent<<<148, 256, 0, st>>>(x, 0);
    cudaEventRecord(b, st); T(cudaStreamSynchronize(st));
    float ms; cudaEventElapsedTime(&ms, a, b); printf("200 parent launches: %.1f us each\n", ms * 1e3 / 200);
    return 0;
}
