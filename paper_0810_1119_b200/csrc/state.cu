// state.cu -- whole-state reductions and point reads of a message state.
//
//   launch_absmax    max |m| over both components of every message, as an ordered bit
//                    pattern (NaN > +inf > every finite value): the "not finite or biggest >
//                    blowup" test of the solve loop (solver.py:333-338) on a whole state,
//                    used after a serial sweep (the test reads the final state, not the
//                    values written on the way)
//   launch_gather    messages of a list of edge ids (compute_message, solver.py:114-143)
#include <float.h>
#include <math.h>

#include "gabp_internal.cuh"

namespace gabp {
namespace {

__device__ __forceinline__ unsigned long long abs_bits(double v) {
    return (unsigned long long)__double_as_longlong(v) & 0x7fffffffffffffffull;
}

__global__ void absmax_kernel(int64_t E, const double2 *a, unsigned long long *out) {
    unsigned long long m = 0ull;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E;
         e += (int64_t)gridDim.x * blockDim.x) {
        const double2 v = __ldcs(a + e);
        m = max(m, max(abs_bits(v.x), abs_bits(v.y)));
    }
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

__global__ void gather_msg_kernel(int64_t cnt, const int64_t *idx, const double2 *m,
                                  double2 *out) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < cnt) out[k] = m[idx[k]];
}

inline unsigned grid_for(int64_t E) {
    int64_t b = (E + 255) / 256;
    return (unsigned)(b < 1 ? 1 : (b > 148 * 16 ? 148 * 16 : b));
}

}  // namespace

cudaError_t launch_absmax(int64_t E, const double2 *a, unsigned long long *d_out,
                          cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(d_out, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess || E <= 0) return e;
    absmax_kernel<<<grid_for(E), 256, 0, st>>>(E, a, d_out);
    return cudaGetLastError();
}

cudaError_t launch_gather(int64_t cnt, const int64_t *idx, const double2 *m, double2 *out,
                          cudaStream_t st) {
    if (cnt <= 0) return cudaSuccess;
    gather_msg_kernel<<<(unsigned)((cnt + 255) / 256), 256, 0, st>>>(cnt, idx, m, out);
    return cudaGetLastError();
}

}  // namespace gabp
