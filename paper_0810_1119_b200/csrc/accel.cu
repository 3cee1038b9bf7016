// accel.cu -- device side of the Steffensen / Aitken wrappers (acceleration.py).
//
// The restart of a Steffensen cycle replaces the mean messages of the current state with
// the componentwise (gated) Aitken extrapolant of three samples (acceleration.py:74-96,
// 177-183); for an E-edge graph that is one HBM pass over three message arrays, so it runs
// here, next to the states, instead of round-tripping 3 x 16 E bytes to the host.  Every
// operation is the numpy expression's, in its order, with IEEE division and no FMA
// contraction (-fmad=false), so the extrapolant is bitwise the reference's:
//   denom = x2 - 2.0 * x1 + x0;  y = |denom| >= guard ? x0 - (x1 - x0)^2 / denom : x2
//   gated: |denom| >= stability * np.maximum(|x1 - x0|, |x2 - x1|) ? y : x2
// np.maximum propagates NaN (then the gate is false); fmax would not, hence nan_max.
#include <float.h>
#include <math.h>

#include "gabp_internal.cuh"

namespace gabp {
namespace {

__device__ __forceinline__ double nan_max(double a, double b) {
    return (a != a || b != b) ? (a + b) : fmax(a, b);  // a + b is NaN when either is
}

__global__ void extrapolate_kernel(int64_t E, const double2 *m0, const double2 *m1, double2 *m2,
                                   double guard, double stability, int gated) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E;
         e += (int64_t)gridDim.x * blockDim.x) {
        const double x0 = m0[e].y, x1 = m1[e].y, x2 = m2[e].y;
        const double denom = x2 - 2.0 * x1 + x0;
        double y = x2;
        if (fabs(denom) >= guard) {
            const double diff = x1 - x0;
            y = x0 - diff * diff / denom;
        }
        if (gated) {
            const double d1 = fabs(x1 - x0), d2 = fabs(x2 - x1);
            if (!(fabs(denom) >= stability * nan_max(d1, d2))) y = x2;
        }
        m2[e].y = y;
    }
}

// max over |v| as ordered bit patterns: NaN > +inf > every finite value
__device__ __forceinline__ unsigned long long abs_bits(double v) {
    return (unsigned long long)__double_as_longlong(v) & 0x7fffffffffffffffull;
}

__global__ void absmax_kernel(int64_t E, const double2 *a, const double2 *b, int which,
                              unsigned long long *out) {
    unsigned long long m = 0ull;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E;
         e += (int64_t)gridDim.x * blockDim.x) {
        const double2 v = a[e];
        if (which == 0) {  // both components of one state
            const unsigned long long p = abs_bits(v.x), q = abs_bits(v.y);
            m = max(m, max(p, q));
        } else {  // |a.mu - b.mu|
            m = max(m, abs_bits(v.y - b[e].y));
        }
    }
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

inline unsigned grid_for(int64_t E) {
    int64_t b = (E + 255) / 256;
    return (unsigned)(b < 1 ? 1 : (b > 148 * 16 ? 148 * 16 : b));
}

}  // namespace

cudaError_t launch_extrapolate(int64_t E, const double2 *m0, const double2 *m1, double2 *m2,
                               double guard, double stability, int gated, cudaStream_t st) {
    if (E <= 0) return cudaSuccess;
    extrapolate_kernel<<<grid_for(E), 256, 0, st>>>(E, m0, m1, m2, guard, stability, gated);
    return cudaGetLastError();
}

cudaError_t launch_absmax(int64_t E, const double2 *a, const double2 *b, int which,
                          unsigned long long *d_out, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(d_out, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess || E <= 0) return e;
    absmax_kernel<<<grid_for(E), 256, 0, st>>>(E, a, b, which, d_out);
    return cudaGetLastError();
}

}  // namespace gabp
