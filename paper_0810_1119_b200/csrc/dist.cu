// dist.cu -- device side of the multi-rank solve.
//
// Per launch s each rank runs sweep_kernel in dist mode (its last CTA publishes the
// rank's statistics in dstats instead of deciding), the host reduces dstats across ranks
// (NCCL all-reduce, or an in-process reduction for the one-GPU partition test), then
// finish_kernel applies the global statistics and takes the decision for sweep s-2 --
// identical on every rank -- and the halo kernels move the node aggregates {P_j, P_j mu~_j}
// and marginals x_j the next launch gathers for remote neighbours.
#include "gabp_internal.cuh"

namespace gabp {
namespace {

__global__ void finish_kernel(const SweepArgs a) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    volatile Ctrl *c = a.ctrl;
    if (c->done) return;
    const int64_t s = c->next_sweep;
    const int slot = (int)(s % kStatSlots);
    const int mslot = (int)((s - a.msg_lag) % kStatSlots);  // sweep of the message stats
    const double *d = a.dstats;
    c->change_bits[mslot] = (unsigned long long)__double_as_longlong(d[0]);
    c->msg_nonfinite[mslot] = (int32_t)d[1];
    c->means_nonfinite[(s - 1) % kStatSlots] = d[2] > 0.0 ? 1 : 0;
    c->singular_min[mslot] = d[3] > -1e299 ? (unsigned long long)(-d[3]) : kNoIndex;
    c->agg_singular[slot] = d[4] > -1e299 ? (unsigned long long)(-d[4]) : kNoIndex;
    decide_sweep(c, a, s - 2, d[5]);
    const int nslot = (int)((s + 1) % kStatSlots);
    c->change_bits[nslot] = 0ull;
    c->msg_nonfinite[nslot] = 0;
    c->means_nonfinite[nslot] = 0;
    c->agg_singular[nslot] = kNoIndex;
    c->singular_min[nslot] = kNoIndex;
    c->next_sweep = s + 1;
    __threadfence();
}

// Halo buffers: cnt records of 4 doubles per node -- {P, P mu~, x, 0}: the node state of
// the slice path verbatim, or the tile path's aggregate and marginal.
// After finish_kernel of launch s (next_sweep == s+1) the launch-s outputs are the state
// of S_{s-1} (rec[(s-1)%3], or agg[(s-1)%3] and x[(s-1)%3]): exactly what launch s+1
// gathers for remote neighbours (indices are local ids, or positions on the slice path).
__global__ void halo_pack_kernel(const SweepArgs a, const uint32_t *idx, int64_t cnt,
                                 double *buf, int pre_finish) {
    const int64_t s = ((volatile Ctrl *)a.ctrl)->next_sweep - (pre_finish ? 0 : 1);
    double4 *b4 = reinterpret_cast<double4 *>(buf);
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < cnt;
         k += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t i = idx[k];
        if (a.slice_path) {
            const NodeState r = a.rec[(s - 1) % 3][i];
            b4[k] = make_double4(r.P, r.P * r.x, r.x, 0.0);
        } else {
            const double2 g = a.agg[(s - 1) % 3][i];
            b4[k] = make_double4(g.x, g.y, a.x[(s - 1) % 3][i], 0.0);
        }
    }
}

__global__ void halo_unpack_kernel(const SweepArgs a, const uint32_t *idx, int64_t cnt,
                                   const double *buf, int pre_finish) {
    const int64_t s = ((volatile Ctrl *)a.ctrl)->next_sweep - (pre_finish ? 0 : 1);
    const double4 *b4 = reinterpret_cast<const double4 *>(buf);
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < cnt;
         k += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t i = idx[k];
        const double4 v = b4[k];
        if (a.slice_path) {
            NodeState &r = a.rec[(s - 1) % 3][i];
            r.P = v.x;
            r.x = v.z;
        } else {
            a.agg[(s - 1) % 3][i] = make_double2(v.x, v.y);
            a.x[(s - 1) % 3][i] = v.z;
        }
    }
}

// ---- diagonal layout (dia.cu) -------------------------------------------------------------
// Launch s of the diagonal kernel decides sweep s-1: its statistics slots are sweep s's, the
// aggregates' singular test is sweep s+1's, the residual is x^{(s-1)}'s; the published (and
// now reduced) statistics are sweep s-1's (dia.cu dia_epilogue).
__global__ void dia_finish_kernel(const SweepArgs a) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    volatile Ctrl *c = a.ctrl;
    if (c->done) return;
    const int64_t s = c->next_sweep;
    const int ms = (int)((s - 1) % kStatSlots);
    const double *d = a.dstats;
    c->change_bits[ms] = (unsigned long long)__double_as_longlong(d[0]);
    c->msg_nonfinite[ms] = (int32_t)d[1];
    c->means_nonfinite[ms] = d[2] > 0.0 ? 1 : 0;
    c->singular_min[ms] = d[3] > -1e299 ? (unsigned long long)(-d[3]) : kNoIndex;
    c->agg_singular[ms] = d[4] > -1e299 ? (unsigned long long)(-d[4]) : kNoIndex;
    decide_sweep(c, a, s - 1, d[5]);
    const int n1 = (int)((s + 1) % kStatSlots), n2 = (int)((s + 2) % kStatSlots);
    c->change_bits[n1] = 0ull;
    c->msg_nonfinite[n1] = 0;
    c->means_nonfinite[n1] = 0;
    c->singular_min[n1] = kNoIndex;
    c->agg_singular[n2] = kNoIndex;
    c->next_sweep = s + 1;
    __threadfence();
}

// Halo of the diagonal layout: per exchanged node {P_i, x_i} of S_s and the row's incoming
// messages on the listed diagonals -- the ones a neighbour across the cut reads as twins
// (the peer's row j needs m_{j -> i} = row i's incoming slot from j for its update of
// m_{i -> j}).  s < 0: the sweep of the launch just run (next_sweep, minus one after its
// finish kernel).
__global__ void dia_pack_kernel(const SweepArgs a, const uint32_t *idx, int64_t cnt,
                                double *buf, DiaHalo h, int64_t s_fix, int post_finish) {
    const int64_t s = s_fix >= 0 ? s_fix
                                 : ((volatile Ctrl *)a.ctrl)->next_sweep - (post_finish ? 1 : 0);
    const double *p = a.p[s % 3], *x = a.x[s % 3];
    const double2 *m = a.msg[s & 1];
    const int w = 2 + 2 * h.nd;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < cnt;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = idx[k];
        double *b = buf + k * w;
        b[0] = p[i];
        b[1] = x[i];
        for (int q = 0; q < h.nd; ++q) {
            const double2 v = m[(int64_t)h.diag[q] * a.dia_nl + i];
            b[2 + 2 * q] = v.x;
            b[3 + 2 * q] = v.y;
        }
    }
}
__global__ void dia_unpack_kernel(const SweepArgs a, const uint32_t *idx, int64_t cnt,
                                  const double *buf, DiaHalo h, int64_t s_fix,
                                  int post_finish) {
    const int64_t s = s_fix >= 0 ? s_fix
                                 : ((volatile Ctrl *)a.ctrl)->next_sweep - (post_finish ? 1 : 0);
    double *p = a.p[s % 3], *x = a.x[s % 3];
    double2 *m = a.msg[s & 1];
    const int w = 2 + 2 * h.nd;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < cnt;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = idx[k];
        const double *b = buf + k * w;
        p[i] = b[0];
        x[i] = b[1];
        for (int q = 0; q < h.nd; ++q)
            m[(int64_t)h.diag[q] * a.dia_nl + i] = make_double2(b[2 + 2 * q], b[3 + 2 * q]);
    }
}

inline unsigned blocks_for(int64_t cnt) {
    int64_t b = (cnt + 255) / 256;
    if (b < 1) b = 1;
    if (b > 148 * 8) b = 148 * 8;
    return (unsigned)b;
}

}  // namespace

cudaError_t launch_finish(const SweepArgs &a, cudaStream_t st) {
    finish_kernel<<<1, 32, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_dia_finish(const SweepArgs &a, cudaStream_t st) {
    dia_finish_kernel<<<1, 32, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_dia_pack(const SweepArgs &a, const uint32_t *idx, int64_t cnt, double *buf,
                            const DiaHalo &h, int64_t s_fix, int post_finish, cudaStream_t st) {
    if (cnt <= 0) return cudaSuccess;
    dia_pack_kernel<<<blocks_for(cnt), 256, 0, st>>>(a, idx, cnt, buf, h, s_fix, post_finish);
    return cudaGetLastError();
}

cudaError_t launch_dia_unpack(const SweepArgs &a, const uint32_t *idx, int64_t cnt,
                              const double *buf, const DiaHalo &h, int64_t s_fix,
                              int post_finish, cudaStream_t st) {
    if (cnt <= 0) return cudaSuccess;
    dia_unpack_kernel<<<blocks_for(cnt), 256, 0, st>>>(a, idx, cnt, buf, h, s_fix, post_finish);
    return cudaGetLastError();
}

cudaError_t launch_halo_pack(const SweepArgs &a, const uint32_t *idx, int64_t cnt, double *buf,
                             cudaStream_t st, int pre_finish) {
    if (cnt <= 0) return cudaSuccess;
    halo_pack_kernel<<<blocks_for(cnt), 256, 0, st>>>(a, idx, cnt, buf, pre_finish);
    return cudaGetLastError();
}

cudaError_t launch_halo_unpack(const SweepArgs &a, const uint32_t *idx, int64_t cnt,
                               const double *buf, cudaStream_t st, int pre_finish) {
    if (cnt <= 0) return cudaSuccess;
    halo_unpack_kernel<<<blocks_for(cnt), 256, 0, st>>>(a, idx, cnt, buf, pre_finish);
    return cudaGetLastError();
}

}  // namespace gabp
