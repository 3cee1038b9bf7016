// dense.cu -- broadcast sweep for a dense A (linear detection, BASELINE config 3).
//
// Storage: A is K x K row-major; messages are a padded K x K matrix M[k][j] = m_{k->j}
// (sender-major, i.e. the out-slot layout of the sparse path; the diagonal and the exact
// zeros of A -- non-edges in the reference, linalg.py:81-82 -- hold zero messages).
// One launch s = two kernels:
//
//   column walk  one CTA per 32 columns: all four warps stream 32-row blocks of A and M
//                (coalesced 256/512-byte row segments) into a 4-stage shared-memory ring
//                with LDGSTS while lane l of warp 0 walks column i0+l -- the incoming
//                messages of node i in ascending sender order, exactly the order of the
//                reference's np.add.at (solver.py:242-243) -- and A's column for the
//                residual row of x^{(s-2)}.  Non-edges are skipped, so the sums are bitwise
//                those of the sparse path.  Writes P_i, P_i*mu~_i, x^{(s-1)}, residual
//                partials.  (A thread-per-column walk without staging ran 3.8 ms at K=4096:
//                4096 threads cannot keep HBM busy; the staged walk runs ~0.2 ms.)
//   edge tiles   32 x 32 tiles: m_ij = f(P_i, N_i, m_ji, A_ij) (broadcast_sweep,
//                solver.py:249-257) with m_ji read from the transposed tile through shared
//                memory; max change / blowup / singular statistics; the last CTA runs the
//                solve decision for sweep s-2 (same Ctrl protocol as the sparse kernel).
#include <float.h>
#include <math.h>

#include "gabp_internal.cuh"

namespace gabp {
namespace {

constexpr int kTile = 32;

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

constexpr int kColRows = 32;     // rows of A / M per pipeline stage
constexpr int kColStages = 4;
constexpr int kColCta = 128;     // 32 columns per CTA; warp 0 sums, all warps load

__device__ __forceinline__ uint32_t s_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cpa16(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s_u32(dst)), "l"(src));
}
__device__ __forceinline__ void cpa8(void *dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s_u32(dst)), "l"(src));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cpa_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

struct ColSmem {
    double A[kColStages][kColRows][32];
    double2 M[kColStages][kColRows][32];
    double X[kColStages][kColRows];
    int64_t sweep;
    int skip;
};

// Stage rows [k0, k0 + kColRows) of columns [i0, i0 + 32) of A and M (and x^{(s-2)}[k]).
__device__ __forceinline__ void col_stage(ColSmem &S, int st, int64_t k0, int64_t i0, int64_t K,
                                          const double *A, const double2 *M,
                                          const double *xprev, int tid) {
    for (int q = tid; q < kColRows * 32; q += kColCta) {
        const int r = q >> 5, c = q & 31;
        const int64_t k = k0 + r, i = i0 + c;
        if (k < K && i < K) {
            cpa8(&S.A[st][r][c], A + k * K + i);
            cpa16(&S.M[st][r][c], M + k * K + i);
        }
    }
    if (xprev && tid < kColRows && k0 + tid < K) cpa8(&S.X[st][tid], xprev + k0 + tid);
}

// Column walk of launch s (solve mode): lane l of warp 0 walks column i0 + l in ascending
// row order from a 4-stage shared-memory ring the whole CTA fills with LDGSTS.
__global__ void __launch_bounds__(kColCta) dense_column_kernel(const SweepArgs a,
                                                               const DenseArgs d) {
    extern __shared__ __align__(16) unsigned char col_raw[];
    ColSmem &S = *reinterpret_cast<ColSmem *>(col_raw);
    const int tid = threadIdx.x;
    if (tid == 0) {
        volatile Ctrl *vc = a.ctrl;
        const int64_t s = vc->next_sweep;
        S.skip = vc->done || s > vc->max_iter + 2;
        S.sweep = s;
    }
    __syncthreads();
    if (S.skip) return;
    const int64_t s = S.sweep;
    const bool resid = s >= 3;
    const int64_t K = d.K;
    const double2 *M = d.msg[(s - 1) % 3];
    const double *xprev = resid ? a.x[(s - 2) % 3] : nullptr;
    const int64_t i0 = (int64_t)blockIdx.x * 32;
    const int64_t nstage = (K + kColRows - 1) / kColRows;
    for (int p = 0; p < kColStages - 1; ++p) {
        if (p < nstage) col_stage(S, p, p * kColRows, i0, K, d.A, M, xprev, tid);
        cpa_commit();
    }
    const int lane = tid & 31;
    const int64_t i = i0 + lane;
    const bool sum_lane = tid < 32 && i < K;
    double sp = 0.0, sn = 0.0, y = 0.0;
    if (sum_lane) {
        const NodeRec nd = a.nd[i];
        sp = nd.diag;
        sn = nd.pnum;
        y = resid ? nd.diag * xprev[i] : 0.0;
    }
    for (int64_t t = 0; t < nstage; ++t) {
        cpa_wait<kColStages - 2>();
        __syncthreads();  // stage t landed for every thread; stage t-1 fully consumed
        const int64_t tn = t + kColStages - 1;
        if (tn < nstage)
            col_stage(S, (int)(tn % kColStages), tn * kColRows, i0, K, d.A, M, xprev, tid);
        cpa_commit();
        if (sum_lane) {
            const int st = (int)(t % kColStages);
            const int64_t k0 = t * kColRows;
            const int rows = (int)((K - k0) < kColRows ? (K - k0) : kColRows);
            for (int r = 0; r < rows; ++r) {  // ascending k: the reference's order
                const int64_t k = k0 + r;
                const double akj = S.A[st][r][lane];
                if (k == i || akj == 0.0) continue;  // no edge
                const double2 m = S.M[st][r][lane];
                sp = sp + m.x;
                sn = sn + m.x * m.y;
                if (resid) y = y + akj * S.X[st][r];
            }
        }
    }
    cpa_wait<0>();
    if (tid >= 32) return;
    double rsq = 0.0;
    unsigned bad = 0u, agg_sing = 0xffffffffu;
    if (sum_lane) {
        double *xcur = a.x[(s - 1) % 3];
        double *pcur = a.p[(s - 1) % 3];
        double *xh = (a.xhist && s >= 2 && s - 1 <= a.xhist_rows) ? a.xhist + (s - 2) * a.n
                                                                   : nullptr;
        const double xi = sn / sp;  // solver.py:286
        xcur[i] = xi;
        pcur[i] = sp;
        if (xh) xh[i] = xi;
        if (!(fabs(xi) <= DBL_MAX)) bad = 1u;
        d.node[i] = make_double2(sp, sp * xi);  // P_i, P_i mu~_i (solver.py:247/255)
        if (sp == 0.0) agg_sing = (unsigned)i;
        if (resid) {
            const double r = y - a.rhs[i];
            rsq = r * r;
        }
    }
    rsq = warp_sum_d(rsq);
    bad = __reduce_or_sync(~0u, bad);
    agg_sing = __reduce_min_sync(~0u, agg_sing);
    if (tid == 0) {
        if (resid) a.rsq_part[blockIdx.x] = rsq;
        if (bad) atomicOr(&a.ctrl->means_nonfinite[(s - 1) % kStatSlots], 1);
        if (agg_sing != 0xffffffffu)
            atomicMin(&a.ctrl->agg_singular[s % kStatSlots], (unsigned long long)agg_sing);
    }
}

struct TileSmem {
    double2 t[kTile][kTile + 1];  // M^{(s-1)}[J][I] block, padded against bank conflicts
    double red_d[8];
    unsigned red_u[8];
    int64_t sweep;
    int skip;
    int last;
};

__global__ void __launch_bounds__(256) dense_edge_kernel(const SweepArgs a, const DenseArgs d,
                                                         int64_t col_blocks) {
    __shared__ TileSmem S;
    const int tid = threadIdx.x;
    Ctrl *ctrl = a.ctrl;
    if (tid == 0) {
        volatile Ctrl *vc = ctrl;
        const int64_t s = vc->next_sweep;
        S.skip = vc->done || s > vc->max_iter + 2;
        S.sweep = s;
    }
    __syncthreads();
    if (S.skip) return;
    const int64_t s = S.sweep;
    const int64_t K = d.K;
    const double2 *M = d.msg[(s - 1) % 3];
    double2 *Mo = d.msg[s % 3];
    const double lim = fmin(ctrl->blowup, DBL_MAX);
    const int64_t nt = (K + kTile - 1) / kTile;
    double chg = 0.0;
    unsigned oor = 0u;
    unsigned long long sing = ~0ull;
    const int tx = tid & 31, ty = tid >> 5;  // 32 x 8 threads
    for (int64_t t = blockIdx.x; t < nt * nt; t += gridDim.x) {
        const int64_t I = (t / nt) * kTile, J = (t % nt) * kTile;
        // stage M[J + r][I + c] (the reverse messages of this tile)
        for (int r = ty; r < kTile; r += 8) {
            const int64_t jr = J + r, ic = I + tx;
            S.t[r][tx] = (jr < K && ic < K) ? __ldcg(M + jr * K + ic) : make_double2(0.0, 0.0);
        }
        __syncthreads();
        for (int r = ty; r < kTile; r += 8) {
            const int64_t i = I + r, j = J + tx;
            if (i >= K || j >= K || i == j) continue;
            const double c = __ldg(d.A + i * K + j);
            if (c == 0.0) continue;
            const double2 rev = S.t[tx][r];  // m_{j->i}
            const double2 nd = __ldg(d.node + i);
            const double pe = nd.x - rev.x;
            const double num = nd.y - rev.x * rev.y;
            const double np_ = (-c * c) / pe;
            const double nm = num / c;
            const int64_t e = i * K + j;
            const double2 old = __ldcs(M + e);
            __stcs(Mo + e, make_double2(np_, nm));
            if (pe == 0.0 && (unsigned long long)e < sing) sing = (unsigned long long)e;
            const double d1 = fabs(np_ - old.x), d2 = fabs(nm - old.y);
            chg = d1 > chg ? d1 : chg;
            chg = d2 > chg ? d2 : chg;
            if (!(fabs(np_) <= lim) || !(fabs(nm) <= lim)) oor = 1u;
        }
        __syncthreads();
    }
    // CTA reductions + last-CTA decision (the sparse kernel's protocol)
    const int warp = tid >> 5, lane = tid & 31;
    chg = warp_max_d(chg);
    oor = __reduce_or_sync(~0u, oor);
    const unsigned sl = (unsigned)(sing & 0xffffffffu), sh = (unsigned)(sing >> 32);
    const unsigned msh = __reduce_min_sync(~0u, sh);
    const unsigned msl = __reduce_min_sync(~0u, sh == msh ? sl : 0xffffffffu);
    if (lane == 0) {
        S.red_d[warp] = chg;
        S.red_u[warp] = oor;
        if (msh != 0xffffffffu || msl != 0xffffffffu) {
            const unsigned long long v = ((unsigned long long)msh << 32) | msl;
            atomicMin(&ctrl->singular_min[s % kStatSlots], v);
        }
    }
    __syncthreads();
    if (tid == 0) {
        double bc = 0.0;
        unsigned f = 0u;
        for (int w = 0; w < 8; ++w) {
            bc = fmax(bc, S.red_d[w]);
            f |= S.red_u[w];
        }
        const int slot = (int)(s % kStatSlots);
        if (bc > 0.0)
            atomicMax(&ctrl->change_bits[slot], (unsigned long long)__double_as_longlong(bc));
        if (f) atomicOr(&ctrl->msg_nonfinite[slot], 1);
        __threadfence();
        const unsigned tkt = atomicAdd(&ctrl->ticket, 1u);
        S.last = (tkt == gridDim.x - 1);
    }
    __syncthreads();
    if (!S.last) return;
    __threadfence();
    double part = 0.0;
    if (s >= 3) {
        volatile const double *rp = a.rsq_part;
        for (int64_t b = tid; b < col_blocks; b += 256) part += rp[b];
    }
    part = warp_sum_d(part);
    if (lane == 0) S.red_d[warp] = part;
    __syncthreads();
    if (tid == 0) {
        double rsq_t = 0.0;
        for (int w = 0; w < 8; ++w) rsq_t += S.red_d[w];
        decide_sweep(ctrl, a, s - 2, rsq_t);
        const int nslot = (int)((s + 1) % kStatSlots);
        ctrl->change_bits[nslot] = 0ull;
        ctrl->msg_nonfinite[nslot] = 0;
        ctrl->means_nonfinite[nslot] = 0;
        ctrl->agg_singular[nslot] = kNoIndex;
        ctrl->singular_min[nslot] = kNoIndex;
        ctrl->ticket = 0u;
        ctrl->next_sweep = s + 1;
        __threadfence();
    }
}

int g_edge_grid = 0;

}  // namespace

cudaError_t launch_dense_sweep(const SweepArgs &a, const DenseArgs &d, cudaStream_t st) {
    if (g_edge_grid == 0) {
        cudaFuncSetAttribute(dense_column_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(ColSmem));
        int dev = 0, sms = 0, occ = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, dense_edge_kernel, 256, 0);
        g_edge_grid = sms * (occ > 0 ? occ : 1);
    }
    const int64_t cb = (d.K + 31) / 32;
    dense_column_kernel<<<(unsigned)cb, kColCta, sizeof(ColSmem), st>>>(a, d);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int64_t nt = (d.K + kTile - 1) / kTile;
    int64_t grid = g_edge_grid;
    if (grid > nt * nt) grid = nt * nt;
    dense_edge_kernel<<<(unsigned)grid, 256, 0, st>>>(a, d, cb);
    return cudaGetLastError();
}

}  // namespace gabp
