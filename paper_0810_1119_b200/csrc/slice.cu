// slice.cu -- broadcast-schedule solve sweep over the slice layout (lane per row).
//
// Layout (build_slices below).  The swept rows are stably
// sorted by degree (descending) inside windows of kSortWin rows and cut into slices of 32
// rows; row r of the sort sits at "position" p = 32 * slice + lane.  Slice s has width
// w_s = its largest degree, and the q-th edge (ascending neighbour, = reference edge order)
// of the row in lane l lives at slot base_s + 32 q + l.  Nodes are numbered by position
// on this path (x, p and the aggregates live in position order; scol holds the neighbour's
// position; a rank's halo rows take positions after the owned ones), so every own-row and
// every per-edge stream is a fully coalesced warp access, and only the neighbour gathers
// are random (node arrays, L2-resident for the headline graph).
//
// State on this path: per edge slot the INCOMING pair I_ij^{(t)} = (P_ji, P_ji mu_ji) of
// S_t (message j -> i, the terms row i sums), a ring of three; per node the aggregate
// {P_i, P_i mu~_i} of S_t, a ring of three.  Launch s (one sweep, solver.py:232-272):
//   m_ij^{(s-2)} = msg(agg_i(S_{s-3}), I_ij^{(s-3)})      own outgoing messages, rebuilt
//   m_ij^{(s-1)} = msg(agg_i(S_{s-2}), I_ij^{(s-2)})      with launch s-1's / s-2's operands
//   I_ij^{(s-1)} = msg(agg_j(S_{s-2}), m_ij^{(s-2)})      = m_ji^{(s-1)}, exactly as row j
//                                                         built it (same operands, same bits)
//   P_i = A_ii + sum_j P_ji, N_i = A_ii mu_ii + sum_j P_ji mu_ji   ascending j (np.add.at)
//   x_i^{(s-1)} = N_i / P_i, agg_i(S_{s-1}) = {P_i, P_i x_i}, residual row of x^{(s-2)}
// with msg(agg, m) = (-A_ij^2 / (agg.P - m.P), (agg.N - m.P m.mu) / A_ij) (solver.py:249-257).
// One streaming pass per edge: 44 B read + 16 B written, no staging, no CTA barrier.  The
// statistics of sweep s-1's messages (max change, blowup, P_excl == 0) are taken here, one
// launch after the sweep itself and still one launch before its decision (Ctrl slots).
// Launch 1 sees I^{(0)} = 0 (solve_setup zeroes the ring); launch 2 uses m^{(0)} = 0.
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_radix_sort.cuh>
#include <stdio.h>

#include "sweep_common.cuh"

#ifndef GABP_SLICE_THREADS
#define GABP_SLICE_THREADS 256
#endif
#ifndef GABP_SLICE_CTAS
#define GABP_SLICE_CTAS 2
#endif
#ifndef GABP_SLICE_U
#define GABP_SLICE_U 2
#endif

namespace gabp {
namespace {

constexpr int kSliceThreads = GABP_SLICE_THREADS;
constexpr int kSliceWarps = kSliceThreads / 32;
constexpr int kU = GABP_SLICE_U;  // edges of one lane in flight per batch

struct SliceSmem {
    TailSmem<kSliceWarps> tail;
    int64_t sweep;
    int skip;
};

// msg(agg, m): the outgoing message of an edge from its row aggregate and the incoming
// pair, as (P, mu); ok is false when a division left the fast path.
__device__ __forceinline__ void edge_msg(double c, double pe, double num, double &P, double &mu,
                                         bool &ok) {
    bool o1, o2;
    P = ddiv_fast(-c * c, pe, o1);
    mu = ddiv_fast(num, c, o2);
    ok = o1 && o2;
}
__device__ __forceinline__ void edge_msg_slow(double c, double pe, double num, double &P,
                                              double &mu) {
    P = div_slow(-c * c, pe);
    mu = div_slow(num, c);
}

// PH: 1 = launch 1 (no incoming yet), 2 = launch 2 (m^{(0)} = 0, no residual), 3 = s >= 3
template <int PH>
__device__ __forceinline__ void slice_sweep(const SweepArgs &a, int64_t s, Stats &st, int lane) {
    const double2 *__restrict__ I2 = a.msg[(s + 1) % 3];   // I^{(s-2)}
    const double2 *__restrict__ I3 = a.msg[s % 3];         // I^{(s-3)}
    double2 *__restrict__ I1 = a.msg[(s - 1) % 3];         // I^{(s-1)}, written
    const double2 *__restrict__ agg2 = a.agg[(s + 1) % 3];  // agg(S_{s-2})
    const double2 *__restrict__ agg3 = a.agg[s % 3];        // agg(S_{s-3})
    double2 *__restrict__ agg1 = a.agg[(s - 1) % 3];        // agg(S_{s-1}), written
    const double *__restrict__ x2 = a.x[(s + 1) % 3];       // x^{(s-2)}
    double *__restrict__ x1 = a.x[(s - 1) % 3];
    double *__restrict__ p1 = a.p[(s - 1) % 3];
    double *xh = (a.xhist && s >= 2 && s - 1 <= a.xhist_rows) ? a.xhist + (s - 2) * a.n : nullptr;
    const uint32_t *__restrict__ scol = a.scol;
    const double *__restrict__ scoef = a.scoef;

    const int64_t nwarps = (int64_t)gridDim.x * kSliceWarps;
    for (int64_t sl = (int64_t)blockIdx.x * kSliceWarps + (threadIdx.x >> 5); sl < a.nslices;
         sl += nwarps) {
        const uint2 si = __ldg(a.slice_info + sl);  // {slot base, width}
        const int64_t p = sl * 32 + lane;
        const uint32_t d = __ldg(a.sdeg + p);
        const uint32_t row = __ldg(a.srow + p);   // ~0: padding lane (d == 0)
        const double2 nd = __ldg(a.snd + p);      // {A_ii, A_ii mu_ii}
        double2 a2 = make_double2(0.0, 0.0), a3 = make_double2(0.0, 0.0);
        double y = 0.0, rhs_i = 0.0;
        if (PH >= 2) a2 = __ldcg(agg2 + p);
        if (PH == 3) {
            a3 = __ldcg(agg3 + p);
            y = nd.x * __ldcg(x2 + p);
            rhs_i = __ldg(a.srhs + p);
        }
        double sp = nd.x, sn = nd.y;
        const uint32_t base = si.x + lane, w = si.y;
        if (PH == 1) {
            if (d > 0) {  // incoming messages of S_0 are +0: P + 0 (+ 0 ...) == P + 0
                sp = sp + 0.0;
                sn = sn + 0.0;
            }
        } else {
            for (uint32_t q0 = 0; q0 < w; q0 += kU) {
                double c[kU], xg[kU];
                uint32_t col[kU];
                double2 i2[kU], i3[kU], ag[kU];
#pragma unroll
                for (int u = 0; u < kU; ++u) {  // contiguous streams, all issued together
                    const uint32_t q = q0 + u, slot = base + 32u * q;
                    const bool v = q < d;
                    c[u] = v ? __ldcs(scoef + slot) : 1.0;
                    col[u] = v ? __ldcs(scol + slot) : 0u;
                    i2[u] = make_double2(0.0, 0.0);
                    i3[u] = make_double2(0.0, 0.0);
                    if (PH == 3) {
                        i2[u] = v ? __ldcs(I2 + slot) : make_double2(0.0, 0.0);
                        i3[u] = v ? __ldcs(I3 + slot) : make_double2(0.0, 0.0);
                    }
                }
#pragma unroll
                for (int u = 0; u < kU; ++u) {  // neighbour gathers
                    const bool v = q0 + u < d;
                    ag[u] = v ? __ldcg(agg2 + col[u]) : make_double2(1.0, 1.0);
                    xg[u] = 0.0;
                    if (PH == 3) xg[u] = v ? __ldcg(x2 + col[u]) : 0.0;
                }
                // own outgoing messages of sweeps s-2 (m2) and s-1 (m1)
                double m2p[kU], m2m[kU], m1p[kU], m1m[kU], pe1[kU], nu1[kU], pe2[kU], nu2[kU];
                bool ok = true;
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    const bool v = q0 + u < d;
                    pe1[u] = v ? a2.x - i2[u].x : 1.0;
                    nu1[u] = v ? a2.y - i2[u].y : 1.0;
                    bool o;
                    edge_msg(c[u], pe1[u], nu1[u], m1p[u], m1m[u], o);
                    ok = ok && o;
                    m2p[u] = 0.0;
                    m2m[u] = 0.0;
                    if (PH == 3) {
                        pe2[u] = v ? a3.x - i3[u].x : 1.0;
                        nu2[u] = v ? a3.y - i3[u].y : 1.0;
                        edge_msg(c[u], pe2[u], nu2[u], m2p[u], m2m[u], o);
                        ok = ok && o;
                    }
                }
                if (!ok) {  // rare: some operand outside the fast-path range
#pragma unroll
                    for (int u = 0; u < kU; ++u) {
                        edge_msg_slow(c[u], pe1[u], nu1[u], m1p[u], m1m[u]);
                        if (PH == 3) edge_msg_slow(c[u], pe2[u], nu2[u], m2p[u], m2m[u]);
                    }
                }
                // incoming of S_{s-1}: m_ji^{(s-1)} rebuilt from agg_j(S_{s-2}) and m_ij^{(s-2)}
                double ip[kU], im[kU], pe[kU], num[kU];
                ok = true;
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    const bool v = q0 + u < d;
                    pe[u] = v ? ag[u].x - m2p[u] : 1.0;
                    num[u] = v ? ag[u].y - m2p[u] * m2m[u] : 1.0;
                    bool o;
                    edge_msg(c[u], pe[u], num[u], ip[u], im[u], o);
                    ok = ok && o;
                }
                if (!ok) {
#pragma unroll
                    for (int u = 0; u < kU; ++u) edge_msg_slow(c[u], pe[u], num[u], ip[u], im[u]);
                }
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    const uint32_t q = q0 + u;
                    if (q < d) {
                        const double pm = ip[u] * im[u];  // (prec * mean), solver.py:243
                        sp = sp + ip[u];
                        sn = sn + pm;
                        if (PH == 3) y = y + c[u] * xg[u];
                        __stcs(I1 + base + 32u * q, make_double2(ip[u], pm));
                        // statistics of sweep s-1 (its message m1 against m2 = S_{s-2})
                        const double d1 = fabs(m1p[u] - m2p[u]), d2 = fabs(m1m[u] - m2m[u]);
                        st.chg = d1 > st.chg ? d1 : st.chg;
                        st.chg = d2 > st.chg ? d2 : st.chg;
                        if (!(fabs(m1p[u]) <= st.lim) || !(fabs(m1m[u]) <= st.lim))
                            st.out_of_range = 1u;
                        if (pe1[u] == 0.0) st.sing = min(st.sing, __ldg(a.row_ptr + row) + q);
                    }
                }
            }
        }
        // ---- node: marginal of S_{s-1}, aggregate, residual row of x^{(s-2)} -------------
        if (row != 0xffffffffu) {
            bool ok;
            double xi = ddiv_fast(sn, sp, ok);  // infer_marginals (solver.py:286)
            if (!ok) xi = div_slow(sn, sp);
            x1[p] = xi;
            p1[p] = sp;
            if (!(fabs(xi) <= DBL_MAX)) st.means_bad = 1u;
            if (xh) xh[row] = xi;
            const double nn = sp * xi;  // (sum_p * mu_tilde), solver.py:247-255
            if (sp == 0.0) st.agg_sing = min(st.agg_sing, row);
            agg1[p] = make_double2(sp, nn);
            if (PH == 3) {
                const double r = y - rhs_i;
                st.rsq += r * r;
            }
        }
    }
}

__global__ void __launch_bounds__(kSliceThreads, GABP_SLICE_CTAS) slice_kernel(const SweepArgs a) {
    __shared__ SliceSmem S;
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
    Stats st;
    st.lim = fmin(a.ctrl->blowup, DBL_MAX);
    if (s >= 3)
        slice_sweep<3>(a, s, st, tid & 31);
    else if (s == 2)
        slice_sweep<2>(a, s, st, tid & 31);
    else
        slice_sweep<1>(a, s, st, tid & 31);
    sweep_epilogue<kSliceThreads, kModeSolve, 1>(S.tail, a, s, s >= 3, st, tid);
}

int g_slice_grid = 0;

// ---- build -------------------------------------------------------------------------------
constexpr int kSortWin = 1024;  // rows per degree-sort window (a multiple of 32)

__global__ void slice_deg_kernel(int64_t row_lo, int64_t m, const uint32_t *row_ptr,
                                 uint32_t *deg, uint32_t *rows) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= m) return;
    const int64_t i = row_lo + r;
    deg[r] = row_ptr[i + 1] - row_ptr[i];
    rows[r] = (uint32_t)i;
}

__global__ void seg_offsets_kernel(int64_t nseg, int64_t m, int64_t *off) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k > nseg) return;
    off[k] = k * kSortWin < m ? k * kSortWin : m;
}

// slots of each slice (degrees are sorted descending inside windows of whole slices)
__global__ void slice_width_kernel(int64_t nslices, int64_t m, const uint32_t *sdeg,
                                   unsigned long long *wslots) {
    const int64_t sl = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (sl >= nslices) return;
    uint32_t w = 0;
    for (int l = 0; l < 32; ++l) {
        const int64_t p = sl * 32 + l;
        if (p < m && sdeg[p] > w) w = sdeg[p];
    }
    wslots[sl] = 32ull * w;
}

__global__ void slice_info_kernel(int64_t nslices, const unsigned long long *wslots,
                                  const unsigned long long *base, uint2 *info) {
    const int64_t sl = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (sl >= nslices) return;
    info[sl] = make_uint2((uint32_t)base[sl], (uint32_t)(wslots[sl] / 32));
}

// position of every local node: owned rows by the sort, halo rows after the slices
__global__ void slice_pos_kernel(int64_t n, int64_t row_lo, int64_t row_hi, int64_t m_pad,
                                 int64_t m, const uint32_t *sorted_rows, uint32_t *pos) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < m) pos[sorted_rows[k]] = (uint32_t)k;
    if (k < row_lo) pos[k] = (uint32_t)(m_pad + k);
    if (k < n - row_hi) pos[row_hi + k] = (uint32_t)(m_pad + row_lo + k);
}

__global__ void slice_lane_kernel(int64_t npos, int64_t m, const uint32_t *sorted_rows,
                                  const uint32_t *sorted_deg, uint32_t *srow, uint32_t *sdeg) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= npos) return;
    srow[p] = p < m ? sorted_rows[p] : 0xffffffffu;
    sdeg[p] = p < m ? sorted_deg[p] : 0u;
}

__global__ void slice_fill_kernel(int64_t nslices, const uint32_t *srow, const uint32_t *sdeg,
                                  const uint32_t *row_ptr, const EdgeRec *er,
                                  const uint32_t *pos, const uint2 *info, uint32_t *scol,
                                  double *scoef) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= nslices * 32) return;
    const uint2 si = info[p >> 5];
    const uint32_t l = (uint32_t)(p & 31), d = sdeg[p];
    const uint32_t eb = d ? row_ptr[srow[p]] : 0u;
    for (uint32_t q = 0; q < si.y; ++q) {
        const uint32_t slot = si.x + 32u * q + l;
        if (q < d) {
            const EdgeRec r = er[eb + q];
            scol[slot] = pos[r.col];
            scoef[slot] = r.coeff;
        } else {
            scol[slot] = 0u;
            scoef[slot] = 0.0;
        }
    }
}

__global__ void slice_nodes_kernel(int64_t npos, const uint32_t *srow, const NodeRec *nd,
                                   const double *rhs, double2 *snd, double *srhs) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= npos) return;
    const uint32_t r = srow[p];
    if (r != 0xffffffffu) {
        snd[p] = make_double2(nd[r].diag, nd[r].pnum);
        srhs[p] = rhs[r];
    } else {
        snd[p] = make_double2(1.0, 0.0);
        srhs[p] = 0.0;
    }
}

__global__ void gather_pos_kernel(int64_t lo, int64_t cnt, const uint32_t *pos, const double *in,
                                  double *out) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < cnt) out[lo + k] = in[pos[lo + k]];
}

__global__ void map_pos_kernel(int64_t cnt, const uint32_t *pos, uint32_t *idx) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < cnt) idx[k] = pos[idx[k]];
}

inline unsigned grid_of(int64_t n) { return (unsigned)((n + 255) / 256 > 0 ? (n + 255) / 256 : 1); }

#define SCHECK(call)                                                                        \
    do {                                                                                    \
        cudaError_t _e = (call);                                                            \
        if (_e != cudaSuccess) {                                                            \
            snprintf(err, errlen, "%s: %s", #call, cudaGetErrorString(_e));                 \
            return _e == cudaErrorMemoryAllocation ? GABP_ENOMEM : GABP_ECUDA;              \
        }                                                                                   \
    } while (0)

}  // namespace

int build_slices(DeviceGraph &g, cudaStream_t st, char *err, size_t errlen) {
    const int64_t m = g.row_hi - g.row_lo;
    if (m <= 0) return GABP_OK;
    const int64_t nslices = (m + 31) / 32;
    const int64_t m_pad = nslices * 32;
    const int64_t npos = m_pad + (g.n - m);
    const int64_t nseg = (m + kSortWin - 1) / kSortWin;
    uint32_t *deg = nullptr, *rows = nullptr, *sorted_deg = nullptr, *sorted_rows = nullptr;
    int64_t *off = nullptr;
    unsigned long long *wslots = nullptr, *base = nullptr;
    SCHECK(cudaMallocAsync(&deg, sizeof(uint32_t) * m, st));
    SCHECK(cudaMallocAsync(&rows, sizeof(uint32_t) * m, st));
    SCHECK(cudaMallocAsync(&sorted_deg, sizeof(uint32_t) * m, st));
    SCHECK(cudaMallocAsync(&sorted_rows, sizeof(uint32_t) * m, st));
    SCHECK(cudaMallocAsync(&off, sizeof(int64_t) * (nseg + 1), st));
    SCHECK(cudaMallocAsync(&wslots, sizeof(unsigned long long) * (nslices + 1), st));
    SCHECK(cudaMallocAsync(&base, sizeof(unsigned long long) * (nslices + 1), st));
    slice_deg_kernel<<<grid_of(m), 256, 0, st>>>(g.row_lo, m, g.row_ptr, deg, rows);
    seg_offsets_kernel<<<grid_of(nseg + 1), 256, 0, st>>>(nseg, m, off);
    SCHECK(cudaGetLastError());
    // stable: rows of equal degree keep their order (structured grids stay contiguous)
    size_t tb = 0;
    SCHECK(cub::DeviceSegmentedRadixSort::SortPairsDescending(
        nullptr, tb, deg, sorted_deg, rows, sorted_rows, m, nseg, off, off + 1, 0, 32, st));
    void *tmp = nullptr;
    SCHECK(cudaMallocAsync(&tmp, tb, st));
    SCHECK(cub::DeviceSegmentedRadixSort::SortPairsDescending(
        tmp, tb, deg, sorted_deg, rows, sorted_rows, m, nseg, off, off + 1, 0, 32, st));
    cudaFreeAsync(tmp, st);
    slice_width_kernel<<<grid_of(nslices), 256, 0, st>>>(nslices, m, sorted_deg, wslots);
    SCHECK(cudaMemsetAsync(wslots + nslices, 0, sizeof(unsigned long long), st));
    size_t sb = 0;
    SCHECK(cub::DeviceScan::ExclusiveSum(nullptr, sb, wslots, base, nslices + 1, st));
    SCHECK(cudaMallocAsync(&tmp, sb, st));
    SCHECK(cub::DeviceScan::ExclusiveSum(tmp, sb, wslots, base, nslices + 1, st));
    cudaFreeAsync(tmp, st);
    unsigned long long nslots = 0;
    SCHECK(cudaMemcpyAsync(&nslots, base + nslices, sizeof(nslots), cudaMemcpyDeviceToHost, st));
    SCHECK(cudaStreamSynchronize(st));
    int rc = GABP_OK;
    if (nslots >= 0xffffffffull) {
        rc = GABP_EINVAL;  // caller keeps the tile layout only
        snprintf(err, errlen, "slice layout needs %llu slots (> 32-bit)", nslots);
    } else {
        g.nslices = nslices;
        g.nslots = (int64_t)nslots;
        g.npos = npos;
        SCHECK(cudaMallocAsync(&g.slice_info, sizeof(uint2) * nslices, st));
        SCHECK(cudaMallocAsync(&g.pos, sizeof(uint32_t) * (g.n > 0 ? g.n : 1), st));
        SCHECK(cudaMallocAsync(&g.srow, sizeof(uint32_t) * npos, st));
        SCHECK(cudaMallocAsync(&g.sdeg, sizeof(uint32_t) * npos, st));
        SCHECK(cudaMallocAsync(&g.snd, sizeof(double2) * npos, st));
        SCHECK(cudaMallocAsync(&g.srhs, sizeof(double) * npos, st));
        SCHECK(cudaMallocAsync(&g.scol, sizeof(uint32_t) * (nslots > 0 ? nslots : 1), st));
        SCHECK(cudaMallocAsync(&g.scoef, sizeof(double) * (nslots > 0 ? nslots : 1), st));
        slice_info_kernel<<<grid_of(nslices), 256, 0, st>>>(nslices, wslots, base,
                                                            g.slice_info);
        const int64_t big = m > g.n - m ? m : g.n - m;
        slice_pos_kernel<<<grid_of(big), 256, 0, st>>>(g.n, g.row_lo, g.row_hi, m_pad, m,
                                                       sorted_rows, g.pos);
        slice_lane_kernel<<<grid_of(npos), 256, 0, st>>>(npos, m, sorted_rows, sorted_deg,
                                                         g.srow, g.sdeg);
        slice_fill_kernel<<<grid_of(m_pad), 256, 0, st>>>(nslices, g.srow, g.sdeg, g.row_ptr,
                                                          g.er, g.pos, g.slice_info, g.scol,
                                                          g.scoef);
        SCHECK(cudaGetLastError());
    }
    cudaFreeAsync(deg, st);
    cudaFreeAsync(rows, st);
    cudaFreeAsync(sorted_deg, st);
    cudaFreeAsync(sorted_rows, st);
    cudaFreeAsync(off, st);
    cudaFreeAsync(wslots, st);
    cudaFreeAsync(base, st);
    SCHECK(cudaStreamSynchronize(st));
    return rc;
}

// per-position copies of the node priors and rhs (after every prior computation)
cudaError_t refresh_slice_nodes(const DeviceGraph &g, cudaStream_t st) {
    if (g.nslices == 0) return cudaSuccess;
    slice_nodes_kernel<<<grid_of(g.npos), 256, 0, st>>>(g.npos, g.srow, g.nd, g.rhs, g.snd,
                                                        g.srhs);
    return cudaGetLastError();
}

// out[i] = in[pos[i]] for local rows [lo, lo + cnt): position order -> row order
cudaError_t slice_to_rows(const DeviceGraph &g, int64_t lo, int64_t cnt, const double *in,
                          double *out, cudaStream_t st) {
    if (cnt <= 0) return cudaSuccess;
    gather_pos_kernel<<<grid_of(cnt), 256, 0, st>>>(lo, cnt, g.pos, in, out);
    return cudaGetLastError();
}

// idx[k] = pos[idx[k]]: a rank's halo lists in position numbering
cudaError_t slice_map_index(const DeviceGraph &g, uint32_t *idx, int64_t cnt, cudaStream_t st) {
    if (cnt <= 0) return cudaSuccess;
    map_pos_kernel<<<grid_of(cnt), 256, 0, st>>>(cnt, g.pos, idx);
    return cudaGetLastError();
}

cudaError_t prepare_slice_kernels() {
    int dev = 0, sms = 0, occ = 0;
    cudaError_t e;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess)
        return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, slice_kernel, kSliceThreads, 0)) !=
        cudaSuccess)
        return e;
    g_slice_grid = sms * (occ > 0 ? occ : 1);
    return cudaSuccess;
}

cudaError_t launch_slice_sweep(const SweepArgs &a, cudaStream_t st) {
    int64_t grid = g_slice_grid > 0 ? g_slice_grid : 148 * GABP_SLICE_CTAS;
    const int64_t need = (a.nslices + kSliceWarps - 1) / kSliceWarps;
    if (grid > need) grid = need > 0 ? need : 1;
    slice_kernel<<<(unsigned)grid, kSliceThreads, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace gabp
