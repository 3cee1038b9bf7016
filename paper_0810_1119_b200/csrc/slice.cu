// slice.cu -- broadcast-schedule solve sweep over the slice layout (lane per row).
//
// Layout (built by build_slices below): the swept rows are
// stably sorted by degree (descending) inside windows of kSortWin rows and cut into
// slices of 32 rows.  Slice s has width w_s = its largest degree; the q-th edge of the
// row in lane l lives at slot base_s + 32 q + l, so for every q a warp reads 32
// consecutive slots: scol/scoef and the messages move as fully coalesced 128-512 B
// requests with no shared-memory staging and no CTA barrier in the sweep.
//
// One launch = one sweep s of the solve loop (kModeSolve, broadcast, solver.py:232-272):
//   pass 1  lane i walks its edges in ascending k (the reference's np.add.at order):
//           incoming m_ki of S_{s-1} recomputed from k's aggregate of S_{s-2} and the own
//           message m_ik of S_{s-2} (exactly the operands launch s-1 used, so the same
//           bits); P_i += P_ki, N_i += P_ki mu_ki, residual row of x^{(s-2)}; the pair
//           (P_ki, P_ki mu_ki) is parked in the output slot (L2-resident until pass 2)
//   node    x_i = N_i / P_i (marginal of S_{s-1}), aggregate {P_i, P_i mu~_i} for launch s+1
//   pass 2  P_ij = -A_ij^2 / (P_i - P_ki), mu_ij = (P_i mu~_i - P_ki mu_ki) / A_ij,
//           coalesced store; change / blowup / singular statistics
// Launch 1 reads S_0 = 0 (solve_setup zeroes the ring), so its incoming messages are 0.
// Messages in this layout never leave the solve: the state API keeps the CSR layout.
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
#define GABP_SLICE_U 4
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

template <int DIST>
__global__ void __launch_bounds__(kSliceThreads, GABP_SLICE_CTAS)
    slice_kernel(const SweepArgs a) {
    __shared__ SliceSmem S;
    const int tid = threadIdx.x, lane = tid & 31;
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
    const bool resid = s >= 3;
    const bool rec = s >= 2;
    const double2 *min_ = a.msg[(s - 1) % 3];     // S_{s-1}: old value of each own message
    const double2 *mold2 = a.msg[(s - 2 + 3) % 3];  // S_{s-2}
    const double2 *aggp = a.agg[s & 1];           // aggregates of S_{s-2} (= (s-2) & 1)
    double2 *aggw = a.agg[(s - 1) & 1];           // aggregates of S_{s-1}, written here
    double2 *mout = a.msg[s % 3];
    const double *xprev = a.x[(s + 1) % 3];       // x^{(s-2)}
    double *xcur = a.x[(s - 1) % 3];
    double *pcur = a.p[(s - 1) % 3];
    double *xh = (a.xhist && s >= 2 && s - 1 <= a.xhist_rows) ? a.xhist + (s - 2) * a.n : nullptr;
    const uint32_t *__restrict__ scol = a.scol;
    const double *__restrict__ scoef = a.scoef;
    Stats st;
    st.lim = fmin(ctrl->blowup, DBL_MAX);

    const int64_t nwarps = (int64_t)gridDim.x * kSliceWarps;
    for (int64_t sl = (int64_t)blockIdx.x * kSliceWarps + (tid >> 5); sl < a.nslices;
         sl += nwarps) {
        const uint2 si = __ldg(a.slice_info + sl);  // {slot base, width}
        const uint4 li = __ldg(a.lane_info + sl * 32 + lane);  // {row, ebase, deg, -}
        const bool active = li.x != 0xffffffffu;
        const uint32_t i = active ? li.x : 0u, d = li.z;
        const uint32_t base = si.x + lane, w = si.y;
        double sp = 0.0, sn = 0.0, y = 0.0, rhs_i = 0.0;
        if (active) {
            const double2 nd = __ldg(reinterpret_cast<const double2 *>(a.nd) + i);  // {A_ii, pnum}
            sp = nd.x;
            sn = nd.y;
            if (resid) {
                y = nd.x * __ldcg(xprev + i);
                rhs_i = __ldg(a.rhs + i);
            }
        }
        // ---- pass 1: row sums in ascending k --------------------------------------------
        for (uint32_t q0 = 0; q0 < w; q0 += kU) {
            double c[kU], xg[kU];
            double2 ag[kU], o2[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const uint32_t q = q0 + u, slot = base + 32u * q;
                c[u] = 1.0;
                xg[u] = 0.0;
                ag[u] = make_double2(1.0, 1.0);
                o2[u] = make_double2(0.0, 0.0);
                if (q < d) {
                    c[u] = __ldg(scoef + slot);
                    const uint32_t col = __ldg(scol + slot);
                    if (rec) {
                        o2[u] = __ldcs(mold2 + slot);
                        ag[u] = __ldcg(aggp + col);
                    }
                    if (resid) xg[u] = __ldcg(xprev + col);
                }
            }
            double pin[kU], mu_in[kU];
            if (rec) {
                bool okp[kU], okm[kU];
                double pe[kU], num[kU];
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    pe[u] = ag[u].x - o2[u].x;
                    num[u] = ag[u].y - o2[u].x * o2[u].y;
                    if (q0 + u >= d) {  // idle slot: 1 / 1 stays on the fast path
                        pe[u] = 1.0;
                        num[u] = 1.0;
                    }
                }
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    pin[u] = ddiv_fast(-c[u] * c[u], pe[u], okp[u]);
                    mu_in[u] = ddiv_fast(num[u], c[u], okm[u]);
                }
#pragma unroll
                for (int u = 0; u < kU; ++u) {  // rare: operands outside the fast-path range
                    if (!okp[u]) pin[u] = div_slow(-c[u] * c[u], pe[u]);
                    if (!okm[u]) mu_in[u] = div_slow(num[u], c[u]);
                }
            } else {
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    pin[u] = 0.0;
                    mu_in[u] = 0.0;
                }
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const uint32_t q = q0 + u;
                if (q < d) {
                    const double pm = pin[u] * mu_in[u];  // (prec * mean), solver.py:243
                    sp = sp + pin[u];
                    sn = sn + pm;
                    if (resid) y = y + c[u] * xg[u];
                    mout[base + 32u * q] = make_double2(pin[u], pm);
                }
            }
        }
        // ---- node: marginal of S_{s-1}, aggregate, residual row -------------------------
        double nn = 0.0;
        if (active) {
            bool ok;
            double xi = ddiv_fast(sn, sp, ok);  // infer_marginals (solver.py:286)
            if (!ok) xi = div_slow(sn, sp);
            xcur[i] = xi;
            pcur[i] = sp;
            if (!(fabs(xi) <= DBL_MAX)) st.means_bad = 1u;
            if (xh) xh[i] = xi;
            nn = sp * xi;  // (sum_p * mu_tilde), solver.py:247-255
            if (sp == 0.0) st.agg_sing = min(st.agg_sing, i);
            aggw[i] = make_double2(sp, nn);
            if (resid) {
                const double r = y - rhs_i;
                st.rsq += r * r;
            }
        }
        // ---- pass 2: outgoing messages --------------------------------------------------
        for (uint32_t q0 = 0; q0 < w; q0 += kU) {
            double c[kU];
            double2 in[kU], old[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const uint32_t q = q0 + u, slot = base + 32u * q;
                c[u] = 1.0;
                in[u] = make_double2(0.0, 0.0);
                old[u] = make_double2(0.0, 0.0);
                if (q < d) {
                    in[u] = __ldcg(mout + slot);  // parked by pass 1 (same thread)
                    c[u] = __ldg(scoef + slot);
                    old[u] = __ldcs(min_ + slot);
                }
            }
            double pe[kU], num[kU], np_[kU], nm[kU];
            bool okp[kU], okm[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                pe[u] = sp - in[u].x;
                num[u] = nn - in[u].y;
                if (q0 + u >= d) {
                    pe[u] = 1.0;
                    num[u] = 1.0;
                }
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                np_[u] = ddiv_fast(-c[u] * c[u], pe[u], okp[u]);
                nm[u] = ddiv_fast(num[u], c[u], okm[u]);
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                if (!okp[u]) np_[u] = div_slow(-c[u] * c[u], pe[u]);
                if (!okm[u]) nm[u] = div_slow(num[u], c[u]);
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const uint32_t q = q0 + u;
                if (q < d) {
                    __stcs(mout + base + 32u * q, make_double2(np_[u], nm[u]));
                    st.edge(li.y + q, pe[u], np_[u], nm[u], old[u]);
                }
            }
        }
    }
    (void)DIST;
    sweep_epilogue<kSliceThreads, kModeSolve>(S.tail, a, s, resid, st, tid);
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

// width of each slice (degrees are sorted descending inside windows of whole slices)
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

__global__ void slice_fill_kernel(int64_t nslices, int64_t m, const uint32_t *srow,
                                  const uint32_t *sdeg, const uint32_t *row_ptr,
                                  const EdgeRec *er, const uint2 *info, uint4 *lane_info,
                                  uint32_t *scol, double *scoef) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= nslices * 32) return;
    const int64_t sl = p >> 5;
    const uint32_t l = (uint32_t)(p & 31);
    const uint2 si = info[sl];
    uint32_t row = 0xffffffffu, eb = 0, d = 0;
    if (p < m) {
        row = srow[p];
        eb = row_ptr[row];
        d = sdeg[p];
    }
    lane_info[p] = make_uint4(row, eb, d, 0u);
    for (uint32_t q = 0; q < si.y; ++q) {
        const uint32_t slot = si.x + 32u * q + l;
        if (q < d) {
            const EdgeRec r = er[eb + q];
            scol[slot] = r.col;
            scoef[slot] = r.coeff;
        } else {
            scol[slot] = 0u;
            scoef[slot] = 0.0;
        }
    }
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
    const int64_t nseg = (m + kSortWin - 1) / kSortWin;
    uint32_t *deg = nullptr, *rows = nullptr, *sdeg = nullptr, *srow = nullptr;
    int64_t *off = nullptr;
    unsigned long long *wslots = nullptr, *base = nullptr;
    SCHECK(cudaMallocAsync(&deg, sizeof(uint32_t) * m, st));
    SCHECK(cudaMallocAsync(&rows, sizeof(uint32_t) * m, st));
    SCHECK(cudaMallocAsync(&sdeg, sizeof(uint32_t) * m, st));
    SCHECK(cudaMallocAsync(&srow, sizeof(uint32_t) * m, st));
    SCHECK(cudaMallocAsync(&off, sizeof(int64_t) * (nseg + 1), st));
    SCHECK(cudaMallocAsync(&wslots, sizeof(unsigned long long) * (nslices + 1), st));
    SCHECK(cudaMallocAsync(&base, sizeof(unsigned long long) * (nslices + 1), st));
    slice_deg_kernel<<<grid_of(m), 256, 0, st>>>(g.row_lo, m, g.row_ptr, deg, rows);
    seg_offsets_kernel<<<grid_of(nseg + 1), 256, 0, st>>>(nseg, m, off);
    SCHECK(cudaGetLastError());
    // stable: rows of equal degree keep their order (structured grids stay contiguous)
    size_t tb = 0;
    SCHECK(cub::DeviceSegmentedRadixSort::SortPairsDescending(nullptr, tb, deg, sdeg, rows, srow,
                                                              m, nseg, off, off + 1, 0, 32, st));
    void *tmp = nullptr;
    SCHECK(cudaMallocAsync(&tmp, tb, st));
    SCHECK(cub::DeviceSegmentedRadixSort::SortPairsDescending(tmp, tb, deg, sdeg, rows, srow, m,
                                                              nseg, off, off + 1, 0, 32, st));
    cudaFreeAsync(tmp, st);
    slice_width_kernel<<<grid_of(nslices), 256, 0, st>>>(nslices, m, sdeg, wslots);
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
        SCHECK(cudaMallocAsync(&g.slice_info, sizeof(uint2) * nslices, st));
        SCHECK(cudaMallocAsync(&g.lane_info, sizeof(uint4) * nslices * 32, st));
        SCHECK(cudaMallocAsync(&g.scol, sizeof(uint32_t) * (nslots > 0 ? nslots : 1), st));
        SCHECK(cudaMallocAsync(&g.scoef, sizeof(double) * (nslots > 0 ? nslots : 1), st));
        slice_info_kernel<<<grid_of(nslices), 256, 0, st>>>(nslices, wslots, base,
                                                            g.slice_info);
        slice_fill_kernel<<<grid_of(nslices * 32), 256, 0, st>>>(
            nslices, m, srow, sdeg, g.row_ptr, g.er, g.slice_info, g.lane_info, g.scol,
            g.scoef);
        SCHECK(cudaGetLastError());
    }
    cudaFreeAsync(deg, st);
    cudaFreeAsync(rows, st);
    cudaFreeAsync(sdeg, st);
    cudaFreeAsync(srow, st);
    cudaFreeAsync(off, st);
    cudaFreeAsync(wslots, st);
    cudaFreeAsync(base, st);
    SCHECK(cudaStreamSynchronize(st));
    return rc;
}

cudaError_t prepare_slice_kernels() {
    int dev = 0, sms = 0, occ = 0;
    cudaError_t e;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess)
        return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, slice_kernel<0>, kSliceThreads,
                                                           0)) != cudaSuccess)
        return e;
    g_slice_grid = sms * (occ > 0 ? occ : 1);
    return cudaSuccess;
}

cudaError_t launch_slice_sweep(const SweepArgs &a, cudaStream_t st) {
    int64_t grid = g_slice_grid > 0 ? g_slice_grid : 148 * GABP_SLICE_CTAS;
    const int64_t need = (a.nslices + kSliceWarps - 1) / kSliceWarps;
    if (grid > need) grid = need > 0 ? need : 1;
    slice_kernel<0><<<(unsigned)grid, kSliceThreads, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace gabp
