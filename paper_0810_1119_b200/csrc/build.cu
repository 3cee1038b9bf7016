// build.cu -- device-side GaussianGraph construction (graph.py:63-120 re-designed).
//
// Input: the SymSystem storage (linalg.py:34-62) as upper-triangle pairs
// (i < j, A_ij != 0) in arbitrary order, already in HBM.  Output (gabp_internal.cuh):
// CSR grouped by source with neighbours ascending -- exactly the reference's edge-id
// numbering -- plus the twin index rev[e] (edge j->i of edge i->j), so a sweep gathers
// the reverse message in O(1) instead of searching.
//
//   1. validate + degree histogram            (one pass over the pairs, atomics)
//   2. row_ptr = exclusive scan(degree)       (CUB DeviceScan)
//   3. keys (row << cb | col) of both directions of every pair, one stable radix sort
//      (CUB DeviceRadixSort, payload 2p+dir): rows ascending, neighbours ascending
//   4. pos[payload] = e, rev[e] = pos[payload ^ 1], duplicate check (equal keys)
//   6. tiles: boundary where the edge bucket changes or every kTileRows rows
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <stdio.h>
#include <stdlib.h>

#include "gabp_internal.cuh"

namespace gabp {
namespace {

enum BuildErr : int { kErrNone = 0, kErrPairRange = 1, kErrZeroValue = 2, kErrDup = 3,
                      kErrZeroDiag = 4 };

__global__ void count_kernel(int64_t n, int64_t np, const int64_t *pi, const int64_t *pj,
                             uint32_t *deg, int *err,
                             unsigned long long *err_at) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < np;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = pi[p], j = pj[p];
        if (!(0 <= i && i < j && j < n)) {
            atomicCAS(err, 0, (int)kErrPairRange);
            atomicMin(err_at, (unsigned long long)p);
            continue;
        }
        atomicAdd(&deg[i], 1u);
        atomicAdd(&deg[j], 1u);
    }
}

// Both directions of every pair as one sort key (row << cb) | col, payload 2p / 2p + 1 (the
// pair and the direction).  One stable radix sort of the keys gives the CSR edge order --
// rows ascending, neighbours ascending (graph.py:84-91) -- with no per-row sort.
__global__ void key_kernel(int64_t np, const int64_t *pi, const int64_t *pj, int cb,
                           unsigned long long *key, uint32_t *pl) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < np;
         p += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long i = (unsigned long long)pi[p], j = (unsigned long long)pj[p];
        key[2 * p] = (i << cb) | j;
        key[2 * p + 1] = (j << cb) | i;
        pl[2 * p] = (uint32_t)(2 * p);
        pl[2 * p + 1] = (uint32_t)(2 * p + 1);
    }
}

// scol and the payload position of every sorted edge; a key equal to its predecessor is a
// duplicate pair (reported by its pair index)
__global__ void pos_key_kernel(int64_t E, const unsigned long long *key, const uint32_t *spl,
                               int cb, uint32_t *scol, uint32_t *pos, int *err,
                               unsigned long long *err_at) {
    const unsigned long long mask = (1ull << cb) - 1ull;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E;
         e += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long k = key[e];
        const uint32_t pl = spl[e];
        scol[e] = (uint32_t)(k & mask);
        pos[pl] = (uint32_t)e;
        if (e > 0 && k == key[e - 1]) {
            atomicCAS(err, 0, (int)kErrDup);
            atomicMin(err_at, (unsigned long long)(pl >> 1));
        }
    }
}

// (the explicit-zero check of the pair values lives here: the values may still be in
// flight from the host while the structural passes run)
__global__ void edge_kernel(int64_t E, const uint32_t *scol, const uint32_t *spl,
                            const uint32_t *pos, const double *pv, EdgeRec *er, int *err,
                            unsigned long long *err_at) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E;
         e += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t pl = spl[e];
        EdgeRec r;
        r.rev = pos[pl ^ 1u];
        r.col = scol[e];
        r.coeff = pv[pl >> 1];
        er[e] = r;
        if (r.coeff == 0.0 && !(pl & 1u)) {
            atomicCAS(err, 0, (int)kErrZeroValue);
            atomicMin(err_at, (unsigned long long)(pl >> 1));
        }
    }
}

__global__ void twin_span_kernel(int64_t E, const EdgeRec *er, double *sum) {
    double acc = 0.0;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = er[e].rev;
        acc += (double)(r > e ? r - e : e - r);
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(sum, acc);  // heuristic only: order irrelevant
}

// Tiles cover the swept rows [row_lo, row_lo + m): flag[k] for row row_lo + k.
__global__ void tile_flag_kernel(int64_t row_lo, int64_t m, const uint32_t *row_ptr,
                                 uint32_t *flag) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = row_lo + k;
        uint32_t f = (k % kTileRows) == 0;
        if (!f) f = (row_ptr[r] / kBucket) != (row_ptr[r - 1] / kBucket);
        flag[k] = f;
    }
}

__global__ void tile_scatter_kernel(int64_t row_lo, int64_t m, const uint32_t *flag,
                                    const uint32_t *idx, uint32_t *tile_start, int64_t ntiles) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m;
         k += (int64_t)gridDim.x * blockDim.x) {
        if (flag[k]) tile_start[idx[k]] = (uint32_t)(row_lo + k);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) tile_start[ntiles] = (uint32_t)(row_lo + m);
}

__global__ void tile_info_kernel(int64_t ntiles, const uint32_t *tile_start,
                                 const uint32_t *row_ptr, uint4 *info) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ntiles;
         t += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t r0 = tile_start[t], r1 = tile_start[t + 1];
        info[t] = make_uint4(r0, r1, row_ptr[r0], row_ptr[r1]);
    }
}

__global__ void prior_kernel(int64_t n, const double *diag, const double *rhs,
                             double *prior_num, NodeRec *nd, int *err,
                             unsigned long long *err_at) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double d = diag[i];
        if (d == 0.0) {
            atomicCAS(err, 0, (int)kErrZeroDiag);
            atomicMin(err_at, (unsigned long long)i);
        }
        const double pm = rhs[i] / d;  // prior mean (graph.py:74)
        prior_num[i] = d * pm;         // prior_prec * prior_mean (solver.py:147)
        NodeRec r;
        r.diag = d;
        r.pnum = d * pm;
        nd[i] = r;
    }
}

__global__ void sumsq_kernel(int64_t n, const double *v, double *part) {
    // fixed-order partials: block b sums [b*4096, (b+1)*4096) sequentially per thread slice
    __shared__ double red[256];
    const int64_t lo = (int64_t)blockIdx.x * 4096;
    double acc = 0.0;
    for (int64_t i = lo + threadIdx.x; i < lo + 4096 && i < n; i += 256) acc += v[i] * v[i];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

inline unsigned grid_for(int64_t work, int threads = 256) {
    int64_t b = (work + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > 148 * 32) b = 148 * 32;
    return (unsigned)b;
}

struct Scratch {
    void *p = nullptr;
    ~Scratch() { if (p) cudaFreeAsync(p, 0); }
};


// rows of more than 32 / 48 / 16 edges (the slot count of rowquad_kernel, rowpar.cu)
__global__ void deg_class_kernel(int64_t n, const uint32_t *deg, unsigned long long *cnt) {
    unsigned long long c16 = 0, c32 = 0, c48 = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t d = deg[i];
        c16 += d > 16u;
        c32 += d > 32u;
        c48 += d > 48u;
    }
    for (int o = 16; o > 0; o >>= 1) {
        c16 += __shfl_xor_sync(~0u, c16, o);
        c32 += __shfl_xor_sync(~0u, c32, o);
        c48 += __shfl_xor_sync(~0u, c48, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (c16) atomicAdd(cnt + 2, c16);
        if (c32) atomicAdd(cnt, c32);
        if (c48) atomicAdd(cnt + 1, c48);
    }
}

// ---- binned message order (build_bins) -----------------------------------------------------
__global__ void bin_key_kernel(int64_t E, const EdgeRec *er, uint32_t rows_per_bin,
                               uint32_t *key, uint32_t *val) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E;
         e += (int64_t)gridDim.x * blockDim.x) {
        key[e] = er[e].col / rows_per_bin;
        val[e] = (uint32_t)e;
    }
}
__global__ void bin_pos_kernel(int64_t E, const uint32_t *sorted, uint32_t *pos) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < E;
         p += (int64_t)gridDim.x * blockDim.x)
        pos[sorted[p]] = (uint32_t)p;
}
__global__ void bin_rec_kernel(int64_t E, const EdgeRec *er, const uint32_t *pos, uint2 *gidx,
                               double *gcoef) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E;
         e += (int64_t)gridDim.x * blockDim.x) {
        const EdgeRec r = er[e];
        gidx[e] = make_uint2(pos[r.rev], r.col);
        gcoef[e] = r.coeff;
    }
}

#define BCHECK(call)                                                                   \
    do {                                                                               \
        cudaError_t _e = (call);                                                       \
        if (_e != cudaSuccess) {                                                       \
            snprintf(err, errlen, "%s: %s", #call, cudaGetErrorString(_e));            \
            return _e == cudaErrorMemoryAllocation ? GABP_ENOMEM : GABP_ECUDA;         \
        }                                                                              \
    } while (0)

}  // namespace

void free_graph(DeviceGraph &g, cudaStream_t st) {
    // stream-ordered: the blocks go back to the device pool (retained, see new_graph)
    if (g.row_ptr) cudaFreeAsync(g.row_ptr, st);
    if (g.tile_start) cudaFreeAsync(g.tile_start, st);
    if (g.tile_info) cudaFreeAsync(g.tile_info, st);
    if (g.er) cudaFreeAsync(g.er, st);
    if (g.nd) cudaFreeAsync(g.nd, st);
    if (g.diag) cudaFreeAsync(g.diag, st);
    if (g.prior_num) cudaFreeAsync(g.prior_num, st);
    if (g.rhs) cudaFreeAsync(g.rhs, st);
    if (g.slice_info) cudaFreeAsync(g.slice_info, st);
    if (g.gorder) cudaFreeAsync(g.gorder, st);
    if (g.dia_coef) cudaFreeAsync(g.dia_coef, st);
    if (g.dia_mask) cudaFreeAsync(g.dia_mask, st);
    g.dia_coef = nullptr;
    g.dia_mask = nullptr;
    g.dia_D = 0;
    if (g.pos) cudaFreeAsync(g.pos, st);
    if (g.srow) cudaFreeAsync(g.srow, st);
    if (g.sdeg) cudaFreeAsync(g.sdeg, st);
    if (g.snd) cudaFreeAsync(g.snd, st);
    if (g.srhs) cudaFreeAsync(g.srhs, st);
    if (g.scol) cudaFreeAsync(g.scol, st);
    if (g.scoef) cudaFreeAsync(g.scoef, st);
    if (g.stwin) cudaFreeAsync(g.stwin, st);
    if (g.gidx) cudaFreeAsync(g.gidx, st);
    if (g.gcoef) cudaFreeAsync(g.gcoef, st);
    if (g.gout) cudaFreeAsync(g.gout, st);
    g = DeviceGraph{};
}

int compute_priors(DeviceGraph &g, cudaStream_t st, char *err, size_t errlen) {
    int *d_err = nullptr;
    unsigned long long *d_at = nullptr;
    BCHECK(cudaMallocAsync(&d_err, sizeof(int) + sizeof(unsigned long long) * 2, st));
    d_at = reinterpret_cast<unsigned long long *>(d_err + 2);
    BCHECK(cudaMemsetAsync(d_err, 0, sizeof(int) * 2, st));
    BCHECK(cudaMemsetAsync(d_at, 0xff, sizeof(unsigned long long), st));
    prior_kernel<<<grid_for(g.n), 256, 0, st>>>(g.n, g.diag, g.rhs, g.prior_num, g.nd, d_err,
                                                d_at);
    BCHECK(cudaGetLastError());
    BCHECK(refresh_slice_nodes(g, st));
    const int64_t nparts = (g.n + 4095) / 4096;
    double *part = nullptr;
    BCHECK(cudaMallocAsync(&part, sizeof(double) * nparts, st));
    sumsq_kernel<<<(unsigned)nparts, 256, 0, st>>>(g.n, g.rhs, part);
    BCHECK(cudaGetLastError());
    int h_err = 0;
    unsigned long long h_at = 0;
    double *h_part = (double *)malloc(sizeof(double) * nparts);
    BCHECK(cudaMemcpyAsync(&h_err, d_err, sizeof(int), cudaMemcpyDeviceToHost, st));
    BCHECK(cudaMemcpyAsync(&h_at, d_at, sizeof(h_at), cudaMemcpyDeviceToHost, st));
    BCHECK(cudaMemcpyAsync(h_part, part, sizeof(double) * nparts, cudaMemcpyDeviceToHost, st));
    BCHECK(cudaStreamSynchronize(st));
    cudaFreeAsync(part, st);
    cudaFreeAsync(d_err, st);
    double ss = 0.0;
    for (int64_t c = 0; c < nparts; ++c) ss += h_part[c];
    free(h_part);
    g.rhs_norm = sqrt(ss);
    if (h_err == kErrZeroDiag) {
        snprintf(err, errlen, "zero diagonal entry at row %llu: node priors need b_i / A_ii", h_at);
        return GABP_EZERODIAG;
    }
    return GABP_OK;
}

int build_graph_device(DeviceGraph &g, int64_t n, int64_t npairs, const double *d_diag,
                       const double *d_rhs, const int64_t *d_pi, const int64_t *d_pj,
                       const double *d_pv, int64_t row_lo, int64_t row_hi, cudaStream_t st,
                       char *err, size_t errlen, cudaEvent_t idx_ready, cudaEvent_t val_ready) {
    if (idx_ready) BCHECK(cudaStreamWaitEvent(st, idx_ready, 0));
    if (row_lo < 0 || row_hi > n || row_lo >= row_hi) {
        row_lo = 0;
        row_hi = n;
    }
    g.row_lo = row_lo;
    g.row_hi = row_hi;
    const int64_t m_rows = row_hi - row_lo;
    if (n < 1) {
        snprintf(err, errlen, "diag must be a non-empty vector");
        return GABP_EINVAL;
    }
    if (npairs < 0 || 2 * npairs >= (int64_t)0xffffffffll || n >= (int64_t)0xffffffffll) {
        snprintf(err, errlen, "graph too large for 32-bit edge ids (n=%lld, pairs=%lld)",
                 (long long)n, (long long)npairs);
        return GABP_EINVAL;
    }
    const int64_t E = 2 * npairs;
    g.n = n;
    g.E = E;
    g.npairs = npairs;
    cudaEvent_t t0, t1;
    cudaEventCreate(&t0);
    cudaEventCreate(&t1);
    cudaEventRecord(t0, st);

    BCHECK(cudaMallocAsync(&g.diag, sizeof(double) * (n + kNodePad), st));
    BCHECK(cudaMallocAsync(&g.rhs, sizeof(double) * (n + kNodePad), st));
    BCHECK(cudaMallocAsync(&g.prior_num, sizeof(double) * (n + kNodePad), st));
    BCHECK(cudaMemsetAsync(g.diag + n, 0, sizeof(double) * kNodePad, st));
    BCHECK(cudaMemsetAsync(g.rhs + n, 0, sizeof(double) * kNodePad, st));
    BCHECK(cudaMemsetAsync(g.prior_num + n, 0, sizeof(double) * kNodePad, st));
    BCHECK(cudaMallocAsync(&g.row_ptr, sizeof(uint32_t) * (n + 1 + kNodePad), st));
    BCHECK(cudaMemsetAsync(g.row_ptr + n + 1, 0, sizeof(uint32_t) * kNodePad, st));
    BCHECK(cudaMallocAsync(&g.er, sizeof(EdgeRec) * (E > 0 ? E : 1), st));
    BCHECK(cudaMallocAsync(&g.nd, sizeof(NodeRec) * (n + kNodePad), st));
    BCHECK(cudaMemsetAsync(g.nd + n, 0, sizeof(NodeRec) * kNodePad, st));

    int *d_err = nullptr;
    BCHECK(cudaMallocAsync(&d_err, 16, st));
    unsigned long long *d_at = reinterpret_cast<unsigned long long *>(d_err + 2);
    BCHECK(cudaMemsetAsync(d_err, 0, 8, st));
    BCHECK(cudaMemsetAsync(d_at, 0xff, 8, st));

    // 1. degrees
    uint32_t *deg = nullptr;
    BCHECK(cudaMallocAsync(&deg, sizeof(uint32_t) * (n + 1), st));
    BCHECK(cudaMemsetAsync(deg, 0, sizeof(uint32_t) * (n + 1), st));
    if (npairs > 0) {
        count_kernel<<<grid_for(npairs), 256, 0, st>>>(n, npairs, d_pi, d_pj, deg, d_err, d_at);
        BCHECK(cudaGetLastError());
    }
    // 2. row_ptr
    size_t tmp_bytes = 0;
    BCHECK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, deg, g.row_ptr, n + 1, st));
    void *tmp = nullptr;
    size_t tmp_cap = tmp_bytes;
    BCHECK(cudaMallocAsync(&tmp, tmp_cap, st));
    BCHECK(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, deg, g.row_ptr, n + 1, st));
    // max degree
    {
        uint32_t *d_max = nullptr;
        BCHECK(cudaMallocAsync(&d_max, sizeof(uint32_t), st));
        unsigned long long *d_cls = nullptr, h_cls[3] = {0ull, 0ull, 0ull};
        BCHECK(cudaMallocAsync(&d_cls, sizeof(h_cls), st));
        BCHECK(cudaMemsetAsync(d_cls, 0, sizeof(h_cls), st));
        deg_class_kernel<<<148 * 4, 256, 0, st>>>(n, deg, d_cls);
        BCHECK(cudaGetLastError());
        size_t b2 = 0;
        BCHECK(cub::DeviceReduce::Max(nullptr, b2, deg, d_max, n, st));
        if (b2 > tmp_cap) {
            cudaFreeAsync(tmp, st);
            tmp_cap = b2;
            BCHECK(cudaMallocAsync(&tmp, tmp_cap, st));
        }
        BCHECK(cub::DeviceReduce::Max(tmp, b2, deg, d_max, n, st));
        uint32_t h_max = 0;
        BCHECK(cudaMemcpyAsync(&h_max, d_max, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        BCHECK(cudaMemcpyAsync(h_cls, d_cls, sizeof(h_cls), cudaMemcpyDeviceToHost, st));
        int h_err0 = 0;
        BCHECK(cudaMemcpyAsync(&h_err0, d_err, sizeof(int), cudaMemcpyDeviceToHost, st));
        unsigned long long h_at0 = 0;
        BCHECK(cudaMemcpyAsync(&h_at0, d_at, 8, cudaMemcpyDeviceToHost, st));
        BCHECK(cudaStreamSynchronize(st));
        cudaFreeAsync(d_max, st);
        cudaFreeAsync(d_cls, st);
        g.max_degree = h_max;
        g.rows_gt32 = (int64_t)h_cls[0];
        g.rows_gt48 = (int64_t)h_cls[1];
        g.rows_gt16 = (int64_t)h_cls[2];
        if (h_err0 != kErrNone) {
            cudaFreeAsync(tmp, st);
            cudaFreeAsync(deg, st);
            cudaFreeAsync(d_err, st);
            cudaStreamSynchronize(st);
            if (h_err0 == kErrPairRange)
                snprintf(err, errlen, "bad off-diagonal key at pair %llu for n=%lld", h_at0,
                         (long long)n);
            else
                snprintf(err, errlen, "explicit zero stored at pair %llu", h_at0);
            return GABP_EINVAL;
        }
    }
    if (E > 0) {
        // 3. CSR order: one stable radix sort of (row, col) keys of both directions
        int cb = 1;
        while (cb < 32 && ((unsigned long long)(n - 1) >> cb) != 0ull) ++cb;
        unsigned long long *kin = nullptr, *kout = nullptr;
        uint32_t *plin = nullptr, *spl = nullptr;
        BCHECK(cudaMallocAsync(&kin, sizeof(unsigned long long) * E, st));
        BCHECK(cudaMallocAsync(&kout, sizeof(unsigned long long) * E, st));
        BCHECK(cudaMallocAsync(&plin, sizeof(uint32_t) * E, st));
        BCHECK(cudaMallocAsync(&spl, sizeof(uint32_t) * E, st));
        key_kernel<<<grid_for(npairs), 256, 0, st>>>(npairs, d_pi, d_pj, cb, kin, plin);
        BCHECK(cudaGetLastError());
        size_t sb = 0;
        BCHECK(cub::DeviceRadixSort::SortPairs(nullptr, sb, kin, kout, plin, spl, (int64_t)E, 0,
                                               2 * cb, st));
        if (sb > tmp_cap) {
            cudaFreeAsync(tmp, st);
            tmp_cap = sb;
            BCHECK(cudaMallocAsync(&tmp, tmp_cap, st));
        }
        BCHECK(cub::DeviceRadixSort::SortPairs(tmp, sb, kin, kout, plin, spl, (int64_t)E, 0,
                                               2 * cb, st));
        // 4. twin index: pos[payload] = edge id; scol from the keys (buffers reused)
        uint32_t *scol = plin;
        uint32_t *pos = reinterpret_cast<uint32_t *>(kin);
        pos_key_kernel<<<grid_for(E), 256, 0, st>>>(E, kout, spl, cb, scol, pos, d_err, d_at);
        BCHECK(cudaGetLastError());
        if (val_ready) BCHECK(cudaStreamWaitEvent(st, val_ready, 0));
        edge_kernel<<<grid_for(E), 256, 0, st>>>(E, scol, spl, pos, d_pv, g.er, d_err, d_at);
        BCHECK(cudaGetLastError());
        cudaFreeAsync(kin, st);
        cudaFreeAsync(kout, st);
        cudaFreeAsync(plin, st);
        cudaFreeAsync(spl, st);
        g.twin_span = -1.0;  // computed only if the tile layout ends up serving the solve
    }
    // 6. tiles
    {
        uint32_t *flag = deg, *idx = nullptr;  // deg no longer needed
        BCHECK(cudaMallocAsync(&idx, sizeof(uint32_t) * (n + 1), st));
        tile_flag_kernel<<<grid_for(m_rows), 256, 0, st>>>(row_lo, m_rows, g.row_ptr, flag);
        BCHECK(cudaGetLastError());
        BCHECK(cudaMemsetAsync(flag + m_rows, 0, sizeof(uint32_t), st));
        size_t b3 = 0;
        BCHECK(cub::DeviceScan::ExclusiveSum(nullptr, b3, flag, idx, m_rows + 1, st));
        if (b3 > tmp_cap) {
            cudaFreeAsync(tmp, st);
            tmp_cap = b3;
            BCHECK(cudaMallocAsync(&tmp, tmp_cap, st));
        }
        BCHECK(cub::DeviceScan::ExclusiveSum(tmp, b3, flag, idx, m_rows + 1, st));
        uint32_t h_nt = 0;
        BCHECK(cudaMemcpyAsync(&h_nt, idx + m_rows, sizeof(uint32_t), cudaMemcpyDeviceToHost,
                               st));
        BCHECK(cudaStreamSynchronize(st));
        g.ntiles = h_nt;
        BCHECK(cudaMallocAsync(&g.tile_start, sizeof(uint32_t) * (h_nt + 1), st));
        tile_scatter_kernel<<<grid_for(m_rows), 256, 0, st>>>(row_lo, m_rows, flag, idx,
                                                              g.tile_start, g.ntiles);
        BCHECK(cudaGetLastError());
        BCHECK(cudaMallocAsync(&g.tile_info, sizeof(uint4) * (h_nt + 1), st));
        tile_info_kernel<<<grid_for(g.ntiles), 256, 0, st>>>(g.ntiles, g.tile_start, g.row_ptr,
                                                            g.tile_info);
        BCHECK(cudaGetLastError());
        cudaFreeAsync(idx, st);
    }
    if (val_ready) BCHECK(cudaStreamWaitEvent(st, val_ready, 0));  // (again if E > 0: harmless)
    BCHECK(cudaMemcpyAsync(g.diag, d_diag, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    BCHECK(cudaMemcpyAsync(g.rhs, d_rhs, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    cudaFreeAsync(tmp, st);
    cudaFreeAsync(deg, st);
    int h_err = 0;
    unsigned long long h_at = 0;
    BCHECK(cudaMemcpyAsync(&h_err, d_err, sizeof(int), cudaMemcpyDeviceToHost, st));
    BCHECK(cudaMemcpyAsync(&h_at, d_at, 8, cudaMemcpyDeviceToHost, st));
    cudaEventRecord(t1, st);
    BCHECK(cudaStreamSynchronize(st));
    cudaFreeAsync(d_err, st);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, t0, t1);
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    g.build_ms = ms;
    if (h_err == kErrDup) {
        snprintf(err, errlen, "duplicate off-diagonal pair (pair index %llu)", h_at);
        return GABP_EDUP;
    }
    if (h_err == kErrZeroValue) {
        snprintf(err, errlen, "explicit zero stored at pair %llu", h_at);
        return GABP_EINVAL;
    }
    if (g.max_degree <= kSliceMaxDegree) {
        const int rc = build_slices(g, st, err, errlen);
        if (rc == GABP_ENOMEM || rc == GABP_ECUDA) return rc;
        err[0] = 0;  // too many slots for 32-bit ids: the row tiles remain
    }
    if (g.nslices == 0 && E > 0) {
        // no slice layout: the tile kernels choose their gather by the twin locality
        double *d_span = nullptr;
        BCHECK(cudaMallocAsync(&d_span, sizeof(double), st));
        BCHECK(cudaMemsetAsync(d_span, 0, sizeof(double), st));
        twin_span_kernel<<<grid_for(E), 256, 0, st>>>(E, g.er, d_span);
        BCHECK(cudaGetLastError());
        double h_span = 0.0;
        BCHECK(cudaMemcpyAsync(&h_span, d_span, sizeof(double), cudaMemcpyDeviceToHost, st));
        BCHECK(cudaStreamSynchronize(st));
        cudaFreeAsync(d_span, st);
        g.twin_span = h_span / (double)E;
    }
    {
        const int rc = build_dia(g, st, err, errlen);
        if (rc != GABP_OK) return rc;
    }
    return compute_priors(g, st, err, errlen);
}

// Binned message order of the four-rows-per-warp parallel kernel (rowpar.cu: rowquad_kernel).
// In CSR order a row's twin messages are spread over the whole message array: every 16-byte
// gather costs a 128-byte line of DRAM.  Here the message of edge i -> j lives at
// pos(i -> j) = rank of the edge in the order (bin of j, i, j), bin = j / rows_per_bin: the
// rows of one bin gather all their incoming messages from one window of E / bins messages
// (a few MB: every line comes from DRAM once and serves its 8 gathers from L2), and rows
// swept in ascending order write each bin's messages as an ascending run (lines fill in L2
// within a few rows).  gout[e] = pos(e), gidx[e] = {pos(rev(e)), j}, gcoef[e] = A_ij.
int build_bins(DeviceGraph &g, cudaStream_t st, char *err, size_t errlen) {
    if (g.bins != 0) return GABP_OK;
    g.bins = -1;
    const int64_t E = g.E;
    const char *wenv = getenv("GABP_BIN_WINDOW_MB");
    const double window = (wenv ? atof(wenv) : 48.0) * 1048576.0;
    // messages that fit L2 anyway, partial graphs, ids past 31 bits: CSR order
    if (E <= 0 || E >= (1ll << 31) || g.row_lo != 0 || g.row_hi != g.n ||
        16.0 * (double)E < (getenv("GABP_BIN_MIN") ? atof(getenv("GABP_BIN_MIN")) : 6.0) * window || window <= 0.0)
        return GABP_OK;
    int64_t nb = (int64_t)(16.0 * (double)E / window + 0.999);
    if (nb > 4096) nb = 4096;
    if (nb < 2) return GABP_OK;
    const uint32_t rpb = (uint32_t)((g.n + nb - 1) / nb);
    int bits = 1;
    while ((1ll << bits) < nb) ++bits;
    uint32_t *key = nullptr, *val = nullptr;
    void *tmp = nullptr;
    auto body = [&]() -> cudaError_t {
        cudaError_t e;
        size_t tb = 0;
        if ((e = cudaMallocAsync(&key, sizeof(uint32_t) * 2 * E, st)) != cudaSuccess) return e;
        if ((e = cudaMallocAsync(&val, sizeof(uint32_t) * 2 * E, st)) != cudaSuccess) return e;
        bin_key_kernel<<<grid_for(E), 256, 0, st>>>(E, g.er, rpb, key, val);
        if ((e = cub::DeviceRadixSort::SortPairs(nullptr, tb, key, key + E, val, val + E, E, 0,
                                                 bits, st)) != cudaSuccess)
            return e;
        if ((e = cudaMallocAsync(&tmp, tb, st)) != cudaSuccess) return e;
        if ((e = cub::DeviceRadixSort::SortPairs(tmp, tb, key, key + E, val, val + E, E, 0, bits,
                                                 st)) != cudaSuccess)
            return e;
        if ((e = cudaMallocAsync(&g.gout, sizeof(uint32_t) * E, st)) != cudaSuccess) return e;
        if ((e = cudaMallocAsync(&g.gidx, sizeof(uint2) * E, st)) != cudaSuccess) return e;
        if ((e = cudaMallocAsync(&g.gcoef, sizeof(double) * E, st)) != cudaSuccess) return e;
        bin_pos_kernel<<<grid_for(E), 256, 0, st>>>(E, val + E, g.gout);
        bin_rec_kernel<<<grid_for(E), 256, 0, st>>>(E, g.er, g.gout, g.gidx, g.gcoef);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        return cudaStreamSynchronize(st);
    };
    const cudaError_t e = body();
    if (tmp) cudaFreeAsync(tmp, st);
    if (key) cudaFreeAsync(key, st);
    if (val) cudaFreeAsync(val, st);
    if (e != cudaSuccess) {
        // (out of memory: the solve runs in CSR order; anything else is reported)
        if (g.gout) cudaFreeAsync(g.gout, st);
        if (g.gidx) cudaFreeAsync(g.gidx, st);
        if (g.gcoef) cudaFreeAsync(g.gcoef, st);
        g.gout = nullptr;
        g.gidx = nullptr;
        g.gcoef = nullptr;
        cudaGetLastError();
        if (e == cudaErrorMemoryAllocation) return GABP_OK;
        snprintf(err, errlen, "build_bins: %s", cudaGetErrorString(e));
        return GABP_ECUDA;
    }
    g.bins = (int)nb;
    return GABP_OK;
}

}  // namespace gabp
