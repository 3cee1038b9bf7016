// rowpar.cu -- the parallel schedule (solver.py:146-173, the reference's default) as a
// warp-per-row sweep over the CSR edge order.
//
// The exclusion sum of edge i -> j is P_i\j = A_ii + sum_{k != j} P_ki, accumulated in
// ascending k (np.add.at over excl_pos, solver.py:149-150).  Bitwise parity forbids the
// subtraction trick of the broadcast schedule, so a row of degree d costs d (d - 1) adds.
// A lane per row (slice.cu: slice_kernel_par) must keep the row's incoming terms in
// registers and re-streams them once per block of outgoing edges; here the row's
// incoming terms sit once in a per-warp shared-memory strip and the d exclusion sums run
// in parallel, lane j walking the strip with one broadcast load per term and skipping
// k == j by predicate.  Per row:
//
//   load     lanes over the row's edge slots (coalesced): EdgeRec {rev, col, A_ij}, own
//            message m_ij of S_{s-1} (change statistic), twin message m_ji = msg[rev]
//            (one gathered sector), x_j^{(s-2)} (residual, L2-resident)
//   strip    T[q] = {P_qi, P_qi * mu_qi} (product rounded first, solver.py:148), padded
//            to a multiple of 8 with {-0, -0} (x + (-0) == x for every x: the exact
//            identity, so the walk has no tail)
//   walk     lane j: p = A_ii, n = A_ii mu_ii; p += T[k].P, n += T[k].N for k != j
//            (rows of 33..64 edges: two sums per lane over one walk)
//   edge     P_ij = -A_ij^2 / P_i\j, mu_ij = N_i\j / A_ij (solver.py:155-156), coalesced
//            store, max |dP|, |dmu|, blow-up test, first singular edge
//   node     lane d-1 holds the full sum (its exclusion sum + its own term, the same
//            additions in the same order): marginal x_i^{(s-1)} = N_i / P_i; residual row
//            of x^{(s-2)} from a warp reduction (the residual is compared to 1e-9, not bits)
//
// Launch protocol, statistics and decision: exactly those of the CSR tile kernel
// (sweep.cu, sweep_epilogue with LAG 0), so the solve loop and controller are unchanged.
#include <float.h>
#include <math.h>
#include <stdlib.h>

#include "sweep_common.cuh"

namespace gabp {
namespace {

constexpr int kRThreads = 256;
constexpr int kRWarps = kRThreads / 32;
constexpr int kRStrip = kRowParMaxDegree + 8;

struct RowSmem {
    double2 T[kRWarps][kRStrip];
    TailSmem<kRWarps> tail;
    int64_t sweep;
    int skip;
};

struct RowCtx {
    const double2 *min_;  // S_{s-1}
    const double *xprev;  // x^{(s-2)} (residual)
    double2 *mout;        // S_s
    double *xcur, *pcur, *xh;
    bool resid;
    uint64_t pol;         // L2 evict-first
    // binned message order (build_bins): per edge {position of the twin message, column} and
    // the position of the edge's own message; null: CSR order
    const uint2 *gidx = nullptr;
    const uint32_t *gout = nullptr;
};

// Streams (edge records, own old messages, twin gathers, new messages) are touched once per
// sweep: L2 evict-first, so the L2-resident x^{(s-2)} gathers of the residual stay cached.
__device__ __forceinline__ uint64_t pol_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ int4 ld_ef_i4(const void *ptr, uint64_t pol) {
    int4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(ptr), "l"(pol));
    return v;
}
__device__ __forceinline__ double2 ld_ef_d2(const double2 *ptr, uint64_t pol) {
    double2 v;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(v.x), "=d"(v.y)
                 : "l"(ptr), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_ef_d2(double2 *ptr, double2 v, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;"
                 ::"l"(ptr), "d"(v.x), "d"(v.y), "l"(pol)
                 : "memory");
}

// Binned message order: a gathered line serves 8 gathers, a written line fills from 8 rows --
// the message traffic keeps the default L2 priority (only the once-read records stream).
__device__ __forceinline__ double2 ld_na_d2(const double2 *ptr) {
    double2 v;
    asm volatile("ld.global.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
                 : "=d"(v.x), "=d"(v.y)
                 : "l"(ptr));
    return v;
}
__device__ __forceinline__ void st_na_d2(double2 *ptr, double2 v) {
    asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1, %2};" ::"l"(ptr), "d"(v.x),
                 "d"(v.y)
                 : "memory");
}

__device__ __forceinline__ EdgeRec er_of(int4 v) {
    EdgeRec r;
    r.rev = (uint32_t)v.x;
    r.col = (uint32_t)v.y;
    r.coeff = __hiloint2double(v.w, v.z);
    return r;
}
__device__ __forceinline__ EdgeRec ld_er_cs(const EdgeRec *p) {
    return er_of(__ldcs(reinterpret_cast<const int4 *>(p)));
}
__device__ __forceinline__ EdgeRec ld_er(const EdgeRec *p) {
    return er_of(__ldg(reinterpret_cast<const int4 *>(p)));
}

template <int MODE>
__device__ __forceinline__ void row_node(const SweepArgs &a, const RowCtx &x, uint32_t i,
                                         double sp, double sn, Stats &st) {
    bool ok;
    double xi = ddiv_fast(sn, sp, ok);  // infer_marginals of the state read (solver.py:286)
    if (!ok) xi = div_slow(sn, sp);
    if (MODE == kModeSolve) {
        x.xcur[i] = xi;
        x.pcur[i] = sp;
        if (!(fabs(xi) <= DBL_MAX)) st.means_bad = 1u;
        if (x.xh) x.xh[i] = xi;
    }
}

template <bool BIN = false>
__device__ __forceinline__ void edge_out(const RowCtx &x, uint32_t e, uint32_t pos, double c,
                                         double pe, double num, double2 old, Stats &st) {
    bool okp, okm;
    double np_ = ddiv_fast(-c * c, pe, okp);
    double nm = ddiv_fast(num, c, okm);
    if (!okp) np_ = div_slow(-c * c, pe);
    if (!okm) nm = div_slow(num, c);
    if (BIN)
        st_na_d2(x.mout + pos, make_double2(np_, nm));
    else
        st_ef_d2(x.mout + pos, make_double2(np_, nm), x.pol);
    st.edge(e, pe, np_, nm, old);
}

// One row of the warp's stream, first 64 edge slots in registers (lane l: slots l, l + 32).
struct RowPre {
    uint32_t i = 0, e0 = 0, d = 0;
    double2 nd = make_double2(0.0, 0.0);  // {A_ii, A_ii mu_ii}
    int4 er[2];                           // EdgeRec {rev, col, A_ij} as loaded
};

__device__ __forceinline__ void pre_load(const SweepArgs &a, RowPre &r, uint32_t i, uint32_t e0,
                                         uint32_t e1, int lane, uint64_t pol) {
    r.i = i;
    r.e0 = e0;
    r.d = e1 - e0;
    r.nd = __ldg(reinterpret_cast<const double2 *>(a.nd + i));
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const uint32_t q = lane + 32 * u;
        r.er[u] = q < r.d ? ld_ef_i4(a.er + e0 + q, pol) : make_int4(0, 0, 0, 0);
    }
}

// The row being gathered: its twin messages, x_j, own old messages in flight.
struct RowGat {
    uint32_t i = 0, e0 = 0, d = 0;
    double2 nd = make_double2(0.0, 0.0);
    double c[2];     // A_ij
    double2 o[2];    // own message of S_{s-1}
    double2 in[2];   // twin message m_ji of S_{s-1}
    double xg[2];    // x_j^{(s-2)}
};

__device__ __forceinline__ void gat_issue(const SweepArgs &a, const RowCtx &x, const RowPre &p,
                                          RowGat &g, int lane) {
    g.i = p.i;
    g.e0 = p.e0;
    g.d = p.d;
    g.nd = p.nd;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const uint32_t q = lane + 32 * u;
        const EdgeRec r = er_of(p.er[u]);
        g.c[u] = r.coeff;
        g.o[u] = make_double2(0.0, 0.0);
        g.in[u] = make_double2(0.0, 0.0);
        g.xg[u] = 0.0;
        if (q < p.d && p.d <= 64) {
            g.o[u] = ld_ef_d2(x.min_ + p.e0 + q, x.pol);
            g.in[u] = ld_ef_d2(x.min_ + r.rev, x.pol);
            if (x.resid) g.xg[u] = __ldcg(x.xprev + r.col);
        }
    }
}

// Walk of a row of at most 32 R edges whose strip is filled.
template <int R, int MODE>
__device__ __forceinline__ void row_walk(const SweepArgs &a, const RowCtx &x, const double2 *T,
                                         const RowGat &g, int lane, Stats &st) {
    const uint32_t d = g.d, dpad = (d + 7u) & ~7u;
    double p[R], n[R];
#pragma unroll
    for (int u = 0; u < R; ++u) {
        p[u] = g.nd.x;
        n[u] = g.nd.y;
    }
    // lane j reads T[t + (t >= j)]: terms 0..j-1, then j+1..dpad (T[dpad] is a {-0, -0}
    // pad), so the skip is an address select off the dependent add chain (a predicated add
    // compiles to add + 2 selects on the chain)
    for (uint32_t t = 0; t < dpad; t += 8) {
        const double2 *b0 = T + t, *b1 = T + t + 1;
#pragma unroll
        for (int u = 0; u < R; ++u) {
            const int jt = lane + 32 * u - (int)t;  // lane's own slot relative to the block
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const double2 v = (jt > k ? b0 : b1)[k];
                p[u] = p[u] + v.x;
                n[u] = n[u] + v.y;
            }
        }
    }
#pragma unroll
    for (int u = 0; u < R; ++u) {
        const uint32_t j = lane + 32 * u;
        if (j < d) {
            edge_out(x, g.e0 + j, g.e0 + j, g.c[u], p[u], n[u], g.o[u], st);
            if (j == d - 1)  // full sums: the last exclusion sum plus the last term
                row_node<MODE>(a, x, g.i, p[u] + g.in[u].x, n[u] + g.in[u].x * g.in[u].y, st);
        }
    }
}

// Strip fill, walk and node work of a gathered row of at most 64 edges.
template <int MODE>
__device__ __forceinline__ void row_fast(const SweepArgs &a, const RowCtx &x, double2 *T,
                                         const RowGat &g, int lane, Stats &st) {
    const uint32_t d = g.d, dpad = (d + 7u) & ~7u;
    double yp = 0.0;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const uint32_t q = lane + 32 * u;
        if (q < d) {
            T[q] = make_double2(g.in[u].x, g.in[u].x * g.in[u].y);  // (prec * mean)
            if (x.resid) yp = yp + g.c[u] * g.xg[u];
        } else if (q <= dpad) {
            T[q] = make_double2(-0.0, -0.0);
        }
    }
    if (dpad == 64 && lane == 0) T[64] = make_double2(-0.0, -0.0);
    __syncwarp();
    if (d <= 32)
        row_walk<1, MODE>(a, x, T, g, lane, st);
    else
        row_walk<2, MODE>(a, x, T, g, lane, st);
    __syncwarp();  // the strip is rewritten by the next row
    if (d == 0 && lane == 0) row_node<MODE>(a, x, g.i, g.nd.x, g.nd.y, st);
    if (x.resid) {
        yp = warp_sum(yp);
        if (lane == 0) {
            const double y = g.nd.x * __ldg(x.xprev + g.i) + yp;
            const double res = y - __ldg(a.rhs + g.i);
            st.rsq += res * res;
        }
    }
}

// Rows of 65 .. kRowParMaxDegree edges: the strip is filled in rounds of 32 slots and
// walked in rounds of 32 exclusion sums; the edge's own operands are reloaded.
template <int MODE>
__device__ void row_long(const SweepArgs &a, const RowCtx &x, double2 *T, uint32_t i,
                         uint32_t e0, uint32_t d, NodeRec nd, int lane, Stats &st) {
    const uint32_t dpad = (d + 7u) & ~7u;
    double yp = 0.0;
    for (uint32_t q = lane; q < dpad; q += 32) {
        if (q < d) {
            EdgeRec r = ld_er(a.er + e0 + q);
            if (x.gidx) r.rev = __ldg(&x.gidx[e0 + q].x);
            const double2 in = __ldcg(x.min_ + r.rev);
            T[q] = make_double2(in.x, in.x * in.y);
            if (x.resid) yp = yp + r.coeff * __ldcg(x.xprev + r.col);
        } else {
            T[q] = make_double2(-0.0, -0.0);
        }
    }
    __syncwarp();
    for (uint32_t jb = 0; jb < d; jb += 32) {
        const uint32_t j = jb + lane;
        double p = nd.diag, n = nd.pnum;
        for (uint32_t t = 0; t < dpad; t += 8) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const double2 v = T[t + k];
                if (t + k != j) {
                    p = p + v.x;
                    n = n + v.y;
                }
            }
        }
        if (j < d) {
            const double2 own = T[j];
            const uint32_t pos = x.gout ? __ldg(x.gout + e0 + j) : e0 + j;
            const double c = __ldg(&a.er[e0 + j].coeff);
            if (x.gout)
                edge_out<true>(x, e0 + j, pos, c, p, n, ld_na_d2(x.min_ + pos), st);
            else
                edge_out<false>(x, e0 + j, pos, c, p, n, __ldcs(x.min_ + pos), st);
            if (j == d - 1) row_node<MODE>(a, x, i, p + own.x, n + own.y, st);
        }
    }
    __syncwarp();
    if (x.resid) {
        yp = warp_sum(yp);
        if (lane == 0) {
            const double y = nd.diag * __ldg(x.xprev + i) + yp;
            const double res = y - __ldg(a.rhs + i);
            st.rsq += res * res;
        }
    }
}

template <int MODE>
__global__ void __launch_bounds__(kRThreads, 2) rowpar_kernel(const SweepArgs a) {
    __shared__ RowSmem S;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    Ctrl *ctrl = a.ctrl;
    if (tid == 0) {
        if (MODE == kModeSolve) {
            volatile Ctrl *vc = ctrl;
            const int64_t s = vc->next_sweep;
            S.skip = vc->done || s > vc->max_iter + 2;
            S.sweep = s;
        } else {
            S.skip = 0;
            S.sweep = 1;
        }
    }
    __syncthreads();
    if (S.skip) return;
    const int64_t s = S.sweep;
    RowCtx x;
    x.resid = (MODE == kModeSolve) && s >= 3;
    x.min_ = a.msg[(s - 1) % 3];
    x.xprev = x.resid ? a.x[(s - 2) % 3] : nullptr;
    x.mout = a.msg[s % 3];
    x.xcur = (MODE == kModeSolve) ? a.x[(s - 1) % 3] : nullptr;
    x.pcur = (MODE == kModeSolve) ? a.p[(s - 1) % 3] : nullptr;
    x.xh = (MODE == kModeSolve && a.xhist && s >= 2 && s - 1 <= a.xhist_rows)
               ? a.xhist + (s - 2) * a.n : nullptr;
    x.pol = pol_evict_first();
    Stats st;
    st.lim = (MODE == kModeSolve) ? fmin(ctrl->blowup, DBL_MAX) : DBL_MAX;
    double2 *T = S.T[warp];

    // The swept rows (a rank's owned block, [first tile row, last tile row)) are cut into
    // one contiguous range per warp.  Software pipeline over the warp's rows: while row i
    // walks, the gathers of row i+1 and the edge records of row i+2 are in flight.
    const uint32_t r_lo = __ldg(&a.tile_info[0].x);
    const uint32_t r_hi = __ldg(&a.tile_info[a.ntiles - 1].y);
    const int64_t nw = (int64_t)gridDim.x * kRWarps, gw = (int64_t)blockIdx.x * kRWarps + warp;
    const uint32_t rb = r_lo + (uint32_t)(((int64_t)(r_hi - r_lo) * gw) / nw);
    const uint32_t re = r_lo + (uint32_t)(((int64_t)(r_hi - r_lo) * (gw + 1)) / nw);
    if (rb < re) {
        RowPre pb, pc;
        RowGat ga, gb;
        uint32_t ep = __ldg(a.row_ptr + rb);
        uint32_t e1 = __ldg(a.row_ptr + rb + 1);
        pre_load(a, pb, rb, ep, e1, lane, x.pol);
        gat_issue(a, x, pb, ga, lane);
        uint32_t rp2 = rb + 2 <= re ? __ldg(a.row_ptr + rb + 2) : 0u;
        if (rb + 1 < re) pre_load(a, pb, rb + 1, e1, rp2, lane, x.pol);
        uint32_t rp3 = rb + 3 <= re ? __ldg(a.row_ptr + rb + 3) : 0u;
        for (uint32_t i = rb; i < re; ++i) {
            if (i + 1 < re) gat_issue(a, x, pb, gb, lane);  // gathers of row i+1
            if (i + 2 < re) {                               // edge records of row i+2
                pre_load(a, pc, i + 2, rp2, rp3, lane, x.pol);
                rp2 = rp3;
                rp3 = i + 4 <= re ? __ldg(a.row_ptr + i + 4) : 0u;
            }
            if (ga.d <= 64) {
                row_fast<MODE>(a, x, T, ga, lane, st);
            } else {
                NodeRec nd;
                nd.diag = ga.nd.x;
                nd.pnum = ga.nd.y;
                row_long<MODE>(a, x, T, ga.i, ga.e0, ga.d, nd, lane, st);
            }
            ga = gb;
            pb = pc;
        }
    }
    __syncthreads();
    sweep_epilogue<kRThreads, MODE, 0>(S.tail, a, s, x.resid, st, tid);
}


// ---- four rows per warp --------------------------------------------------------------------
// rowpar_kernel spends 6 instructions per exclusion-sum term (compare, two moves that select
// the strip base, the load, two adds) because a lane's own slot sits at a lane-specific place
// of every 8-term block, and runs rows of 33..64 edges as two sums per lane with most lanes
// of the second idle.  Here a warp takes FOUR consecutive rows; lane (g, o) = (lane / 8,
// lane % 8) works on row g.  The outgoing edges of a row are taken 8 at a time -- own block b,
// edge j = 8 b + o -- so "is this term block my own block" is the same question for every
// lane of the warp: term blocks b' != b add their 8 terms with immediate offsets (load + two
// adds per term), and only the own block (7 terms) pays for the skip.  Lanes are busy for any
// row length (a row of 40 edges: 5 own blocks of 8 lanes), and the edge divisions run with all
// 32 lanes.  The rows' twin messages land through cp.async in a per-warp shared-memory buffer
// (the next quad's gathers under this quad's walk) and are converted in place into the strip
// {P, P mu}; strips are padded with {-0, -0} to a whole number of blocks and sit at a row
// stride of 66 entries, so the four rows' broadcast loads hit different banks.
//
// QT = slots per lane: the quads hold rows of up to 8 QT edges (longer rows: row_long).  The
// per-slot loops of every stage run QT times under predicates, so a graph is swept by the
// instantiation that just covers its rows (QT = 2, 4, 6 or 8, chosen from the degree counts of
// the build: launch_rowpar) -- config 1 (rows of 17..56 edges) 0.877 ms/sweep with 8 slots,
// 0.798 with 6.
constexpr int kQThreads = 128;
constexpr int kQWarps = kQThreads / 32;
constexpr int kQStride = 66;
template <int QT>
struct __align__(16) QuadBuf {
    static constexpr int kQCap = 8 * QT;
    double2 tw[2][4][kQStride];  // twin messages m_ji of S_{s-1}; then the strip {P, P mu}
                                 // (two quads: the next one lands under this one's walk)
    double c[2][4][kQCap];       // A_ij
    double2 xg[4][kQCap];        // the aligned pair of doubles holding x_j^{(s-2)}: consumed
                                 // by the strip pass, so the next quad's land under the walk
                                 // (which half: a bit mask in the issuing lane's register)
    uint32_t go[2][4][kQCap];    // binned message order: position of the edge's own message
};
static_assert(sizeof(double2) * 4 * kQStride >= sizeof(double2) * (kRowParMaxDegree + 8),
              "a long row's strip fits a quad's strips");
template <int QT>
constexpr size_t quad_bytes() {
    return sizeof(QuadBuf<QT>) * kQWarps;
}

__device__ __forceinline__ void cpa_tw_n(double2 *dst, const double2 *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cpa_u32(uint32_t *dst, const uint32_t *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cpa_f64(double *dst, const double *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ uint2 ld_ef_u2(const uint2 *ptr, uint64_t pol) {
    uint2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;"
                 : "=r"(v.x), "=r"(v.y)
                 : "l"(ptr), "l"(pol));
    return v;
}
__device__ __forceinline__ void cpa_tw(double2 *dst, const double2 *src, uint64_t pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src), "l"(pol)
                 : "memory");
}
// x_j as the aligned 16 bytes around it: cp.async.cg bypasses the L1 (an 8-byte
// cp.async.ca allocates L1 lines: the random x gathers then cost 0.47 ms of a 1.6 ms sweep)
__device__ __forceinline__ void cpa_x2(double2 *dst, const double *x, uint32_t col) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(x + (col & ~1u))
                 : "memory");
}

// this lane's row of a quad
struct QRow {
    uint32_t i = 0xffffffffu, e0 = 0, d = 0;  // d: edges walked here (0 for long rows)
    uint32_t dl = 0;                          // the row's degree when it is a long row
    uint32_t e1 = 0;                          // end offset as loaded (d, dl: QRow::fin)
    // the offsets are loaded a stage before anything depends on them: d and dl are formed
    // when the row moves on, not behind the loads
    __device__ __forceinline__ void fin(uint32_t cap) {
        const uint32_t dd = e1 - e0;
        d = dd <= cap ? dd : 0u;
        dl = dd <= cap ? 0u : dd;
    }
    double2 nd = make_double2(0.0, 0.0);      // {A_ii, A_ii mu_ii}
    double xi = 0.0, bi = 0.0;                // x_i^{(s-2)}, b_i
};

template <int MODE, bool BIN, int QT>
__global__ void __launch_bounds__(kQThreads, 3) rowquad_kernel(const SweepArgs a) {
    constexpr int kQT = QT;
    __shared__ TailSmem<kQWarps> tail;
    __shared__ int64_t s_sweep;
    __shared__ int s_skip;
    extern __shared__ __align__(16) unsigned char quad_raw[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    Ctrl *ctrl = a.ctrl;
    if (tid == 0) {
        if (MODE == kModeSolve) {
            volatile Ctrl *vc = ctrl;
            const int64_t s = vc->next_sweep;
            s_skip = vc->done || s > vc->max_iter + 2;
            s_sweep = s;
        } else {
            s_skip = 0;
            s_sweep = 1;
        }
    }
    __syncthreads();
    if (s_skip) return;
    const int64_t s = s_sweep;
    RowCtx x;
    x.resid = (MODE == kModeSolve) && s >= 3;
    x.min_ = a.msg[(s - 1) % 3];
    x.xprev = x.resid ? a.x[(s - 2) % 3] : nullptr;
    x.mout = a.msg[s % 3];
    x.xcur = (MODE == kModeSolve) ? a.x[(s - 1) % 3] : nullptr;
    x.pcur = (MODE == kModeSolve) ? a.p[(s - 1) % 3] : nullptr;
    x.xh = (MODE == kModeSolve && a.xhist && s >= 2 && s - 1 <= a.xhist_rows)
               ? a.xhist + (s - 2) * a.n : nullptr;
    x.pol = pol_evict_first();
    if (BIN) {
        x.gidx = a.gidx;
        x.gout = a.gout;
    }
    Stats st;
    st.lim = (MODE == kModeSolve) ? fmin(ctrl->blowup, DBL_MAX) : DBL_MAX;
    QuadBuf<QT> &W = reinterpret_cast<QuadBuf<QT> *>(quad_raw)[warp];
    const int g = lane >> 3, o = lane & 7;

    const uint32_t r_lo = __ldg(&a.tile_info[0].x);
    const uint32_t r_hi = __ldg(&a.tile_info[a.ntiles - 1].y);
    const int64_t nw = (int64_t)gridDim.x * kQWarps, gw = (int64_t)blockIdx.x * kQWarps + warp;
    // CSR order: a contiguous block of rows per warp.  Binned order: the quads dealt round
    // robin, so the launch sweeps the rows as one ascending front -- all warps gather from
    // the same bin's window and every bin's writes advance as one run.
    const uint32_t tq = (r_hi - r_lo + 3u) / 4u;
    const uint32_t rb =
        BIN ? r_lo + 4u * (uint32_t)gw : r_lo + (uint32_t)(((int64_t)(r_hi - r_lo) * gw) / nw);
    const uint32_t re =
        BIN ? r_hi : r_lo + (uint32_t)(((int64_t)(r_hi - r_lo) * (gw + 1)) / nw);
    const uint32_t qs = BIN ? 4u * (uint32_t)nw : 4u;  // row stride between a warp's quads
    const uint32_t nq = BIN ? ((int64_t)tq > gw ? (uint32_t)((tq - gw + nw - 1) / nw) : 0u)
                            : (re - rb + 3u) / 4u;

    // row offsets of quad q for this lane's row (empty past the range)
    auto row_of = [&](uint32_t q, QRow &r) {
        r = QRow();
        const uint32_t i = rb + qs * q + (uint32_t)g;
        if (q < nq && i < re) {
            r.i = i;
            r.e0 = __ldg(a.row_ptr + i);
            r.e1 = __ldg(a.row_ptr + i + 1);
        }
    };
    // edge records of the row's slots o, o + 8, ... (registers, consumed by the issue stage)
    auto load_er = [&](const QRow &r, int4 (&er)[kQT]) {
#pragma unroll
        for (int t = 0; t < kQT; ++t) {
            const uint32_t q = (uint32_t)o + 8u * t;
            if (BIN) {  // the two indices only: A_ij goes straight to shared memory later
                const uint2 v = q < r.d ? ld_ef_u2(a.gidx + r.e0 + q, x.pol) : make_uint2(0u, 0u);
                er[t] = make_int4((int)v.x, (int)v.y, 0, 0);
            } else {
                er[t] = q < r.d ? ld_ef_i4(a.er + r.e0 + q, x.pol) : make_int4(0, 0, 0, 0);
            }
        }
    };
    // issue stage, part 1: twin gathers of the row into strip buffer `nb`, coefficients, node
    // operands into registers
    // (issued after the stage's cp.async traffic: a load in flight on the scoreboard of the
    // edge records would hold their consumers back)
    auto node_loads = [&](QRow &r) {
        if (r.i != 0xffffffffu) {
            r.nd = __ldg(reinterpret_cast<const double2 *>(a.nd + r.i));
            if (x.resid) {
                r.xi = __ldg(x.xprev + r.i);
                r.bi = __ldg(a.rhs + r.i);
            }
        }
    };
    auto issue_tw = [&](const QRow &r, const int4 (&er)[kQT], int nb) {
#pragma unroll
        for (int t = 0; t < kQT; ++t) {
            const uint32_t q = (uint32_t)o + 8u * t;
            if (q < r.d) {
                const EdgeRec e = er_of(er[t]);
                if (BIN)
                    cpa_f64(&W.c[nb][g][q], a.gcoef + r.e0 + q);
                else
                    W.c[nb][g][q] = e.coeff;
#ifdef GABP_ROW_PROBE_COALESCED  // probe build (wrong results): no random twin gather
                cpa_tw(&W.tw[nb][g][q], x.min_ + r.e0 + q, x.pol);
#else
                if (BIN) {
                    cpa_tw_n(&W.tw[nb][g][q], x.min_ + e.rev);
                    cpa_u32(&W.go[nb][g][q], a.gout + r.e0 + q);
                } else {
                    cpa_tw(&W.tw[nb][g][q], x.min_ + e.rev, x.pol);
                }
#endif
            }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    // part 2 (after the strip pass has consumed the previous quad's x): the x_j gathers
    uint32_t pm = 0u;  // which half of the landed pair is x_j, a bit per slot of this lane
    auto issue_x = [&](const QRow &r, const int4 (&er)[kQT]) {
#ifndef GABP_ROW_PROBE_NOX
        if (x.resid) {
            pm = 0u;
#pragma unroll
            for (int t = 0; t < kQT; ++t) {
                    const uint32_t q = (uint32_t)o + 8u * t;
                if (q < r.d) {
                    const uint32_t col = (uint32_t)er[t].y;
                    pm |= (col & 1u) << t;
                    cpa_x2(&W.xg[g][q], x.xprev, col);
                }
            }
        }
#endif
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };

    if (nq > 0) {
        QRow rc, ri, rl, rn;  // rows of the quad being walked, issued, loaded; offsets ahead
        int4 er[kQT];
        row_of(0, ri);
        ri.fin(8u * QT);
        load_er(ri, er);
        issue_tw(ri, er, 0);
        issue_x(ri, er);
        node_loads(ri);
        row_of(1, rl);
        rl.fin(8u * QT);
        row_of(2, rn);
        load_er(rl, er);
        for (uint32_t q = 0; q < nq; ++q) {
            const int cb = (int)(q & 1u);
            rc = ri;
            ri = rl;
            rl = rn;  // (its offsets were loaded a quad ago: no dependent load before load_er)
            rl.fin(8u * QT);
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");  // quad q has landed
            __syncwarp();
            issue_tw(ri, er, cb ^ 1);  // quad q + 1 (empty past the range)
            double2 *Tg = W.tw[cb][g];
            const double *Cg = W.c[cb][g];
            // strip in place, the row's residual partial
            const uint32_t nbmax = __reduce_max_sync(~0u, (rc.d + 7u) >> 3);
            double yp = 0.0;
#pragma unroll
            for (int t = 0; t < kQT; ++t) {
                const uint32_t k = (uint32_t)o + 8u * t;
                if (k < rc.d) {
                    const double2 v = Tg[k];
                    Tg[k] = make_double2(v.x, v.x * v.y);  // (prec * mean), solver.py:148
                    if (x.resid) {
                        const double2 xp = W.xg[g][k];
                        yp = yp + Cg[k] * ((pm >> t) & 1u ? xp.y : xp.x);
                    }
                } else if (k < 8u * nbmax) {
                    Tg[k] = make_double2(-0.0, -0.0);
                }
            }
            __syncwarp();
            issue_x(ri, er);  // (the x buffer is free again)
            node_loads(ri);
            load_er(rl, er);
            row_of(q + 3, rn);
            if (x.resid) {  // sum over the row's 8 lanes
                yp += __shfl_xor_sync(~0u, yp, 1);
                yp += __shfl_xor_sync(~0u, yp, 2);
                yp += __shfl_xor_sync(~0u, yp, 4);
            }
            // Own blocks two at a time: the lane's edges j0 = 8 b + o and j1 = j0 + 8 share
            // every term load outside their own blocks and give the lane four independent add
            // chains.  The edges' own messages of S_{s-1} (change statistic) are loaded a
            // step ahead.
            const uint32_t *Gg = W.go[cb][g];
            auto ld_old = [&](uint32_t j) {
                if (j >= rc.d) return make_double2(0.0, 0.0);
                return BIN ? ld_na_d2(x.min_ + Gg[j]) : ld_ef_d2(x.min_ + rc.e0 + j, x.pol);
            };
            // the row's full sums: the last exclusion sum + the last term, kept by the lane of
            // the row's last edge (the node division runs once per quad, after the walk)
            double fsp = rc.nd.x, fsn = rc.nd.y;
            auto finish = [&](uint32_t j, double p, double n, double2 old) {
                if (j < rc.d) {
                    edge_out<BIN>(x, rc.e0 + j, BIN ? Gg[j] : rc.e0 + j, Cg[j], p, n, old, st);
                    if (j == rc.d - 1u) {
                        const double2 own = Tg[j];
                        fsp = p + own.x;
                        fsn = n + own.y;
                    }
                }
            };
            double2 oa = ld_old((uint32_t)o), ob = ld_old((uint32_t)o + 8u);
            // The sequential sum before term block b -- prior + t_0 + ... + t_{8b-1} -- is
            // common to every exclusion sum of the blocks from b on: it is carried (rp, rn_)
            // and each own block's sums start from it and walk only the blocks b.., the same
            // additions in the same order.  Sum 1 of a pair *is* the carried prefix while it
            // runs through block b; the prefix past block b + 1 is one more addition on the
            // lane that skipped the block's last slot (o = 7), broadcast to the row's lanes.
            double rp = rc.nd.x, rn_ = rc.nd.y;
            // one step: own blocks b and b + 1 (their old messages in o0, o1)
            auto walk_pair = [&](uint32_t b, const double2 &o0, const double2 &o1) {
                const uint32_t j0 = 8u * b + (uint32_t)o, j1 = j0 + 8u;
                double p0 = rp, n0 = rn_, p1 = rp, n1 = rn_;
                {  // block b: sum 0 skips its slot (an address select), sum 1 adds all
                    const double2 *base = Tg + 8u * b;
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const double2 v = base[k];
                        p1 = p1 + v.x;
                        n1 = n1 + v.y;
                        if (k < 7) {
                            const double2 w = (o > k ? base : base + 1)[k];
                            p0 = p0 + w.x;
                            n0 = n0 + w.y;
                        }
                    }
                }
                {  // block b + 1: the other way round
                    const double2 *base = Tg + 8u * (b + 1u);
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const double2 v = base[k];
                        p0 = p0 + v.x;
                        n0 = n0 + v.y;
                        if (k < 7) {
                            const double2 w = (o > k ? base : base + 1)[k];
                            p1 = p1 + w.x;
                            n1 = n1 + w.y;
                        } else if (b + 2u < nbmax) {  // lane o = 7: (p1, n1) + t_7 = the prefix
                            rp = __shfl_sync(~0u, p1 + v.x, 7, 8);
                            rn_ = __shfl_sync(~0u, n1 + v.y, 7, 8);
                        }
                    }
                }
                for (uint32_t bp = b + 2u; bp < nbmax; ++bp) {
                    const double2 *base = Tg + 8u * bp;
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const double2 v = base[k];
                        p0 = p0 + v.x;
                        n0 = n0 + v.y;
                        p1 = p1 + v.x;
                        n1 = n1 + v.y;
                    }
                }
                finish(j0, p0, n0, o0);
                finish(j1, p1, n1, o1);
            };
            auto walk_last = [&](uint32_t b, const double2 &o0) {  // an odd last own block:
                const uint32_t j0 = 8u * b + (uint32_t)o;           // terms 0..o-1, o+1..7
                double p0 = rp, n0 = rn_;
                const double2 *base = Tg + 8u * b;
#pragma unroll
                for (int k = 0; k < 7; ++k) {
                    const double2 v = (o > k ? base : base + 1)[k];
                    p0 = p0 + v.x;
                    n0 = n0 + v.y;
                }
                finish(j0, p0, n0, o0);
            };
            // The old messages of a step are loaded a step ahead into the register pair the
            // step before last used (two alternating pairs: no copy of a register whose load
            // is still in flight).
            double2 oc = make_double2(0.0, 0.0), od = oc;
            uint32_t b = 0;
            for (;;) {
                if (b + 1 >= nbmax) {
                    if (b < nbmax) walk_last(b, oa);
                    break;
                }
                oc = ld_old(8u * b + 16u + (uint32_t)o);
                od = ld_old(8u * b + 24u + (uint32_t)o);
                walk_pair(b, oa, ob);
                b += 2;
                if (b + 1 >= nbmax) {
                    if (b < nbmax) walk_last(b, oc);
                    break;
                }
                oa = ld_old(8u * b + 16u + (uint32_t)o);
                ob = ld_old(8u * b + 24u + (uint32_t)o);
                walk_pair(b, oc, od);
                b += 2;
            }
            const bool plain = rc.i != 0xffffffffu && rc.dl == 0u;
            // (an isolated row: its prior, on lane o = 0)
            if (plain && (uint32_t)o == (rc.d == 0u ? 0u : (rc.d - 1u) & 7u))
                row_node<MODE>(a, x, rc.i, fsp, fsn, st);
            if (x.resid && plain && o == 0) {
                const double y = rc.nd.x * rc.xi + yp;
                const double res = y - rc.bi;
                st.rsq += res * res;
            }
            __syncwarp();
            // rows of more than 8 QT edges: the whole warp, one row at a time, on the buffer
            const unsigned lmask = __ballot_sync(~0u, rc.dl != 0u && o == 0);
            for (int gg = 0; lmask != 0u && gg < 4; ++gg) {
                if (lmask & (1u << (8 * gg))) {
                    const int src = 8 * gg;
                    NodeRec nd;
                    nd.diag = __shfl_sync(~0u, rc.nd.x, src);
                    nd.pnum = __shfl_sync(~0u, rc.nd.y, src);
                    row_long<MODE>(a, x, &W.tw[cb][0][0], __shfl_sync(~0u, rc.i, src),
                                   __shfl_sync(~0u, rc.e0, src), __shfl_sync(~0u, rc.dl, src),
                                   nd, lane, st);
                    __syncwarp();
                }
            }
        }
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    sweep_epilogue<kQThreads, MODE, 0>(tail, a, s, x.resid, st, tid);
}


// ---- serial schedule (solver.py:176-217) as dependency levels ------------------------------
// The reference updates node by node in a given order, in place: node i recomputes all its
// outgoing messages m_ij from its current incoming messages m_ki.  Two tasks interact only
// when they are on the same node or on adjacent nodes (i reads m_ki that k writes, and k
// reads m_ik that i writes), so tasks grouped into dependency levels (level(t) = 1 + the
// highest level of an earlier task on node(t) or a neighbour; capi.cu: serial_levels) and
// run level after level give the sequential result bit for bit: a task sees exactly the
// messages the sequential loop would show it.  One launch per level, a warp per task; the
// task's d exclusion sums run one per lane as in rowpar_kernel (rows <= 256 edges).
// One serial task {node, order position}: node i's outgoing messages from its current
// incoming ones, in place on msg (solver.py:181-209).
// Tasks longer than the shared-memory strip (kRowParMaxDegree) keep their terms in the
// warp's slice of a global scratch strip (a.strip, gw = the warp's global index).
__device__ __forceinline__ void serial_task(const SweepArgs &a, double2 *msg, uint2 tk,
                                            double2 *Tsm, int64_t gw, int lane, Stats &st) {
    const uint32_t i = tk.x;
    const uint32_t e0 = __ldg(a.row_ptr + i), d = __ldg(a.row_ptr + i + 1) - e0;
    double2 *T = d > (uint32_t)kRowParMaxDegree ? a.strip + gw * a.strip_stride : Tsm;
    const double2 nd = __ldg(reinterpret_cast<const double2 *>(a.nd + i));
    const uint32_t dpad = (d + 7u) & ~7u;
    for (uint32_t q = lane; q < dpad; q += 32) {
        if (q < d) {
            const EdgeRec r = ld_er(a.er + e0 + q);
            const double2 in = __ldcg(msg + r.rev);  // m_ki as the loop would see it
            T[q] = make_double2(in.x, in.x * in.y);
        } else {
            T[q] = make_double2(-0.0, -0.0);
        }
    }
    __syncwarp();
    for (uint32_t jb = 0; jb < d; jb += 32) {
        const uint32_t j = jb + lane;
        double p = nd.x, n = nd.y;
        for (uint32_t t = 0; t < dpad; t += 8) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const double2 v = T[t + k];
                if (t + k != j) {
                    p = p + v.x;
                    n = n + v.y;
                }
            }
        }
        if (j < d) {
            const uint32_t e = e0 + j;
            const double c = __ldg(&a.er[e].coeff);
            const double2 old = __ldcg(msg + e);
            bool okp, okm;
            double np_ = ddiv_fast(-c * c, p, okp);
            double nm = ddiv_fast(n, c, okm);
            if (!okp) np_ = div_slow(-c * c, p);
            if (!okm) nm = div_slow(n, c);
            if (p == 0.0)  // the first in loop order: (order position, edge)
                atomicMin(&a.ctrl->singular_min[1],
                          ((unsigned long long)tk.y << 32) | (unsigned long long)e);
            __stcg(msg + e, make_double2(np_, nm));
            const double d1 = fabs(np_ - old.x), d2 = fabs(nm - old.y);
            st.chg = d1 > st.chg ? d1 : st.chg;
            st.chg = d2 > st.chg ? d2 : st.chg;
            if (!(fabs(np_) <= st.lim) || !(fabs(nm) <= st.lim)) st.out_of_range = 1u;
        }
    }
    __syncwarp();  // the strip is rewritten by the next task
}

// Software grid barrier of a cooperative launch (every CTA resident): arrive, and the last
// CTA to arrive opens the next generation.  Writes before it are visible after it (fences
// on both sides; messages are read through L2).
__device__ __forceinline__ void grid_barrier(Ctrl *c, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned *gen = &c->bar_gen;
        const unsigned g = *gen;
        __threadfence();
        if (atomicAdd(&c->bar_count, 1u) == nblocks - 1u) {
            c->bar_count = 0u;
            __threadfence();
            atomicAdd(&c->bar_gen, 1u);
        } else {
            while (*gen == g) __nanosleep(20);
        }
        __threadfence();
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kRThreads, 2) serial_level_kernel(const SweepArgs a,
                                                                   const uint2 *tasks,
                                                                   int64_t cnt, double lim) {
    __shared__ RowSmem S;
    double2 *msg = reinterpret_cast<double2 *>(
        __ldcg(reinterpret_cast<const unsigned long long *>(&a.ctrl->serial_msg)));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    Stats st;
    st.lim = lim;
    const int64_t nw = (int64_t)gridDim.x * kRWarps, gw = (int64_t)blockIdx.x * kRWarps + warp;
    for (int64_t w = gw; w < cnt; w += nw)
        serial_task(a, msg, __ldg(tasks + w), S.T[warp], gw, lane, st);
    __syncthreads();
    sweep_epilogue<kRThreads, kModeSingle, 0>(S.tail, a, 1, false, st, tid);
}

// The whole sweep in one cooperative launch: level after level, a grid barrier between
// levels.  Used for orders with few, wide levels (config 1: 88 levels, 2.89 -> 2.46 ms per
// sweep against the graph of level launches); with thousands of narrow levels (a 4096^2
// grid: 8191) a barrier costs more than a dependent launch in a graph (44.7 vs 39.8 ms).
__global__ void __launch_bounds__(kRThreads, 2) serial_sweep_kernel(const SweepArgs a,
                                                                   const uint2 *tasks,
                                                                   const int64_t *lvl,
                                                                   int nlev, double lim) {
    __shared__ RowSmem S;
    double2 *msg = reinterpret_cast<double2 *>(
        __ldcg(reinterpret_cast<const unsigned long long *>(&a.ctrl->serial_msg)));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    Stats st;
    st.lim = lim;
    const int64_t nw = (int64_t)gridDim.x * kRWarps;
    const int64_t gw = (int64_t)blockIdx.x * kRWarps + warp;
    for (int l = 0; l < nlev; ++l) {
        const int64_t lo = __ldg(lvl + l), cnt = __ldg(lvl + l + 1) - lo;
        for (int64_t w = gw; w < cnt; w += nw)
            serial_task(a, msg, __ldg(tasks + lo + w), S.T[warp], gw, lane, st);
        if (l + 1 < nlev) grid_barrier(a.ctrl, gridDim.x);
    }
    __syncthreads();
    sweep_epilogue<kRThreads, kModeSingle, 0>(S.tail, a, 1, false, st, tid);
}

// Destination column of every edge record (the host builds the serial levels from the CSR
// without copying the 16-byte records).
__global__ void edge_col_kernel(int64_t E, const EdgeRec *er, uint32_t *col) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E;
         e += (int64_t)gridDim.x * blockDim.x)
        col[e] = __ldg(&er[e].col);
}

constexpr int kMaxDevices = 64;
int g_row_grid[kMaxDevices][2] = {};   // persistent grids per device (prepare_rowpar_kernels)
int g_coop_grid[kMaxDevices] = {};     // cooperative serial sweep: every CTA resident
// rowquad_kernel grids: [device][slots per lane / 2 - 1][solve CSR, solve binned, single]
int g_quad_grid[kMaxDevices][4][3] = {};

int cur_dev() {
    int d = 0;
    cudaGetDevice(&d);
    return d >= 0 && d < kMaxDevices ? d : 0;
}

template <int QT>
cudaError_t prepare_quad(int dv, int sms) {
    const int bytes = (int)quad_bytes<QT>();
    const void *fn[3] = {(const void *)rowquad_kernel<kModeSolve, false, QT>,
                         (const void *)rowquad_kernel<kModeSolve, true, QT>,
                         (const void *)rowquad_kernel<kModeSingle, false, QT>};
    for (int k = 0; k < 3; ++k) {
        cudaError_t e =
            cudaFuncSetAttribute(fn[k], cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        if (e != cudaSuccess) return e;
        int occ = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn[k], kQThreads, bytes);
        if (e != cudaSuccess) return e;
        g_quad_grid[dv][QT / 2 - 1][k] = sms * (occ > 0 ? occ : 1);
    }
    return cudaSuccess;
}

template <int QT>
cudaError_t launch_quad(const SweepArgs &a, int which, int dv, cudaStream_t st) {
    int64_t grid = g_quad_grid[dv][QT / 2 - 1][which];
    if (grid <= 0) grid = 148 * 3;
    const int64_t need = (a.ntiles + kQWarps - 1) / kQWarps;
    if (grid > need) grid = need;
    const size_t bytes = quad_bytes<QT>();
    if (which == 1)
        rowquad_kernel<kModeSolve, true, QT><<<(unsigned)grid, kQThreads, bytes, st>>>(a);
    else if (which == 0)
        rowquad_kernel<kModeSolve, false, QT><<<(unsigned)grid, kQThreads, bytes, st>>>(a);
    else
        rowquad_kernel<kModeSingle, false, QT><<<(unsigned)grid, kQThreads, bytes, st>>>(a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t prepare_rowpar_kernels() {
    int dev = 0, sms = 0;
    cudaError_t e;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess)
        return e;
    int occ = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, rowpar_kernel<kModeSolve>,
                                                           kRThreads, 0)) != cudaSuccess)
        return e;
    const int dv = dev >= 0 && dev < kMaxDevices ? dev : 0;
    g_row_grid[dv][kModeSolve] = sms * (occ > 0 ? occ : 1);
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, rowpar_kernel<kModeSingle>,
                                                           kRThreads, 0)) != cudaSuccess)
        return e;
    g_row_grid[dv][kModeSingle] = sms * (occ > 0 ? occ : 1);
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, serial_sweep_kernel, kRThreads,
                                                           0)) != cudaSuccess)
        return e;
    g_coop_grid[dv] = sms * (occ > 0 ? occ : 1);
    if ((e = prepare_quad<2>(dv, sms)) != cudaSuccess ||
        (e = prepare_quad<4>(dv, sms)) != cudaSuccess ||
        (e = prepare_quad<6>(dv, sms)) != cudaSuccess ||
        (e = prepare_quad<8>(dv, sms)) != cudaSuccess)
        return e;
    return cudaSuccess;
}

cudaError_t launch_serial_level(const SweepArgs &a, const uint2 *tasks, int64_t cnt, double lim,
                                cudaStream_t st) {
    if (cnt <= 0) return cudaSuccess;
    const int dv = cur_dev();
    int64_t grid = g_row_grid[dv][kModeSingle] > 0 ? g_row_grid[dv][kModeSingle] : 148 * 2;
    const int64_t need = (cnt + kRWarps - 1) / kRWarps;
    if (grid > need) grid = need;
    serial_level_kernel<<<(unsigned)grid, kRThreads, 0, st>>>(a, tasks, cnt, lim);
    return cudaGetLastError();
}

int64_t serial_strip_warps() {
    const int dv = cur_dev();
    const int64_t a = g_coop_grid[dv], b = g_row_grid[dv][kModeSingle];
    return (a > b ? a : b) * kRWarps;
}

cudaError_t launch_edge_col(int64_t E, const EdgeRec *er, uint32_t *col, cudaStream_t st) {
    if (E <= 0) return cudaSuccess;
    edge_col_kernel<<<148 * 8, 256, 0, st>>>(E, er, col);
    return cudaGetLastError();
}

cudaError_t launch_serial_sweep(const SweepArgs &a, const uint2 *tasks, const int64_t *lvl,
                                int nlev, int64_t max_cnt, double lim, cudaStream_t st) {
    if (nlev <= 0) return cudaSuccess;
    const int dv = cur_dev();
    if (g_coop_grid[dv] <= 0) return cudaErrorInitializationError;  // prepare_rowpar_kernels
    int64_t grid = g_coop_grid[dv];
    const int64_t need = (max_cnt + kRWarps - 1) / kRWarps;
    if (grid > need) grid = need > 0 ? need : 1;
    void *args[] = {(void *)&a, (void *)&tasks, (void *)&lvl, (void *)&nlev, (void *)&lim};
    return cudaLaunchCooperativeKernel((const void *)serial_sweep_kernel, dim3((unsigned)grid),
                                       dim3(kRThreads), args, 0, st);
}

cudaError_t launch_rowpar(const SweepArgs &a, int mode, cudaStream_t st) {
    if (a.ntiles <= 0) return cudaSuccess;
    const int m = mode == kModeSolve ? kModeSolve : kModeSingle;
    const int dv = cur_dev();
    const bool quad = !getenv("GABP_ROW_NO_QUAD");
    if (quad) {
        const bool bin = m == kModeSolve && a.gout && a.gidx && a.gcoef;
        const int which = bin ? 1 : m == kModeSolve ? 0 : 2;
        // slots per lane: the instantiation that just covers the graph's rows (a.quad_slots
        // from the degree counts of the build; rows past it take the long-row path)
        const int qt = a.quad_slots <= 2 ? 2 : a.quad_slots <= 4 ? 4 : a.quad_slots <= 6 ? 6 : 8;
        if (qt == 2) return launch_quad<2>(a, which, dv, st);
        if (qt == 4) return launch_quad<4>(a, which, dv, st);
        if (qt == 6) return launch_quad<6>(a, which, dv, st);
        return launch_quad<8>(a, which, dv, st);
    }
    int64_t grid = g_row_grid[dv][m] > 0 ? g_row_grid[dv][m] : 148 * 4;
    const int64_t need = (a.ntiles + kRWarps - 1) / kRWarps;
    if (grid > need) grid = need;
    if (m == kModeSolve)
        rowpar_kernel<kModeSolve><<<(unsigned)grid, kRThreads, 0, st>>>(a);
    else
        rowpar_kernel<kModeSingle><<<(unsigned)grid, kRThreads, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace gabp
