// slice.cu -- broadcast-schedule solve sweep over the slice layout (lane per row).
//
// Layout (build_slices below).  The swept rows are stably
// sorted by degree (descending) inside windows of kSortWin rows and cut into slices of 32
// rows; row r of the sort sits at "position" p = 32 * slice + lane.  kGroup consecutive
// slices form a group of width w_g = its largest degree (the first row's, as the rows are
// sorted), and the q-th edge (ascending neighbour, = reference edge order) of the row in
// lane l of slice s lives at slot base_s + kStride q + l, base_s = gbase_g + 32 (s % kGroup):
// column q of a group is kStride = 32 kGroup contiguous slots.  Nodes are numbered by
// position on this path (x, p and the aggregates live in position order; scol holds the
// neighbour's position; a rank's halo rows take positions after the owned ones), so every
// own-row and every per-edge stream is a fully coalesced warp access (and a group chunk one
// bulk copy per stream), and only the neighbour gathers are random (node arrays,
// L2-resident for the headline graph).
//
// State on this path: per edge slot the INCOMING message I_ij^{(t)} = m_ji^{(t)} = (P, mu)
// of S_t (the term row i sums), a ring of three; per node the aggregate {P_i, P_i mu~_i}
// of S_t, a ring of three.  Launch s (one sweep, solver.py:232-272):
//   m_ij^{(s-2)} = msg(agg_i(S_{s-3}), I_ij^{(s-3)})    own outgoing message, rebuilt with
//                                                     the operands launch s-2 used
//   I_ij^{(s-1)} = msg(agg_j(S_{s-2}), m_ij^{(s-2)})    = m_ji^{(s-1)} exactly as row j's
//                                                     sweep s-1 built it (same bits)
//   P_i = A_ii + sum_j P_ji, N_i = A_ii mu_ii + sum_j P_ji mu_ji   ascending j (np.add.at)
//   x_i^{(s-1)} = N_i / P_i, agg_i(S_{s-1}) = {P_i, P_i x_i}, residual row of x^{(s-2)}
// with msg(agg, m) = (-A_ij^2 / (agg.P - m.P), (agg.N - m.P m.mu) / A_ij) (solver.py:249-257).
// Every directed message is exactly one row's incoming message, so sweep s-1's statistics
// (max |change| against I^{(s-2)}, blowup, P_excl == 0 with the reference's edge id) are
// taken on I^{(s-1)} here -- one launch after the sweep, one launch before its decision
// (Ctrl statistic slots, LAG = 1).  Per edge: 4 divisions, 44 B read + 16 B written in one
// streaming pass; no staging, no CTA barrier.
// Launch 1 sees I^{(0)} = 0 (solve_setup zeroes the ring); launch 2 uses m^{(0)} = 0.
#include <cub/device/device_scan.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <stdio.h>
#include <stdlib.h>

#include "sweep_common.cuh"

namespace gabp {
namespace {

#ifndef GABP_SLICE_GROUP
#define GABP_SLICE_GROUP 15
#endif
constexpr int kGroup = GABP_SLICE_GROUP;  // slices per group (consumer warps per CTA)
constexpr int kStride = 32 * kGroup;      // slots per group column

// ---- shared pieces -----------------------------------------------------------------------
struct SliceSmem {
    TailSmem<8> tail;  // up to 256 threads per CTA
    int64_t sweep;
    int skip;
    int probe;
};

// IEEE a / b.  The fast kernels use the replicated div.rn fast path only and flag the
// launch when an operand leaves its range (the exact twin then redoes the sweep): no call
// in the hot loop, so no ABI-preserved registers.
template <bool EXACT>
__device__ __forceinline__ double qdiv(double a, double b, Stats &st) {
    if (EXACT) return a / b;
    return ddiv_fast_acc(a, b, st.dr);
}

// msg(agg, m): the outgoing message of an edge from its row aggregate and the incoming
// pair, as (P, mu) (solver.py:249-257)
// rc = ddiv_rcp(c): both messages of an edge divide by A_ij and share the reciprocal
template <bool EXACT>
__device__ __forceinline__ void edge_msg(double c, double rc, double pe, double num, double &P,
                                         double &mu, Stats &st) {
    P = qdiv<EXACT>(-c * c, pe, st);
    mu = EXACT ? num / c : ddiv_fast_acc_r(num, c, rc, st.dr);
}

// CSR edge id of the message j -> i held in slot q of position p (exact launch only)
__device__ __forceinline__ uint32_t twin_edge(const SweepArgs &a, int64_t p, uint32_t q) {
    return a.er[a.row_ptr[a.srow[p]] + q].rev;
}

// (the numerator (sum_p * mu_tilde), solver.py:254, is formed where it is used -- P * x at
// the load would make the lane wait for the gather it has just issued)
__device__ __forceinline__ void ld_node(const NodeState *g, double &P, double &x) {
#ifdef GABP_NODE16
    asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];" : "=d"(P), "=d"(x) : "l"(g));
#else
    double p0, p1;  // (the whole sector: one 256-bit load)
    asm volatile("ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(P), "=d"(x), "=d"(p0), "=d"(p1) : "l"(g));
#endif
}
// L2 policies of the node-state traffic (GABP_GATHER_POLICY): the gathered states S_{s-2}
// are a random-access working set of 32 B x nodes that the message streams (evict-first)
// must not push out of L2; the written states S_{s-1} are next launch's gather set.
// Measured on config 1 (tools/gpu/lib_ab.sh, profiles/r02_evidence.md): 0 = no hints 0.365
// ms/sweep; 1 = gathered and written states evict-last, the own S_{s-3} read evict-first
// 0.362; 2 = also the once-per-launch row header (prior, degree, b_i) without L1 allocation
// and evict-first 0.360 (the L1 holds the in-flight gathers: a 5-stage ring, which leaves
// 28 KB of L1, runs 0.448).
#ifndef GABP_GATHER_POLICY
#define GABP_GATHER_POLICY 2
#endif
__device__ __forceinline__ uint64_t pol_evict_last_node() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t pol_evict_first_node() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void ld_node_pol(const NodeState *g, double &P, double &x,
                                            uint64_t pol) {
#ifdef GABP_NODE16
    asm volatile("ld.global.cg.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(P), "=d"(x) : "l"(g), "l"(pol));
#else
    double p0, p1;
    asm volatile("ld.global.cg.L2::cache_hint.v4.f64 {%0, %1, %2, %3}, [%4], %5;"
                 : "=d"(P), "=d"(x), "=d"(p0), "=d"(p1) : "l"(g), "l"(pol));
#endif
}
__device__ __forceinline__ void st_node_pol(NodeState *g, double P, double x, uint64_t pol) {
#ifdef GABP_NODE16
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(g), "d"(P), "d"(x),
                 "l"(pol) : "memory");
#else
    asm volatile("st.global.L2::cache_hint.v4.f64 [%0], {%1, %2, %3, %3}, %4;" ::"l"(g), "d"(P),
                 "d"(x), "d"(0.0), "l"(pol) : "memory");
#endif
}
__device__ __forceinline__ double2 ld_f64x2_pol(const double2 *p, uint64_t pol) {
    double2 v;
    asm volatile("ld.global.cg.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_node(NodeState *g, double P, double x) {
#ifdef GABP_NODE16
    asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(g), "d"(P), "d"(x) : "memory");
#else  // (whole sectors: a partial-sector store costs a fill)
    asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %3};" ::"l"(g), "d"(P), "d"(x), "d"(0.0)
                 : "memory");
#endif
}

// Statistics of sweep s-1 on its message j -> i = (ip, im) against S_{s-2}'s (i2).
// A zero P_excl is reported by the exact launch only: in the fast one the division by it
// yields a NaN quotient, which fails the deferred range test and flags the launch.
template <bool EXACT>
__device__ __forceinline__ void msg_stats(Stats &st, const SweepArgs &a, double ip, double im,
                                          double2 i2, double pe, int64_t p, uint32_t q) {
    const double d1 = fabs(ip - i2.x), d2 = fabs(im - i2.y);
    st.chg = fmax(st.chg, fmax(d1, d2));  // NaN differences ignored, as '>' ignores them
    if (!(fabs(ip) <= st.lim) || !(fabs(im) <= st.lim))
        st.out_of_range |= (ip != ip || im != im) ? 3u : 1u;  // bit 1: a NaN change
    if (EXACT && pe == 0.0) st.sing = min(st.sing, twin_edge(a, p, q));
}

// Row done: marginal of S_{s-1} and the node state record (solver.py:247-255, 286).
template <int PH, bool EXACT, bool ACC = true>
__device__ __forceinline__ double node_done(Stats &st, const SweepArgs &a, NodeState *rec1,
                                            double *xh, int64_t p, double sp, double sn,
                                            double y, double rhs_i) {
    const double xi = qdiv<EXACT>(sn, sp, st);
    if (!(fabs(xi) <= DBL_MAX)) st.means_bad = 1u;
    if (xh) xh[__ldg(a.srow + p)] = xi;
    if (EXACT && sp == 0.0)  // (fast launch: N / 0 fails the deferred range test)
        st.agg_sing = min(st.agg_sing, __ldg(a.srow + p));
#if GABP_GATHER_POLICY >= 1
    st_node_pol(rec1 + p, sp, xi, pol_evict_last_node());
#else
    st_node(rec1 + p, sp, xi);
#endif
    if (PH == 3) {
        const double r = y - rhs_i;
        if (ACC) st.rsq += r * r;
        return r * r;
    }
    return 0.0;
}

// Ring pointers of launch s, R = s % 3 as a constant (kernel-parameter loads).
template <int R>
struct Ring {
    const double2 *I2, *I3;  // I^{(s-2)}, I^{(s-3)}
    double2 *I1;             // I^{(s-1)}, written
    const NodeState *g2, *g3;  // node state of S_{s-2} (gathered), S_{s-3} (own)
    NodeState *g1;           // node state of S_{s-1}, written
    __device__ __forceinline__ Ring(const SweepArgs &a)
        : I2(a.msg[(R + 1) % 3]), I3(a.msg[R]), I1(a.msg[(R + 2) % 3]),
          g2(a.rec[(R + 1) % 3]), g3(a.rec[R]), g1(a.rec[(R + 2) % 3]) {}
};

__device__ __forceinline__ double *xhist_row(const SweepArgs &a, int64_t s) {
    return (a.xhist && s >= 2 && s - 1 <= a.xhist_rows) ? a.xhist + (s - 2) * a.n : nullptr;
}

// Launch 1: the incoming messages of S_0 are +0, so each row's sums are its prior plus +0.
template <int NW, bool EXACT>
__device__ __forceinline__ void slice_first(const SweepArgs &a, int64_t s, Stats &st, int lane) {
    NodeState *rec1 = a.rec[0];  // S_0 (s = 1)
    double *xh = xhist_row(a, s);
    const int64_t nwarps = (int64_t)gridDim.x * NW;
    for (int64_t sl = a.sl_lo + (int64_t)blockIdx.x * NW + (threadIdx.x >> 5); sl < a.sl_hi;
         sl += nwarps) {
        const int64_t p = sl * 32 + lane;
        const double2 nd = __ldg(a.snd + p);
        const uint32_t d = __ldg(a.sdeg + p);
        double sp = nd.x, sn = nd.y;
        if (d > 0) {  // P + 0 (+ 0 ...) == P + 0
            sp = sp + 0.0;
            sn = sn + 0.0;
        }
        if (nd.x != 0.0) node_done<1, EXACT>(st, a, rec1, xh, p, sp, sn, 0.0, 0.0);
    }
}

// ---- variant 0: register batches (long rows) -----------------------------------------------
// A warp walks its slices; per batch of kUL edge columns every lane issues its contiguous
// loads (scoef, scol, I^{(s-2)}, I^{(s-3)}) as one group, then the 256-bit neighbour
// gathers, then computes.  Slot arrays are padded by kUL columns, so loads past a slice's
// width stay in bounds and need no predicate.
#ifndef GABP_SLICE_UL
#define GABP_SLICE_UL 3
#endif
constexpr int kUL = GABP_SLICE_UL;
constexpr int kLThreads = 256;
constexpr int kLWarps = kLThreads / 32;

__device__ __forceinline__ double ldcs_f64(const double *p) {
    double v;
    asm volatile("ld.global.cs.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint32_t ldcs_u32(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.global.cs.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ double2 ldcs_f64x2(const double2 *p) {
    double2 v;
    asm volatile("ld.global.cs.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}

template <int PH, int R, bool EXACT>
__device__ __forceinline__ void slice_sweep_ldg(const SweepArgs &a, int64_t s, Stats &st,
                                                int lane) {
    const Ring<R> r(a);
    double *xh = xhist_row(a, s);
    const int64_t nwarps = (int64_t)gridDim.x * kLWarps;
    for (int64_t sl = a.sl_lo + (int64_t)blockIdx.x * kLWarps + (threadIdx.x >> 5); sl < a.sl_hi;
         sl += nwarps) {
        const uint2 si = __ldg(a.slice_info + sl);
        const int64_t p = sl * 32 + lane;
        const uint32_t d = __ldg(a.sdeg + p);
        const double2 nd = __ldg(a.snd + p);
        double2 a3 = make_double2(0.0, 0.0);
        double y = 0.0, rhs_i = 0.0;
        if (PH == 3) {
            a3 = __ldcg(reinterpret_cast<const double2 *>(r.g3 + p));  // {P_i, x_i}
            a3.y = a3.x * a3.y;  // (sum_p * mu_tilde), solver.py:254
            y = nd.x * __ldcg(&r.g2[p].x);
            rhs_i = __ldg(a.srhs + p);
        }
        double sp = nd.x, sn = nd.y;
        const uint32_t base = si.x + lane, w = si.y;
        uint32_t coln[kUL];  // scol of the next batch, loaded one batch ahead
#pragma unroll
        for (int u = 0; u < kUL; ++u) coln[u] = ldcs_u32(a.scol + base + (uint32_t)kStride * u);
        for (uint32_t q0 = 0; q0 < w; q0 += kUL) {
            double c[kUL];
            uint32_t col[kUL];
            double2 i2[kUL], i3[kUL];
#pragma unroll
            for (int u = 0; u < kUL; ++u) col[u] = coln[u];
            double gP[kUL], gx[kUL];
#pragma unroll
            for (int u = 0; u < kUL; ++u) ld_node(r.g2 + col[u], gP[u], gx[u]);
#pragma unroll
            for (int u = 0; u < kUL; ++u) {
                const uint32_t slot = base + (uint32_t)kStride * (q0 + u);
                c[u] = ldcs_f64(a.scoef + slot);
                coln[u] = ldcs_u32(a.scol + slot + (uint32_t)kStride * kUL);  // in bounds: padding
                if (PH == 3) {
                    i2[u] = ldcs_f64x2(r.I2 + slot);
                    i3[u] = ldcs_f64x2(r.I3 + slot);
                } else {
                    i2[u] = make_double2(0.0, 0.0);  // I^{(0)} = 0 at launch 2
                    i3[u] = make_double2(0.0, 0.0);
                }
            }
            double m2p[kUL], m2m[kUL], ip[kUL], im[kUL], pe[kUL], rc[kUL];
#pragma unroll
            for (int u = 0; u < kUL; ++u) {
                const bool v = q0 + u < d;
                if (!v) c[u] = 1.0;
                rc[u] = EXACT ? 0.0 : ddiv_rcp(c[u]);
                m2p[u] = 0.0;  // m^{(0)} = 0 at launch 2
                m2m[u] = 0.0;
                if (PH == 3) {  // own outgoing message of sweep s-2
                    const double pe2 = v ? a3.x - i3[u].x : 1.0;
                    const double nu2 = v ? a3.y - i3[u].x * i3[u].y : 1.0;
                    edge_msg<EXACT>(c[u], rc[u], pe2, nu2, m2p[u], m2m[u], st);
                }
            }
#pragma unroll
            for (int u = 0; u < kUL; ++u) {  // incoming of S_{s-1}
                const bool v = q0 + u < d;
                pe[u] = v ? gP[u] - m2p[u] : 1.0;
                const double num = v ? gP[u] * gx[u] - m2p[u] * m2m[u] : 1.0;  // (sum_p * mu_tilde)
                edge_msg<EXACT>(c[u], rc[u], pe[u], num, ip[u], im[u], st);
            }
#pragma unroll
            for (int u = 0; u < kUL; ++u) {
                const uint32_t q = q0 + u;
                if (q < d) {
                    sp = sp + ip[u];
                    sn = sn + ip[u] * im[u];  // (prec * mean), solver.py:243
                    if (PH == 3) y = y + c[u] * gx[u];
                    __stcs(r.I1 + base + (uint32_t)kStride * q, make_double2(ip[u], im[u]));
                    msg_stats<EXACT>(st, a, ip[u], im[u], i2[u], pe[u], p, q);
                }
            }
        }
        if (nd.x != 0.0) node_done<PH, EXACT>(st, a, r.g1, xh, p, sp, sn, y, rhs_i);
    }
}

// ---- variant 1: cp.async ring (short rows) -----------------------------------------------
// Each warp walks the flat item sequence (slice, batch of kUP edge columns) of its slices.
// Everything an item reads is brought in by cp.async, each lane copying its own elements
// (lane-interleaved, conflict-free; a lane only reads what it copied, so completion is the
// per-thread cp.async.wait_group): at iteration k a lane issues, as one commit group,
//   item k+D: scoef, I^{(s-2)}, I^{(s-3)}, the neighbour state {P, N} and x (addresses from
//             scol, already resident), and on a slice's first item the row header
//             (A_ii, prior numerator, degree, own state of S_{s-3} / x^{(s-2)}, b_i)
//   item k+2D: scol into its own (D+1)-entry ring
// then waits for the group of iteration k-D and computes item k from shared memory only.
// DRAM and L2 latency are covered by D items of every resident warp.
#ifndef GABP_SLICE_UP
#define GABP_SLICE_UP 2
#endif
#ifndef GABP_SLICE_DEPTH
#define GABP_SLICE_DEPTH 2
#endif
constexpr int kUP = GABP_SLICE_UP;
constexpr int kDepth = GABP_SLICE_DEPTH;
constexpr int kStages = kDepth + 1;
constexpr int kPThreads = 128;
constexpr int kPWarps = kPThreads / 32;

struct __align__(16) WarpStage {
    double2 i2[kUP][32];
    double2 i3[kUP][32];
    double2 ag[kUP][32];
    double2 nd[32];
    double2 a3[32];
    double c[kUP][32];
    double xg[kUP][32];
    double xo[32];
    double rhs[32];
    uint32_t deg[32];
};
struct __align__(16) WarpRing {
    WarpStage st[kStages];
    uint32_t col[kStages][kUP][32];
};
constexpr size_t kPipeSmem = sizeof(WarpRing) * kPWarps;

__device__ __forceinline__ uint32_t su32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cpa4(void *d, const void *g, bool p) {
    asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q cp.async.ca.shared.global [%0], [%1], 4;\n}\n"
                 ::"r"(su32(d)), "l"(g), "r"((int)p) : "memory");
}
__device__ __forceinline__ void cpa8(void *d, const void *g, bool p) {
    asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q cp.async.ca.shared.global [%0], [%1], 8;\n}\n"
                 ::"r"(su32(d)), "l"(g), "r"((int)p) : "memory");
}
__device__ __forceinline__ void cpa16(void *d, const void *g, bool p) {
    asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q cp.async.cg.shared.global [%0], [%1], 16;\n}\n"
                 ::"r"(su32(d)), "l"(g), "r"((int)p) : "memory");
}
__device__ __forceinline__ void cpa16ca(void *d, const void *g, bool p) {
    asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q cp.async.ca.shared.global [%0], [%1], 16;\n}\n"
                 ::"r"(su32(d)), "l"(g), "r"((int)p) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// position in a warp's item sequence; {base, width} of the warp's next two slices are
// loaded ahead so crossing into a slice never waits on its descriptor
struct Cursor {
    int64_t sl;           // slice (>= nslices: past the end)
    uint32_t b, nb;       // batch within the slice, batches of the slice (>= 1)
    uint32_t base, w;     // slot base and width of the slice
    uint2 next, next2;    // {base, width} of slices sl + nwarps, sl + 2 nwarps
};

__device__ __forceinline__ uint2 slice_at(const SweepArgs &a, int64_t sl) {
    return sl < a.nslices ? __ldg(a.slice_info + sl) : make_uint2(0u, 0u);
}
__device__ __forceinline__ void cursor_enter(Cursor &c, uint2 si) {
    c.b = 0;
    c.base = si.x;
    c.w = si.y;
    c.nb = si.y > 0 ? (si.y + kUP - 1) / kUP : 1u;
}
__device__ __forceinline__ void cursor_init(Cursor &c, const SweepArgs &a, int64_t sl,
                                            int64_t nwarps) {
    c.sl = sl;
    cursor_enter(c, slice_at(a, sl));
    c.next = slice_at(a, sl + nwarps);
    c.next2 = slice_at(a, sl + 2 * nwarps);
}
__device__ __forceinline__ void cursor_next(Cursor &c, const SweepArgs &a, int64_t nwarps) {
    if (c.b + 1 < c.nb) {
        ++c.b;
    } else {
        c.sl += nwarps;
        cursor_enter(c, c.next);
        c.next = c.next2;
        c.next2 = slice_at(a, c.sl + 2 * nwarps);
    }
}

template <int PH, int R>
__device__ __forceinline__ void issue_item(WarpStage &S, const uint32_t (&col)[kUP][32],
                                           const Cursor &c, const SweepArgs &a,
                                           const Ring<R> &r, int lane) {
    if (c.sl >= a.nslices) return;
    if (c.b == 0) {
        const int64_t p = c.sl * 32 + lane;
        cpa16(&S.nd[lane], a.snd + p, true);
        cpa4(&S.deg[lane], a.sdeg + p, true);
        if (PH == 3) {
            cpa16(&S.a3[lane], r.g3 + p, true);
            cpa8(&S.xo[lane], &r.g2[p].x, true);
            cpa8(&S.rhs[lane], a.srhs + p, true);
        }
    }
#pragma unroll
    for (int u = 0; u < kUP; ++u) {
        const uint32_t q = c.b * kUP + u;
        const bool v = q < c.w;
        const uint32_t slot = c.base + lane + (uint32_t)kStride * q;
        const uint32_t j = col[u][lane];
        cpa8(&S.c[u][lane], a.scoef + slot, v);
        cpa16(&S.ag[u][lane], r.g2 + j, v);
        if (PH == 3) {
            cpa16(&S.i2[u][lane], r.I2 + slot, v);
            cpa16(&S.i3[u][lane], r.I3 + slot, v);
            cpa8(&S.xg[u][lane], &r.g2[j].x, v);
        }
    }
}

__device__ __forceinline__ void issue_col(uint32_t (&col)[kUP][32], const Cursor &c,
                                          const SweepArgs &a, int lane) {
    if (c.sl >= a.nslices) return;
#pragma unroll
    for (int u = 0; u < kUP; ++u) {
        const uint32_t q = c.b * kUP + u;
        cpa4(&col[u][lane], a.scol + c.base + lane + (uint32_t)kStride * q, q < c.w);
    }
}

template <int PH, int R, bool EXACT>
__device__ __forceinline__ void slice_sweep_pipe(const SweepArgs &a, int64_t s, Stats &st,
                                                 int lane, WarpRing &ring) {
    const Ring<R> r(a);
    double *xh = xhist_row(a, s);
    const int64_t nwarps = (int64_t)gridDim.x * kPWarps;
    const int64_t first = (int64_t)blockIdx.x * kPWarps + (threadIdx.x >> 5);
    Cursor C, P, Q;  // items k (compute), k + D (stage), k + 2D (scol)
    cursor_init(C, a, first, nwarps);
    P = C;
    Q = C;
    // prologue: scol of items 0 .. D-1; then items 0 .. D-1 with scol of D .. 2D-1
#pragma unroll
    for (int k = 0; k < kDepth; ++k) {
        issue_col(ring.col[k], Q, a, lane);
        cursor_next(Q, a, nwarps);
    }
    cpa_commit();
    cpa_wait<0>();
#pragma unroll
    for (int k = 0; k < kDepth; ++k) {
        issue_item<PH, R>(ring.st[k], ring.col[k], P, a, r, lane);
        cursor_next(P, a, nwarps);
        issue_col(ring.col[(k + kDepth) % kStages], Q, a, lane);
        cursor_next(Q, a, nwarps);
        cpa_commit();
    }

    uint32_t d = 0;
    double2 a3 = make_double2(0.0, 0.0);
    double sp = 0.0, sn = 0.0, y = 0.0, rhs_i = 0.0, diag = 0.0;
    for (uint32_t k = 0; C.sl < a.nslices; ++k) {
        cpa_wait<kDepth - 1>();  // item k and scol of item k+D landed
        const uint32_t sk = k % kStages, sd = (k + kDepth) % kStages;
        issue_item<PH, R>(ring.st[sd], ring.col[sd], P, a, r, lane);
        cursor_next(P, a, nwarps);
        issue_col(ring.col[(k + 2 * kDepth) % kStages], Q, a, lane);
        cursor_next(Q, a, nwarps);
        cpa_commit();

        const WarpStage &S = ring.st[sk];
        if (C.b == 0) {  // row header
            d = S.deg[lane];
            const double2 nd = S.nd[lane];
            diag = nd.x;
            sp = nd.x;
            sn = nd.y;
            if (PH == 3) {
                a3 = S.a3[lane];  // {P_i, x_i}
                a3.y = a3.x * a3.y;
                y = nd.x * S.xo[lane];
                rhs_i = S.rhs[lane];
            }
        }
        double c[kUP], m2p[kUP], m2m[kUP], ip[kUP], im[kUP], pe[kUP], rc[kUP];
#pragma unroll
        for (int u = 0; u < kUP; ++u) {
            const bool v = C.b * kUP + u < d;
            c[u] = v ? S.c[u][lane] : 1.0;
            rc[u] = ddiv_rcp(c[u]);
            m2p[u] = 0.0;  // m^{(0)} = 0 at launch 2
            m2m[u] = 0.0;
            if (PH == 3) {  // own outgoing message of sweep s-2
                const double2 i3 = S.i3[u][lane];
                const double pe2 = v ? a3.x - i3.x : 1.0;
                const double nu2 = v ? a3.y - i3.x * i3.y : 1.0;
                edge_msg<EXACT>(c[u], rc[u], pe2, nu2, m2p[u], m2m[u], st);
            }
        }
#pragma unroll
        for (int u = 0; u < kUP; ++u) {  // incoming of S_{s-1}
            const bool v = C.b * kUP + u < d;
            const double2 ag = S.ag[u][lane];  // {P_j, x_j}
            pe[u] = v ? ag.x - m2p[u] : 1.0;
            const double num = v ? ag.x * ag.y - m2p[u] * m2m[u] : 1.0;
            edge_msg<EXACT>(c[u], rc[u], pe[u], num, ip[u], im[u], st);
        }
        const int64_t p = C.sl * 32 + lane;
#pragma unroll
        for (int u = 0; u < kUP; ++u) {
            const uint32_t q = C.b * kUP + u;
            if (q < d) {
                sp = sp + ip[u];
                sn = sn + ip[u] * im[u];  // (prec * mean), solver.py:243
                if (PH == 3) y = y + c[u] * S.xg[u][lane];
                __stcs(r.I1 + C.base + lane + (uint32_t)kStride * q, make_double2(ip[u], im[u]));
                const double2 i2 = PH == 3 ? S.i2[u][lane] : make_double2(0.0, 0.0);
                msg_stats<EXACT>(st, a, ip[u], im[u], i2, pe[u], p, q);
            }
        }
        if (C.b + 1 == C.nb && diag != 0.0)  // row done (A_ii == 0: padding lane)
            node_done<PH, EXACT>(st, a, r.g1, xh, p, sp, sn, y, rhs_i);
        cursor_next(C, a, nwarps);
    }
    cpa_wait<0>();  // nothing may land in the ring after the warp leaves
}

// ---- variant 2: CTA-lockstep TMA ring over slice groups (default) ----------------------
// A CTA owns one slice group (kGroup slices, column q of the group = kStride contiguous
// slots, see the layout note at the top) at a time: consumer warp w runs slice w of the
// group, lane per row, and all consumers walk the group's columns together in chunks of
// kGC columns.  One producer warp claims groups dynamically (Ctrl.work, claims and
// descriptor loads kept two groups ahead), and for every chunk issues one 1-D bulk copy
// (TMA, cp.async.bulk) per slot stream -- scoef, scol, I^{(s-2)}, I^{(s-3)}, kGC x kStride
// slots each -- into a kGS-stage shared-memory ring: full[stage] completes on the copies'
// byte count, empty[stage] on the kGroup consumers' releases.  So the DRAM stream stays in
// flight independently of the compute, and a chunk costs a consumer one barrier wait and
// one release.  Only the neighbour gathers (L2-resident node states) and the 32-row header
// are register loads, issued one chunk ahead of use.
#ifndef GABP_GRP_C
#define GABP_GRP_C 2
#endif
#ifndef GABP_GRP_NS
#define GABP_GRP_NS 4
#endif
constexpr int kGC = GABP_GRP_C;   // edge columns per chunk
constexpr int kGS = GABP_GRP_NS;  // ring stages
constexpr int kGThreads = 32 * (kGroup + 1);
static_assert(kGS >= 2, "the ring needs two stages");

struct __align__(128) GStage {
    double2 i2[kGC][kStride];  // I^{(s-2)} (statistics)
    double2 i3[kGC][kStride];  // I^{(s-3)} (own message rebuild)
    double c[kGC][kStride];
    uint32_t col[kGC][kStride];
};
struct __align__(16) GMeta {
    int32_t g;            // group (< 0: end of the launch's work)
    uint32_t b, nb;       // chunk within the group, chunks of the group (>= 1)
    uint32_t w;           // group width (columns)
    uint32_t gbase;       // first slot of the group
    uint32_t pad[3];
};
constexpr int kGResSlots = kGS + 4;  // groups a CTA's consumers can be apart (< kGS + 2)
static_assert(kGResSlots >= kGS + 2, "residual slots must outlast the ring's lag");
struct __align__(128) GRing {
    GStage st[kGS];
    uint64_t full[kGS];
    uint64_t empty[kGS];
    GMeta meta[kGS];
#ifndef GABP_R1_GRP
    double gres[kGResSlots][kGroup];  // slice partials of a group's residual rows
    uint32_t gcnt[kGResSlots];        // slices committed
#endif
};

// Residual of group g (the seq-th group this CTA ran): every consumer warp sums its slice's
// rows (fixed shuffle tree) and the last of the kGroup warps adds the slice partials in
// slice order into rsq_grp[g].  The launch total is then a sum in group order: the same
// bits whichever CTA claimed which group (the claims are dynamic).
__device__ __forceinline__ void grp_resid_commit(const SweepArgs &a, GRing &G, int warp,
                                                 int lane, int64_t g, uint32_t seq, double rr) {
#if defined(GABP_NO_RESID_COMMIT) || defined(GABP_R1_GRP)
    return;
#else
    rr = warp_sum(rr);
    const int k = (int)(seq % kGResSlots);
    unsigned last = 0u;
    if (lane == 0) {
        G.gres[k][warp] = rr;
        __threadfence_block();
        last = atomicAdd(&G.gcnt[k], 1u) == (unsigned)kGroup - 1u ? 1u : 0u;
        if (last) {
            __threadfence_block();
            volatile const double *v = G.gres[k];
            double b = 0.0;
#pragma unroll
            for (int w = 0; w < kGroup; ++w) b += v[w];
            a.rsq_grp[g] = b;
            G.gcnt[k] = 0u;
        }
    }
#endif
}
constexpr size_t kGrpSmem = sizeof(GRing);

__device__ __forceinline__ void t_mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(bar)), "r"(count));
}
__device__ __forceinline__ void t_expect_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void t_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void t_wait(uint64_t *bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "TW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        " @!p bra TW_%=;\n}\n" ::"r"(su32(bar)),
        "r"(parity), "r"(0x989680u)
        : "memory");
}
// streamed once per sweep: evict-first, so the gathered node states keep the L2
__device__ __forceinline__ void t_bulk_ef(void *dst, const void *src, unsigned bytes,
                                          uint64_t *bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;\n" ::"r"(su32(dst)),
        "l"(src), "r"(bytes), "r"(su32(bar)), "l"(pol)
        : "memory");
}

__device__ __forceinline__ void grp_ring_init(GRing &G, int tid) {
    if (tid < kGS) {
        t_mbar_init(&G.full[tid], 1u);
        t_mbar_init(&G.empty[tid], (unsigned)kGroup);
    }
#ifndef GABP_R1_GRP
    if (tid < kGResSlots) G.gcnt[tid] = 0u;
#endif
}

__device__ __forceinline__ uint2 group_info(const SweepArgs &a, int64_t g, int64_t g_hi) {
    return g < g_hi ? __ldg(a.slice_info + g * kGroup) : make_uint2(0u, 0u);
}
// group of claim c (c counts from the launch's first group): the claim order lists the
// widest groups first (gorder), so the last claims of a launch are its shortest units;
// g_hi (no group) once the claims run out
__device__ __forceinline__ int64_t claim_group(const SweepArgs &a, int64_t c, int64_t g_hi) {
    if (c >= g_hi) return g_hi;
    return a.gorder ? (int64_t)__ldg(a.gorder + c) : c;
}
template <int CW = kGC>
__device__ __forceinline__ uint32_t chunks_of(uint32_t w) {
    return w > 0 ? (w + CW - 1) / CW : 1u;
}

// Launch kinds of the group kernel (PH): 3 a full launch (scoef, scol, I^{(s-2)}, I^{(s-3)}:
// 44 B per slot); 4 launch 3, whose I^{(s-3)} = I^{(0)} is +0 (no stream: 28 B); 2 launch 2,
// whose m^{(0)} = 0 (scoef, scol: 12 B); 5 a residual-only launch (12 B).  The 12-byte kinds
// lay a stage out as NStage, kNC2 / kNCR columns per chunk instead of kGC: the same bytes
// per ring trip, so the ring keeps as much DRAM traffic in flight as a full launch does.
template <int CW>
struct NStage {
    double c[CW][kStride];
    uint32_t col[CW][kStride];
};
#ifndef GABP_NC2
#define GABP_NC2 3
#endif
constexpr int kNC2 = GABP_NC2;  // launch 2: gathers {P, N} and the edge divisions in registers
#ifndef GABP_NCR
#define GABP_NCR 6
#endif
constexpr int kNCR = GABP_NCR;  // residual-only launch
static_assert(sizeof(NStage<kNCR>) <= sizeof(GStage) && sizeof(NStage<kNC2>) <= sizeof(GStage),
              "a narrow stage must fit a ring stage");
template <int PH>
constexpr int stage_cw() {
    return PH == 2 ? kNC2 : PH == 5 ? kNCR : kGC;
}
template <int PH>
constexpr unsigned stage_bytes() {
    return PH == 3 ? 44u : PH == 4 ? 28u : 12u;
}
template <int PH>
__device__ __forceinline__ const double *st_c(const GStage &S, int u) {
    if constexpr (PH == 2 || PH == 5)
        return reinterpret_cast<const NStage<stage_cw<PH>()> &>(S).c[u];
    else
        return S.c[u];
}
template <int PH>
__device__ __forceinline__ const uint32_t *st_col(const GStage &S, int u) {
    if constexpr (PH == 2 || PH == 5)
        return reinterpret_cast<const NStage<stage_cw<PH>()> &>(S).col[u];
    else
        return S.col[u];
}

// Producer warp: claims groups and fills the ring until the claims run out.
template <int PH, int R>
__device__ __forceinline__ void grp_produce(const SweepArgs &a, GRing &G, uint32_t *ctr,
                                            int lane) {
    const Ring<R> r(a);
    const int64_t g_lo = a.sl_lo / kGroup, ngroups = a.sl_hi / kGroup;  // claims from g_lo
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    uint32_t u0 = 0, u1 = 0, pend = 0;
    if (lane == 0) {
        u0 = atomicAdd(ctr, 1u);
        u1 = atomicAdd(ctr, 1u);
        pend = atomicAdd(ctr, 1u);
    }
    int64_t gcur = claim_group(a, g_lo + __shfl_sync(~0u, u0, 0), ngroups),
            gnxt = claim_group(a, g_lo + __shfl_sync(~0u, u1, 0), ngroups);
    uint2 icur = group_info(a, gcur, ngroups), inxt = group_info(a, gnxt, ngroups);
    constexpr int CW = stage_cw<PH>();
    uint32_t b = 0, nb = chunks_of<CW>(icur.y);
    for (uint32_t k = 0;; ++k) {
        const int stg = (int)(k % kGS);
        if (k >= (uint32_t)kGS) t_wait(&G.empty[stg], ((k / kGS) - 1u) & 1u);
        if (gcur >= ngroups) {  // no more work: wake the consumers with an end marker
            if (lane == 0) {
                G.meta[stg].g = -1;
                t_arrive(&G.full[stg]);
            }
            return;
        }
        if (lane == 0) {
            const uint32_t w = icur.y, q0 = b * CW;
            const uint32_t nc = w > q0 ? min((uint32_t)CW, w - q0) : 0u;
            const uint32_t slot = icur.x + (uint32_t)kStride * q0;
            GMeta &m = G.meta[stg];
            m.g = (int32_t)gcur;
            m.b = b;
            m.nb = nb;
            m.w = w;
            m.gbase = icur.x;
            // (0 bytes: a group of isolated rows; the arrive alone completes the phase)
            t_expect_tx(&G.full[stg], nc * (uint32_t)kStride * stage_bytes<PH>());
            if (nc) {
                if constexpr (PH == 2 || PH == 5) {
                    NStage<CW> &N = reinterpret_cast<NStage<CW> &>(G.st[stg]);
                    t_bulk_ef(&N.c[0][0], a.scoef + slot, nc * kStride * 8u, &G.full[stg], pol);
                    t_bulk_ef(&N.col[0][0], a.scol + slot, nc * kStride * 4u, &G.full[stg], pol);
                } else {
                    GStage &S = G.st[stg];
                    t_bulk_ef(&S.c[0][0], a.scoef + slot, nc * kStride * 8u, &G.full[stg], pol);
                    t_bulk_ef(&S.col[0][0], a.scol + slot, nc * kStride * 4u, &G.full[stg], pol);
                    t_bulk_ef(&S.i2[0][0], r.I2 + slot, nc * kStride * 16u, &G.full[stg], pol);
                    if (PH == 3)
                        t_bulk_ef(&S.i3[0][0], r.I3 + slot, nc * kStride * 16u, &G.full[stg],
                                  pol);
                }
            }
        }
        if (++b >= nb) {  // next group: claimed two groups ago, descriptor loaded one ago
            gcur = gnxt;
            icur = inxt;
            gnxt = claim_group(a, g_lo + __shfl_sync(~0u, pend, 0), ngroups);
            inxt = group_info(a, gnxt, ngroups);
            if (lane == 0) pend = atomicAdd(ctr, 1u);
            b = 0;
            nb = chunks_of<CW>(icur.y);
        }
    }
}

// Own-row header of a slice (lane = row): prior, degree, and the own node states of
// S_{s-3} (message rebuild) and S_{s-2} (x_i of the residual row), register loads issued
// one chunk ahead of use like the gathers.
struct THdr {
    double2 nd;   // {A_ii, prior numerator}
    double2 a3;   // {P_i, x_i} of S_{s-3}
    double xo;    // x_i^{(s-2)}
    double rhs;
    uint32_t d;
};
template <int PH, int R>
__device__ __forceinline__ void t_header(const SweepArgs &a, const Ring<R> &r, int64_t p,
                                         THdr &h) {
#if GABP_GATHER_POLICY >= 2  // read once per launch: no L1 allocation, demoted in L2
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(h.nd.x), "=d"(h.nd.y) : "l"(a.snd + p), "l"(pol_evict_first_node()));
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
                 : "=r"(h.d) : "l"(a.sdeg + p), "l"(pol_evict_first_node()));
#else
    h.nd = __ldg(a.snd + p);
    h.d = __ldg(a.sdeg + p);
#endif
    if (PH == 3 || PH == 4) {
#if GABP_GATHER_POLICY >= 1
        // S_{s-3}: last use of the state (demoted); S_{s-2}: still gathered this launch
        h.a3 = ld_f64x2_pol(reinterpret_cast<const double2 *>(r.g3 + p), pol_evict_first_node());
#else
        h.a3 = __ldcg(reinterpret_cast<const double2 *>(r.g3 + p));
#endif
        h.xo = __ldcg(&r.g2[p].x);
#if GABP_GATHER_POLICY >= 2
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
                     : "=d"(h.rhs) : "l"(a.srhs + p), "l"(pol_evict_first_node()));
#else
        h.rhs = __ldg(a.srhs + p);
#endif
    }
}

// neighbour gathers of a landed chunk (node states of S_{s-2}), one chunk ahead of use
template <int PH, int CW = stage_cw<PH>()>
__device__ __forceinline__ void t_gather(const GStage &S, const GMeta &m, const NodeState *g2,
                                         int t, double (&gP)[CW], double (&gx)[CW]) {
#pragma unroll
    for (int u = 0; u < CW; ++u) {
        if (m.b * CW + u < m.w) {
#if GABP_GATHER_POLICY >= 1
            ld_node_pol(g2 + st_col<PH>(S, u)[t], gP[u], gx[u], pol_evict_last_node());
#else
            ld_node(g2 + st_col<PH>(S, u)[t], gP[u], gx[u]);
#endif
        } else {
            gP[u] = 1.0;
            gx[u] = 0.0;
        }
    }
}

// Stage data a consumer reads from shared memory and uses only after releasing the stage
// must have ARRIVED in registers before the release: the mbarrier arrive does not wait for
// the lane's outstanding shared loads, and the producer's next bulk copy may overwrite the
// stage while one is still in flight (seen as a rare wrong change statistic -- the old
// message I^{(s-2)} is the one operand used after the release).  An empty asm that takes
// the values as inputs makes the lane wait on their scoreboard first.
// (the token is an integer fold of the values' bits, fed to the arrive as an operand: the
// folding instructions read the loaded registers, so they wait for the loads, and the arrive
// cannot issue before them)
__device__ __forceinline__ uint32_t hold(uint32_t tok, double v) {
    return tok ^ (uint32_t)__double2hiint(v) ^ (uint32_t)__double2loint(v);
}
__device__ __forceinline__ uint32_t hold(uint32_t tok, double2 v) {
    return hold(hold(tok, v.x), v.y);
}
__device__ __forceinline__ void t_arrive_after(uint64_t *bar, uint32_t tok) {
    asm volatile(
        "{\n .reg .b32 t;\n mov.b32 t, %1;\n"
        " mbarrier.arrive.shared::cta.b64 _, [%0];\n}\n" ::"r"(su32(bar)),
        "r"(tok)
        : "memory");
}

// Running sums of the rows a consumer lane owns (one row per group).
struct GRow {
    uint32_t d = 0, seq = 0;
    double2 a3 = make_double2(0.0, 0.0);
    double sp = 0.0, sn = 0.0, y = 0.0, rhs_i = 0.0, diag = 0.0;
};

// Chunk k of a consumer warp: waits for chunk k+1 and issues its header and gathers into
// (nP, nx), then computes chunk k from its stage and the gathers (gP, gx).  Returns
// false after the last chunk; otherwise m becomes chunk k+1's descriptor.  The loop calls
// it with the two gather buffers swapped on alternate chunks (no register copies).
template <int PH, int R, int CW = stage_cw<PH>()>
__device__ __forceinline__ bool grp_step(const SweepArgs &a, const Ring<R> &r, double *xh,
                                         Stats &st, GRing &G, int lane, int warp, int t,
                                         uint32_t k, GMeta &m, THdr &hn, GRow &row,
                                         const double (&gP)[CW], const double (&gx)[CW],
                                         double (&nP)[CW], double (&nx)[CW]) {
    if (m.b == 0) {  // row header (loaded one chunk ago)
        row.d = hn.d;
        row.diag = hn.nd.x;
        row.sp = hn.nd.x;
        row.sn = hn.nd.y;
        if (PH == 3 || PH == 4) {
            row.a3 = make_double2(hn.a3.x, hn.a3.x * hn.a3.y);  // {P_i, (sum_p * mu_tilde)}
            row.y = hn.nd.x * hn.xo;
            row.rhs_i = hn.rhs;
        }
    }
    // header and gathers of chunk k+1
    const int s1 = (int)((k + 1) % kGS);
    t_wait(&G.full[s1], ((k + 1) / kGS) & 1u);
    const GMeta mn = G.meta[s1];
    if (mn.g >= 0) {
        if (mn.b == 0) t_header<PH, R>(a, r, ((int64_t)mn.g * kGroup + warp) * 32 + lane, hn);
        t_gather<PH>(G.st[s1], mn, r.g2, t, nP, nx);
    }
    const int s0 = (int)(k % kGS);
    const GStage &S = G.st[s0];
    const uint32_t d = row.d;
    double cc[CW], m2p[CW], m2m[CW], ip[CW], im[CW], pe[CW], rc[CW];
    double2 i2v[CW];
#pragma unroll
    for (int u = 0; u < CW; ++u) {
        const bool v = m.b * CW + u < d;
        cc[u] = v ? st_c<PH>(S, u)[t] : 1.0;
        rc[u] = ddiv_rcp(cc[u]);
        m2p[u] = 0.0;  // m^{(0)} = 0 at launch 2
        m2m[u] = 0.0;
        i2v[u] = make_double2(0.0, 0.0);
        if (PH == 3 || PH == 4) {  // own outgoing message of sweep s-2
            // (launch 3: I^{(0)} = +0, not streamed; x - (+0) == x bit for bit)
            const double2 i3 = PH == 3 ? S.i3[u][t] : make_double2(0.0, 0.0);
            i2v[u] = S.i2[u][t];
            const double pe2 = v ? row.a3.x - i3.x : 1.0;
            const double nu2 = v ? row.a3.y - i3.x * i3.y : 1.0;
            edge_msg<false>(cc[u], rc[u], pe2, nu2, m2p[u], m2m[u], st);
        }
    }
#ifndef GABP_LATE_RELEASE
    uint32_t tok = 0u;
#pragma unroll
    for (int u = 0; u < CW; ++u) tok = hold(tok, i2v[u]);  // (used after the release)
    tok = __reduce_or_sync(~0u, tok);  // every lane's loads landed
    if (lane == 0) t_arrive_after(&G.empty[s0], tok);  // the stage's data is in registers now
#endif
#pragma unroll
    for (int u = 0; u < CW; ++u) {  // incoming of S_{s-1}
        const bool v = m.b * CW + u < d;
        pe[u] = v ? gP[u] - m2p[u] : 1.0;
        const double num = v ? gP[u] * gx[u] - m2p[u] * m2m[u] : 1.0;  // (sum_p * mu_tilde)
        edge_msg<false>(cc[u], rc[u], pe[u], num, ip[u], im[u], st);
    }
    const int64_t p = ((int64_t)m.g * kGroup + warp) * 32 + lane;
#pragma unroll
    for (int u = 0; u < CW; ++u) {
        const uint32_t q = m.b * CW + u;
        if (q < d) {
            row.sp = row.sp + ip[u];
            row.sn = row.sn + ip[u] * im[u];  // (prec * mean), solver.py:243
            if (PH == 3 || PH == 4) row.y = row.y + cc[u] * gx[u];
            __stcs(r.I1 + m.gbase + (uint32_t)kStride * q + t, make_double2(ip[u], im[u]));
            msg_stats<false>(st, a, ip[u], im[u], i2v[u], pe[u], p, q);
        }
    }
#ifdef GABP_LATE_RELEASE
    {  // release after the last use of the stage (no operand outlives it in registers)
        uint32_t tok = 0u;
#pragma unroll
        for (int u = 0; u < CW; ++u) tok = hold(tok, i2v[u]);
        tok = __reduce_or_sync(~0u, tok);
        if (lane == 0) t_arrive_after(&G.empty[s0], tok);
    }
#endif
#if defined(GABP_R1_GRP) || defined(GABP_R1_ROWDONE)
    if (m.b + 1 == m.nb && row.diag != 0.0)  // row done (A_ii == 0: padding lane)
        node_done<(PH == 4 ? 3 : PH), false>(st, a, r.g1, xh, p, row.sp, row.sn, row.y, row.rhs_i);
    if (false) {
#else
    if (m.b + 1 == m.nb) {  // rows done (A_ii == 0: padding lane)
#endif
        double rr = 0.0;
        if (row.diag != 0.0)
            rr = node_done<(PH == 4 ? 3 : PH), false, false>(st, a, r.g1, xh, p, row.sp, row.sn,
                                                             row.y, row.rhs_i);
        if (PH == 3 || PH == 4) grp_resid_commit(a, G, warp, lane, m.g, row.seq, rr);
        row.seq++;
    }
    if (mn.g < 0) return false;
    m = mn;
    return true;
}

// Consumer warp `warp`: slice warp of every group, lane per row.
template <int PH, int R>
__device__ __forceinline__ void grp_consume(const SweepArgs &a, int64_t s, Stats &st, int lane,
                                            int warp, GRing &G) {
    const Ring<R> r(a);
    double *xh = xhist_row(a, s);
    const int t = warp * 32 + lane;  // index within a group column
    t_wait(&G.full[0], 0u);
    GMeta m = G.meta[0];
    if (m.g < 0) return;
    constexpr int CW = stage_cw<PH>();
    double gA[2][CW], gB[2][CW];  // gathers {P, x}: chunk k in one, k+1 in the other
    THdr hn;
    t_header<PH, R>(a, r, ((int64_t)m.g * kGroup + warp) * 32 + lane, hn);
    t_gather<PH>(G.st[0], m, r.g2, t, gA[0], gA[1]);
    GRow row;
    for (uint32_t k = 0;; k += 2) {
        if (!grp_step<PH, R>(a, r, xh, st, G, lane, warp, t, k, m, hn, row, gA[0], gA[1], gB[0],
                             gB[1]))
            break;
        if (!grp_step<PH, R>(a, r, xh, st, G, lane, warp, t, k + 1, m, hn, row, gB[0], gB[1],
                             gA[0], gA[1]))
            break;
    }
}

// Residual-only group launch (the probe on the TMA ring): the producer streams scoef and
// scol (12 B per slot, kNCR columns per stage); consumers gather x^{(s-2)} and form the
// residual rows of x^{(s-2)} exactly as a full launch s would (grp_step, PH 3).  The pass is
// bound by the gathers' L2 latency, so a consumer copies a landed stage's coefficients into
// registers, issues its gathers and releases the stage at once, keeping kRD chunks of
// gathers in flight.
constexpr int kRD = 3;  // chunks of gathers in flight per consumer
template <int R>
__device__ __forceinline__ void grp_consume_res(const SweepArgs &a, Stats &st, int lane,
                                                int warp, GRing &G) {
    constexpr int CW = kNCR;
    const Ring<R> r(a);
    const int t = warp * 32 + lane;
    double cv[kRD][CW], xv[kRD][CW];
    GMeta mq[kRD];
    // chunk k: wait for its stage, take coefficients and gathers, release the stage
    auto issue = [&](uint32_t k, int slot) -> bool {
        const int sg = (int)(k % kGS);
        t_wait(&G.full[sg], (k / kGS) & 1u);
        const GMeta m = G.meta[sg];
        mq[slot] = m;
        if (m.g < 0) return false;
        const GStage &S = G.st[sg];
#pragma unroll
        for (int u = 0; u < CW; ++u) {
            const bool v = m.b * CW + u < m.w;
            const uint32_t j = st_col<5>(S, u)[t];
            cv[slot][u] = st_c<5>(S, u)[t];
            xv[slot][u] = v ? __ldcg(&r.g2[j].x) : 0.0;
        }
        uint32_t tok = 0u;
#pragma unroll
        for (int u = 0; u < CW; ++u) tok = hold(tok, cv[slot][u]);  // (used after the release)
        tok = __reduce_or_sync(~0u, tok);
        if (lane == 0) t_arrive_after(&G.empty[sg], tok);
        return true;
    };
    // chunks are issued strictly in order and never past the end marker (the producer
    // fills no stage after it): `more` is the liveness of the last chunk issued
    bool live[kRD], more = true;
#pragma unroll
    for (int q = 0; q < kRD; ++q) {
        if (more) more = issue(q, q);
        live[q] = more;
    }
    if (!live[0]) return;
    uint32_t d = 0, seq = 0;
    double y = 0.0, rhs_i = 0.0, diag = 0.0;
    for (uint32_t k = 0;; k += kRD) {
#pragma unroll
        for (int q = 0; q < kRD; ++q) {
            if (!live[q]) return;
            const GMeta m = mq[q];
            if (m.b == 0) {  // row header
                const int64_t p = ((int64_t)m.g * kGroup + warp) * 32 + lane;
                const double2 nd = __ldg(a.snd + p);
                d = __ldg(a.sdeg + p);
                diag = nd.x;
                y = nd.x * __ldcg(&r.g2[p].x);
                rhs_i = __ldg(a.srhs + p);
            }
#pragma unroll
            for (int u = 0; u < CW; ++u)
                if (m.b * CW + u < d) y = y + cv[q][u] * xv[q][u];
            if (m.b + 1 == m.nb) {
                const double rr = diag != 0.0 ? y - rhs_i : 0.0;
                grp_resid_commit(a, G, warp, lane, m.g, seq++, rr * rr);
            }
            if (more) more = issue(k + kRD + q, q);
            live[q] = more;
        }
    }
}

template <int R>
__device__ __forceinline__ void slice_res_grp(const SweepArgs &a, Stats &st, int lane, int warp,
                                              GRing &G, uint32_t *ctr) {
    if (warp == kGroup)
        grp_produce<5, R>(a, G, ctr, lane);
    else
        grp_consume_res<R>(a, st, lane, warp, G);
}

template <int PH, int R>
__device__ __forceinline__ void slice_sweep_grp(const SweepArgs &a, int64_t s, Stats &st,
                                                int lane, int warp, GRing &G, uint32_t *ctr) {
    if (warp == kGroup)
        grp_produce<PH, R>(a, G, ctr, lane);
    else
        grp_consume<PH, R>(a, s, st, lane, warp, G);
}

// ---- kernels ---------------------------------------------------------------------------------
template <class SM>
__device__ __forceinline__ bool slice_prologue(SM &S, const SweepArgs &a, bool exact) {
    if (threadIdx.x == 0) {
        volatile Ctrl *vc = a.ctrl;
        const int64_t s = vc->next_sweep;
        const bool twin = exact && !a.exact_primary;
        if (twin && blockIdx.x == 0) atomicAdd(&a.ctrl->twin_launches, 1);
        S.skip = vc->done || s > vc->max_iter + 2 || (twin && vc->redo != 2);
        // the residual probe the last launch asked for (probe_next): run by an idle exact
        // twin (a.probe == 1) or as a residual-only group launch (a.probe == 2)
        const bool mine = twin ? (a.probe == 1 && vc->redo != 2) : (!exact && a.probe == 2);
        S.probe = mine && !vc->done && vc->probe_t != 0 && vc->probe_t == s - 2;
        S.sweep = s;
    }
    __syncthreads();
    return !S.skip;
}

// ---- residual probe ----------------------------------------------------------------------
// Run by the exact twin after launch T+1 when that launch's decision step expects sweep T
// to end the solve (probe_next, gabp_internal.cuh): the residual of x^{(T)} in one pass over
// scol / scoef (12 B per slot) with gathers of x^{(T)}, then the decision for T -- so launch
// T+2, which would otherwise compute it next to a whole discarded sweep T+1, exits at once.
// Per row the sweep kernels' sum (A_ii x_i, then + A_ij x_j in ascending j); rows summed per
// warp, CTA partials in CTA order.  Batches of kRU columns: all slot loads, then all
// gathers, then the sums (memory-level parallelism of a latency-bound pass).
constexpr int kRU = 16;

// Residual of x^{(t)} summed over the CTAs (partials in CTA order), then the decision for
// t.  work_slot >= 0: a residual-only group launch, which leaves next_sweep alone (the next
// launch runs the same sweep when t was not the last) and re-arms its claim counter.
template <int NT>
__device__ __forceinline__ void probe_finish(TailSmem<NT / 32> &T, const SweepArgs &a,
                                             int64_t t, double rsq, int work_slot) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    rsq = warp_sum(rsq);
    if (lane == 0) T.red_d[0][warp] = rsq;
    __syncthreads();
    if (tid == 0) {
        double b = 0.0;
        for (int w = 0; w < NT / 32; ++w) b += T.red_d[0][w];
        a.rsq_part[blockIdx.x] = b;
        __threadfence();
        T.last = atomicAdd(&a.ctrl->ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!T.last) return;
    __threadfence();
    double part = 0.0;
    volatile const double *rp = a.rsq_part;
    for (int64_t b = tid; b < (int64_t)gridDim.x; b += NT) part += rp[b];
    if (work_slot >= 0) part += group_resid_part<NT>(a, tid);  // (group launch)
    part = warp_sum(part);
    __syncthreads();
    if (lane == 0) T.red_d[0][warp] = part;
    __syncthreads();
    if (tid == 0) {
        double rsq_t = 0.0;
        for (int w = 0; w < NT / 32; ++w) rsq_t += T.red_d[0][w];
        volatile Ctrl *c = a.ctrl;
        decide_sweep(c, a, t, rsq_t);
        if (work_slot >= 0) c->work[work_slot] = 0u;
        c->ticket = 0u;
        c->probe_t = 0;
        c->probes = c->probes + 1;
        __threadfence();
    }
}

template <int NT>
__device__ __noinline__ void probe_residual(TailSmem<NT / 32> &T, const SweepArgs &a, int64_t t) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const NodeState *xr = a.rec[t % 3];
    const int64_t nw = (int64_t)gridDim.x * (NT / 32);
    double rsq = 0.0;
    for (int64_t sl = (int64_t)blockIdx.x * (NT / 32) + warp; sl < a.nslices; sl += nw) {
        const int64_t p = sl * 32 + lane;
        const uint2 si = __ldg(a.slice_info + sl);
        const double2 nd = __ldg(a.snd + p);
        const uint32_t d = __ldg(a.sdeg + p);
        double y = nd.x * __ldcg(&xr[p].x);
        for (uint32_t q0 = 0; q0 < si.y; q0 += kRU) {  // (si.y: the group width, warp-uniform)
            const uint32_t slot = si.x + (uint32_t)kStride * q0 + (uint32_t)lane;
            uint32_t cj[kRU];
            double cv[kRU], xv[kRU];
#pragma unroll
            for (int u = 0; u < kRU; ++u) {
                cj[u] = 0u;
                cv[u] = 0.0;
                if (q0 + u < si.y) {
                    cj[u] = __ldcs(a.scol + slot + (uint32_t)kStride * u);
                    cv[u] = __ldcs(a.scoef + slot + (uint32_t)kStride * u);
                }
            }
#pragma unroll
            for (int u = 0; u < kRU; ++u) xv[u] = q0 + u < si.y ? __ldcg(&xr[cj[u]].x) : 0.0;
#pragma unroll
            for (int u = 0; u < kRU; ++u)
                if (q0 + u < d) y = y + cv[u] * xv[u];
        }
        if (nd.x != 0.0) {  // (A_ii == 0: padding lane)
            const double r = y - __ldg(a.srhs + p);
            rsq += r * r;
        }
    }
    probe_finish<NT>(T, a, t, rsq, -1);
}
template <bool EXACT>
__global__ void __launch_bounds__(kLThreads, 2) slice_kernel_ldg(const SweepArgs a) {
    __shared__ SliceSmem S;
    if (!slice_prologue(S, a, EXACT)) {
        if (EXACT && S.probe)
            probe_residual<kLThreads>(*reinterpret_cast<TailSmem<kLWarps> *>(&S.tail), a,
                                      S.sweep - 2);
        return;
    }
    const int64_t s = S.sweep;
    const int tid = threadIdx.x, lane = tid & 31;
    Stats st;
    st.lim = fmin(a.ctrl->blowup, DBL_MAX);
    if (s >= 3) {
        const int r = (int)(s % 3);
        if (r == 0)
            slice_sweep_ldg<3, 0, EXACT>(a, s, st, lane);
        else if (r == 1)
            slice_sweep_ldg<3, 1, EXACT>(a, s, st, lane);
        else
            slice_sweep_ldg<3, 2, EXACT>(a, s, st, lane);
    } else if (s == 2) {
        slice_sweep_ldg<2, 2, EXACT>(a, s, st, lane);
    } else {
        slice_first<kLWarps, EXACT>(a, s, st, lane);
    }
    sweep_epilogue<kLThreads, kModeSolve, 1>(*reinterpret_cast<TailSmem<kLWarps> *>(&S.tail), a,
                                              s, s >= 3, st, tid);
}

__global__ void __launch_bounds__(kPThreads, 3) slice_kernel_pipe(const SweepArgs a) {
    __shared__ SliceSmem S;
    extern __shared__ __align__(16) unsigned char pipe_raw[];
    WarpRing &ring = reinterpret_cast<WarpRing *>(pipe_raw)[threadIdx.x >> 5];
    if (!slice_prologue(S, a, false)) return;
    const int64_t s = S.sweep;
    const int tid = threadIdx.x, lane = tid & 31;
    Stats st;
    st.lim = fmin(a.ctrl->blowup, DBL_MAX);
    if (s >= 3) {
        const int r = (int)(s % 3);
        if (r == 0)
            slice_sweep_pipe<3, 0, false>(a, s, st, lane, ring);
        else if (r == 1)
            slice_sweep_pipe<3, 1, false>(a, s, st, lane, ring);
        else
            slice_sweep_pipe<3, 2, false>(a, s, st, lane, ring);
    } else if (s == 2) {
        slice_sweep_pipe<2, 2, false>(a, s, st, lane, ring);
    } else {
        slice_first<kPWarps, false>(a, s, st, lane);
    }
    sweep_epilogue<kPThreads, kModeSolve, 1>(*reinterpret_cast<TailSmem<kPWarps> *>(&S.tail), a,
                                              s, s >= 3, st, tid);
}

struct GrpSmem {
    TailSmem<kGroup + 1> tail;
    int64_t sweep;
    int skip;
    int probe;
};

__global__ void __launch_bounds__(kGThreads, 1) slice_kernel_grp(const SweepArgs a) {
    __shared__ GrpSmem S;
    extern __shared__ __align__(128) unsigned char grp_raw[];
    GRing &G = *reinterpret_cast<GRing *>(grp_raw);
    if (!slice_prologue(S, a, false)) return;
    const int64_t s = S.sweep;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    grp_ring_init(G, tid);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    __syncthreads();
    uint32_t *ctr = &a.ctrl->work[s % kStatSlots];
    Stats st;
    st.lim = fmin(a.ctrl->blowup, DBL_MAX);
    if (S.probe) {  // residual-only launch: decide sweep s-2 without computing sweep s-1
        const int r = (int)(s % 3);
        if (r == 0)
            slice_res_grp<0>(a, st, lane, warp, G, ctr);
        else if (r == 1)
            slice_res_grp<1>(a, st, lane, warp, G, ctr);
        else
            slice_res_grp<2>(a, st, lane, warp, G, ctr);
        probe_finish<kGThreads>(S.tail, a, s - 2, st.rsq, (int)(s % kStatSlots));
        return;
    }
    if (s >= 4) {
        const int r = (int)(s % 3);
        if (r == 0)
            slice_sweep_grp<3, 0>(a, s, st, lane, warp, G, ctr);
        else if (r == 1)
            slice_sweep_grp<3, 1>(a, s, st, lane, warp, G, ctr);
        else
            slice_sweep_grp<3, 2>(a, s, st, lane, warp, G, ctr);
    } else if (s == 3) {
        slice_sweep_grp<4, 0>(a, s, st, lane, warp, G, ctr);
    } else if (s == 2) {
        slice_sweep_grp<2, 2>(a, s, st, lane, warp, G, ctr);
    } else {
        slice_first<kGroup + 1, false>(a, s, st, lane);
    }
    const bool flagged =
        sweep_epilogue<kGThreads, kModeSolve, 1, true>(S.tail, a, s, s >= 3, st, tid);
    if (flagged && a.twin_tail) {
        // a fast-path division left its range: the exact twin redoes this sweep, launched
        // from here into the tail of this grid (CUDA dynamic parallelism) -- it runs after
        // this grid and before the next launch of the stream, and only when needed (a
        // host-launched twin that exits at once cost 16 us of every config-1 sweep)
        SweepArgs t = a;
        t.sl_lo = 0;
        t.sl_hi = a.nslices;
        t.part_base = 0;
        t.exact_primary = 0;
        t.twin_tail = 0;
        slice_kernel_ldg<true><<<(unsigned)a.twin_grid, kLThreads, 0, cudaStreamTailLaunch>>>(t);
    }
}

// ---- parallel schedule over the slice groups ------------------------------------------------
// _sweep_parallel (solver.py:146-173): every directed edge i -> j gets its exclusion sums
//   P_excl = A_ii + sum_{k != j} P_ki,  N_excl = A_ii mu_ii + sum_{k != j} P_ki mu_ki
// in ascending k (np.add.at over excl_pos), then m_ij = (-A_ij^2 / P_excl, N_excl / A_ij).
// Storage is the incoming layout of the broadcast slice path: slot (i, q) holds
// I_iq = m_{k_q -> i}.  Launch s reads row i's incoming messages of S_{s-1} -- contiguous
// slots, streamed by the group producer -- and writes its outgoing messages of S_s into
// the twin slots (stwin, scattered 16-byte stores).  The exclusion sums are O(degree^2):
// the outgoing edges of a row are taken kPB at a time (register accumulators), one pass
// over the row's incoming columns per block -- pass 0 from DRAM with everything else
// (I^{(s-2)} for the change statistic, coefficients and columns for the residual), later
// passes re-read only I^{(s-1)}, which stays in L2 (a group's columns are 16 B x 480 per
// column).  Pass 0 also forms the full sums: marginal x^{(s-1)} and the residual row of
// x^{(s-2)}, as the broadcast kernel.  Statistics of sweep s-1 (LAG 1): every message is
// exactly one row's incoming slot.
#ifndef GABP_PAR_BLOCK
#define GABP_PAR_BLOCK 8
#endif
constexpr int kPB = GABP_PAR_BLOCK;  // outgoing edges per exclusion pass
static_assert(kPB % kGC == 0, "a block starts on a chunk boundary");

__device__ __forceinline__ uint32_t par_passes(uint32_t w) {
    return w > kPB ? (w + kPB - 1) / kPB : 1u;
}

// Producer of the parallel kernel: per group, np passes; pass 0 streams every column in
// chunks of kGC (all streams), pass p >= 1 streams I^{(s-1)} alone from column p kPB in
// chunks of kPC columns (a stage holds kPC x kStride messages: as many bytes per ring trip
// as a pass-0 chunk).  Descriptor: b = first column of the chunk, nb = 1 on the last chunk
// of a pass, pad = {pass, passes, columns in the chunk}.
#ifndef GABP_PAR_PC
#define GABP_PAR_PC 5
#endif
constexpr int kPC = GABP_PAR_PC;
struct PStage {
    double2 i[kPC][kStride];
};
static_assert(sizeof(PStage) <= sizeof(GStage), "a later-pass chunk must fit a ring stage");

template <bool STATS, bool RESID, bool EXACT>
__device__ __forceinline__ void par_produce(const SweepArgs &a, GRing &G, uint32_t *ctr,
                                            const double2 *I1, const double2 *I2, int lane) {
    const int64_t g_lo = a.sl_lo / kGroup, ngroups = a.sl_hi / kGroup;
    uint64_t pol_ef, pol_el;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_ef));
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_el));
    uint32_t u0 = 0, u1 = 0, pend = 0;
    if (lane == 0) {
        u0 = atomicAdd(ctr, 1u);
        u1 = atomicAdd(ctr, 1u);
        pend = atomicAdd(ctr, 1u);
    }
    int64_t gcur = claim_group(a, g_lo + __shfl_sync(~0u, u0, 0), ngroups),
            gnxt = claim_group(a, g_lo + __shfl_sync(~0u, u1, 0), ngroups);
    uint2 icur = group_info(a, gcur, ngroups), inxt = group_info(a, gnxt, ngroups);
    uint32_t q0 = 0, pass = 0, np = par_passes(icur.y);
    for (uint32_t k = 0;; ++k) {
        const int stg = (int)(k % kGS);
        if (k >= (uint32_t)kGS) t_wait(&G.empty[stg], ((k / kGS) - 1u) & 1u);
        if (gcur >= ngroups) {
            if (lane == 0) {
                G.meta[stg].g = -1;
                t_arrive(&G.full[stg]);
            }
            return;
        }
        const uint32_t w = icur.y, cw = pass == 0 ? (uint32_t)kGC : (uint32_t)kPC;
        const uint32_t nc = w > q0 ? min(cw, w - q0) : 0u;
        const bool last = q0 + cw >= w;
        if (lane == 0) {
            const uint32_t slot = icur.x + (uint32_t)kStride * q0;
            GMeta &m = G.meta[stg];
            m.g = (int32_t)gcur;
            m.b = q0;
            m.nb = last ? 1u : 0u;
            m.w = w;
            m.gbase = icur.x;
            m.pad[0] = pass;
            m.pad[1] = np;
            m.pad[2] = nc;
            const unsigned per = pass == 0 ? 16u + (STATS ? 16u : 0u) + (RESID ? 12u : 0u) : 16u;
            t_expect_tx(&G.full[stg], nc * (uint32_t)kStride * per);
            if (nc) {
                // I^{(s-1)} is re-read by the later passes: keep it in L2 while they run
                const uint64_t pol = np > 1 && pass + 1 < np ? pol_el : pol_ef;
                if (pass == 0) {
                    GStage &S = G.st[stg];
                    t_bulk_ef(&S.i3[0][0], I1 + slot, nc * kStride * 16u, &G.full[stg], pol);
                    if (STATS)
                        t_bulk_ef(&S.i2[0][0], I2 + slot, nc * kStride * 16u, &G.full[stg], pol_ef);
                    if (RESID) {
                        t_bulk_ef(&S.c[0][0], a.scoef + slot, nc * kStride * 8u, &G.full[stg],
                                  pol_ef);
                        t_bulk_ef(&S.col[0][0], a.scol + slot, nc * kStride * 4u, &G.full[stg],
                                  pol_ef);
                    }
                } else {
                    PStage &P = reinterpret_cast<PStage &>(G.st[stg]);
                    t_bulk_ef(&P.i[0][0], I1 + slot, nc * kStride * 16u, &G.full[stg], pol);
                }
            }
        }
        if (last) {
            if (++pass >= np) {
                pass = 0;
                gcur = gnxt;
                icur = inxt;
                gnxt = claim_group(a, g_lo + __shfl_sync(~0u, pend, 0), ngroups);
                inxt = group_info(a, gnxt, ngroups);
                if (lane == 0) pend = atomicAdd(ctr, 1u);
                np = par_passes(icur.y);
            }
            q0 = pass * kPB;
        } else {
            q0 += cw;
        }
    }
}

struct ParRow {
    uint32_t d = 0;
    double pP = 0.0, pN = 0.0;             // prior precision and numerator
    double sp = 0.0, sn = 0.0, y = 0.0, rhs_i = 0.0;
    double preP = 0.0, preN = 0.0;         // prefix sums up to the current block's first edge
    double aP[kPB], aN[kPB];               // exclusion sums of the current block
    double cb[kPB];                        // A_ij of the block's edges
    uint32_t tw[kPB];                      // their twin slots
};

// One incoming term of column q into the block's exclusion sums (and the next block's
// prefix while q is one of the block's own columns); q is warp-uniform.  Pass p >= 1
// starts at column p kPB: the exclusion sums of edges p kPB .. p kPB + kPB - 1 share the
// sequential prefix A_ii + sum_{q < p kPB} P_qi (no edge of the block is excluded from it),
// carried over from pass p-1 -- the same operations in the same order as summing from
// column 0, and half the column visits of a full re-walk per block.
__device__ __forceinline__ void par_accum(ParRow &row, uint32_t q, uint32_t blk, double vP,
                                          double vN) {
    if (q < blk + kPB) {
        row.preP = row.preP + vP;
        row.preN = row.preN + vN;
#pragma unroll
        for (int jj = 0; jj < kPB; ++jj)
            if (q != blk + jj) {
                row.aP[jj] = row.aP[jj] + vP;
                row.aN[jj] = row.aN[jj] + vN;
            }
    } else {
#pragma unroll
        for (int jj = 0; jj < kPB; ++jj) {
            row.aP[jj] = row.aP[jj] + vP;
            row.aN[jj] = row.aN[jj] + vN;
        }
    }
}

// Consumer of the parallel kernel (warp `warp`, lane per row).
template <bool STATS, bool RESID, bool EXACT>
__device__ __forceinline__ void par_consume(const SweepArgs &a, int64_t s, Stats &st, int lane,
                                            int warp, GRing &G, const NodeState *g2,
                                            NodeState *g1, double2 *I0) {
    double *xh = xhist_row(a, s);
    const int t = warp * 32 + lane;
    t_wait(&G.full[0], 0u);
    GMeta m = G.meta[0];
    if (m.g < 0) return;
    ParRow row;
    THdr hn;
    uint32_t seq = 0;  // groups this CTA ran (residual slots)
    const int64_t p_first = ((int64_t)m.g * kGroup + warp) * 32 + lane;
    hn.nd = __ldg(a.snd + p_first);
    hn.d = __ldg(a.sdeg + p_first);
    if (RESID) {
        hn.xo = __ldcg(&g2[p_first].x);
        hn.rhs = __ldg(a.srhs + p_first);
    }
    double gx[kGC] = {}, nx[kGC] = {};
    if (RESID) {  // residual gathers of chunk 0 (x_j^{(s-2)})
#pragma unroll
        for (int u = 0; u < kGC; ++u)
            if (u < (int)m.w) gx[u] = __ldcg(&g2[G.st[0].col[u][t]].x);
    }
    for (uint32_t k = 0;; ++k) {
        const uint32_t pass = m.pad[0];
        const uint32_t blk = pass * kPB;  // first edge of the block (warp-uniform)
        const int64_t p = ((int64_t)m.g * kGroup + warp) * 32 + lane;
        const uint32_t slot0 = m.gbase + (uint32_t)t;
        if (m.b == blk) {  // first chunk of the pass
            if (pass == 0) {  // row header (loaded one chunk ago)
                row.d = hn.d;
                row.pP = hn.nd.x;
                row.pN = hn.nd.y;
                row.sp = hn.nd.x;
                row.sn = hn.nd.y;
                row.preP = hn.nd.x;
                row.preN = hn.nd.y;
                if (RESID) {
                    row.y = hn.nd.x * hn.xo;
                    row.rhs_i = hn.rhs;
                }
            }
#pragma unroll
            for (int jj = 0; jj < kPB; ++jj) {  // block `pass`: sums start at its prefix
                row.aP[jj] = row.preP;
                row.aN[jj] = row.preN;
            }
        }
        // last chunk of the pass: the block's coefficients and twin slots (loading them on
        // the pass's first chunk instead, held across the pass, measured 2 % slower)
        if (m.nb) {
#pragma unroll
            for (int jj = 0; jj < kPB; ++jj) {
                const uint32_t j = blk + jj;
                row.cb[jj] = 1.0;
                row.tw[jj] = 0u;
                if (j < row.d) {
                    row.cb[jj] = __ldg(a.scoef + slot0 + (uint32_t)kStride * j);
                    row.tw[jj] = __ldg(a.stwin + slot0 + (uint32_t)kStride * j);
                }
            }
        }
        // next chunk: header and residual gathers
        const int s1 = (int)((k + 1) % kGS);
        t_wait(&G.full[s1], ((k + 1) / kGS) & 1u);
        const GMeta mn = G.meta[s1];
        if (mn.g >= 0) {
            if (mn.b == 0 && mn.pad[0] == 0) {  // (pass 0 of a group starts at column 0)
                const int64_t pn = ((int64_t)mn.g * kGroup + warp) * 32 + lane;
                hn.nd = __ldg(a.snd + pn);
                hn.d = __ldg(a.sdeg + pn);
                if (RESID) {
                    hn.xo = __ldcg(&g2[pn].x);
                    hn.rhs = __ldg(a.srhs + pn);
                }
            }
            if (RESID && mn.pad[0] == 0) {
#pragma unroll
                for (int u = 0; u < kGC; ++u)
                    if (mn.b + u < mn.w) nx[u] = __ldcg(&g2[G.st[s1].col[u][t]].x);
            }
        }
        const int s0 = (int)(k % kGS);
        const uint32_t d = row.d;
        if (pass == 0) {
            const GStage &S = G.st[s0];
#pragma unroll
            for (int u = 0; u < kGC; ++u) {
                const uint32_t q = m.b + u;
                if (q < d) {
                    const double2 v = S.i3[u][t];  // I^{(s-1)}_iq = m_{k_q -> i}
                    const double vP = v.x, vN = v.x * v.y;  // (prec * mean), solver.py:148
                    row.sp = row.sp + vP;
                    row.sn = row.sn + vN;
                    if (RESID) row.y = row.y + S.c[u][t] * gx[u];
                    if (STATS) {
                        const double2 o = S.i2[u][t];
                        const double d1 = fabs(v.x - o.x), d2 = fabs(v.y - o.y);
                        st.chg = fmax(st.chg, fmax(d1, d2));
                        if (!(fabs(v.x) <= st.lim) || !(fabs(v.y) <= st.lim))
                            st.out_of_range |= (v.x != v.x || v.y != v.y) ? 3u : 1u;
                    }
                    par_accum(row, q, blk, vP, vN);
                }
            }
        } else {
            const PStage &P = reinterpret_cast<const PStage &>(G.st[s0]);
#pragma unroll
            for (int u = 0; u < kPC; ++u) {
                const uint32_t q = m.b + u;
                if (q < d) {
                    const double2 v = P.i[u][t];
                    par_accum(row, q, blk, v.x, v.x * v.y);
                }
            }
        }
        __syncwarp();
        if (lane == 0) t_arrive(&G.empty[s0]);
        if (m.nb) {  // end of pass: the block's messages, scattered to the twins
#pragma unroll
            for (int jj = 0; jj < kPB; ++jj) {
                const uint32_t j = blk + jj;
                if (j < d) {
                    const double c = row.cb[jj];
                    const double rc = EXACT ? 0.0 : ddiv_rcp(c);
                    double P, mu;
                    edge_msg<EXACT>(c, rc, row.aP[jj], row.aN[jj], P, mu, st);
                    __stcg(I0 + row.tw[jj], make_double2(P, mu));
                    // P_excl(i -> j) = 0 (solver.py:150-154): sweep s itself, so the slot of
                    // the launch's own sweep (agg_sing), not the lagged message slot
                    if (EXACT && row.aP[jj] == 0.0)
                        st.agg_sing = min(st.agg_sing, a.row_ptr[__ldg(a.srow + p)] + j);
                }
            }
            if (pass == 0) {  // marginal of S_{s-1}, residual of x^{(s-2)}
                double rr = 0.0;
                if (row.pP != 0.0) {
                    const double xi = qdiv<EXACT>(row.sn, row.sp, st);
                    if (!(fabs(xi) <= DBL_MAX)) st.means_bad = 1u;
                    if (xh) xh[__ldg(a.srow + p)] = xi;
                    st_node(g1 + p, row.sp, xi);
                    if (RESID) {
                        const double r = row.y - row.rhs_i;
                        rr = r * r;
                    }
                }
                if (RESID) grp_resid_commit(a, G, warp, lane, m.g, seq, rr);
                seq++;
            }
        }
        if (mn.g < 0) break;
        m = mn;
#pragma unroll
        for (int u = 0; u < kGC; ++u) gx[u] = nx[u];
    }
}

template <bool EXACT>
__global__ void __launch_bounds__(kGThreads, 1) slice_kernel_par(const SweepArgs a) {
    __shared__ GrpSmem S;
    extern __shared__ __align__(128) unsigned char par_raw[];
    GRing &G = *reinterpret_cast<GRing *>(par_raw);
    if (!slice_prologue(S, a, EXACT)) {
        if (EXACT && S.probe) probe_residual<kGThreads>(S.tail, a, S.sweep - 2);
        return;
    }
    const int64_t s = S.sweep;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    grp_ring_init(G, tid);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    __syncthreads();
    uint32_t *ctr = EXACT ? &a.ctrl->work_twin : &a.ctrl->work[s % kStatSlots];
    const double2 *I1 = a.msg[(s + 2) % 3];  // I^{(s-1)}
    const double2 *I2 = a.msg[(s + 1) % 3];  // I^{(s-2)}
    double2 *I0 = a.msg[s % 3];              // I^{(s)}, written
    const NodeState *g2 = a.rec[(s + 1) % 3];
    NodeState *g1 = a.rec[(s + 2) % 3];
    Stats st;
    st.lim = fmin(a.ctrl->blowup, DBL_MAX);
    if (warp == kGroup) {
        if (s >= 3)
            par_produce<true, true, EXACT>(a, G, ctr, I1, I2, lane);
        else if (s == 2)
            par_produce<true, false, EXACT>(a, G, ctr, I1, I2, lane);
        else
            par_produce<false, false, EXACT>(a, G, ctr, I1, I2, lane);
    } else {
        if (s >= 3)
            par_consume<true, true, EXACT>(a, s, st, lane, warp, G, g2, g1, I0);
        else if (s == 2)
            par_consume<true, false, EXACT>(a, s, st, lane, warp, G, g2, g1, I0);
        else
            par_consume<false, false, EXACT>(a, s, st, lane, warp, G, g2, g1, I0);
    }
    sweep_epilogue<kGThreads, kModeSolve, 1, true>(S.tail, a, s, s >= 3, st, tid);
}

int g_grid_ldg = 0, g_grid_pipe = 0, g_grid_grp = 0, g_grid_par = 0;

// ---- build -------------------------------------------------------------------------------
constexpr int kSortWin = kStride * 2048;  // rows per degree-sort window (whole groups)
static_assert(kSlotPad >= kStride * (kUL + 1), "slot padding must cover a register batch");

// Sort key of a swept row: window id above 13 bits of (8191 - degree), so one ascending
// stable radix sort orders every window by degree, descending (degrees <= 4096).
constexpr int kDegBits = 13;
static_assert(kSliceMaxDegree < (1 << kDegBits), "degree must fit the key");
// A rank's rows with a halo neighbour (a neighbour outside [row_lo, row_hi)) are
// *boundary* rows: with split != 0 they sort before every interior row (top key bit), so
// the first groups hold exactly the rows whose new states the peers need (DESIGN.md
// "Multi-GPU"); *nbnd counts them.
__global__ void slice_key_kernel(int64_t row_lo, int64_t m, const uint32_t *row_ptr,
                                 const EdgeRec *er, int split, uint32_t *key, uint32_t *rows,
                                 unsigned long long *nbnd) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= m) return;
    const int64_t i = row_lo + r;
    const uint32_t d = row_ptr[i + 1] - row_ptr[i];
    uint32_t interior = 0u;
    if (split) {
        interior = 1u;
        for (uint32_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
            const int64_t j = er[e].col;
            if (j < row_lo || j >= row_lo + m) {
                interior = 0u;
                break;
            }
        }
        if (!interior) atomicAdd(nbnd, 1ull);
    }
    key[r] = (interior << 31) | ((uint32_t)(r / kSortWin) << kDegBits) |
             ((1u << kDegBits) - 1u - d);
    rows[r] = (uint32_t)i;
}

__global__ void key_to_deg_kernel(int64_t m, uint32_t *k) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < m) k[r] = (1u << kDegBits) - 1u - (k[r] & ((1u << kDegBits) - 1u));
}

// slots of each group: kStride x its largest degree (degrees are sorted descending inside
// windows of whole groups, so that is the degree of its first row)
__global__ void group_width_kernel(int64_t ngroups, int64_t m, const uint32_t *sdeg,
                                   unsigned long long *gslots) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= ngroups) return;
    uint32_t w = 0;
    for (int64_t p = g * kStride; p < (g + 1) * kStride && p < m; ++p)
        if (sdeg[p] > w) w = sdeg[p];
    gslots[g] = (unsigned long long)kStride * w;
}

// {slot base, width} of every slice: base_s = gbase_g + 32 (s % kGroup)
__global__ void slice_info_kernel(int64_t nslices, const unsigned long long *gslots,
                                  const unsigned long long *gbase, uint2 *info) {
    const int64_t sl = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (sl >= nslices) return;
    const int64_t g = sl / kGroup;
    info[sl] = make_uint2((uint32_t)(gbase[g] + 32 * (sl % kGroup)),
                          (uint32_t)(gslots[g] / kStride));
}

// claim-order key of every group: boundary groups first (split sweeps claim them in a
// launch of their own), then by width, descending -- the degree sort runs inside windows of
// kSortWin rows, so the last window would otherwise start over with wide groups and leave
// the launch a tail of its longest work units
__global__ void gorder_key_kernel(int64_t ngroups, int64_t bnd_groups, const uint2 *info,
                                  uint32_t *key, uint32_t *ids) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= ngroups) return;
    const uint32_t w = info[g * kGroup].y;
    key[g] = ((g < bnd_groups ? 0u : 1u) << kDegBits) | ((1u << kDegBits) - 1u - w);
    ids[g] = (uint32_t)g;
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
        const uint32_t slot = si.x + (uint32_t)kStride * q + l;
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
        snd[p] = make_double2(0.0, 0.0);  // A_ii == 0 marks a padding lane
        srhs[p] = 0.0;
    }
}

__global__ void gather_pos_kernel(int64_t lo, int64_t cnt, const uint32_t *pos, const double *in,
                                  int stride, double *out) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < cnt) out[lo + k] = in[(int64_t)pos[lo + k] * stride];
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
    const int64_t ngroups = (m + kStride - 1) / kStride;
    const int64_t nslices = ngroups * kGroup;  // padding slices complete the last group
    const int64_t m_pad = nslices * 32;
    const int64_t npos = m_pad + (g.n - m);
    const int64_t nseg = (m + kSortWin - 1) / kSortWin;
    uint32_t *deg = nullptr, *rows = nullptr, *sorted_deg = nullptr, *sorted_rows = nullptr;
    unsigned long long *gslots = nullptr, *gbase = nullptr;
    SCHECK(cudaMallocAsync(&deg, sizeof(uint32_t) * m, st));
    SCHECK(cudaMallocAsync(&rows, sizeof(uint32_t) * m, st));
    SCHECK(cudaMallocAsync(&sorted_deg, sizeof(uint32_t) * m, st));
    SCHECK(cudaMallocAsync(&sorted_rows, sizeof(uint32_t) * m, st));
    SCHECK(cudaMallocAsync(&gslots, sizeof(unsigned long long) * (ngroups + 1), st));
    SCHECK(cudaMallocAsync(&gbase, sizeof(unsigned long long) * (ngroups + 1), st));
    // multi-rank row block: boundary rows first (their groups run before the exchange)
    const int split = (g.row_lo > 0 || g.row_hi < g.n) ? 1 : 0;
    unsigned long long *d_nbnd = gslots;  // (scratch until the group widths)
    SCHECK(cudaMemsetAsync(d_nbnd, 0, sizeof(unsigned long long), st));
    slice_key_kernel<<<grid_of(m), 256, 0, st>>>(g.row_lo, m, g.row_ptr, g.er, split, deg, rows,
                                                 d_nbnd);
    SCHECK(cudaGetLastError());
    unsigned long long nbnd = 0;
    SCHECK(cudaMemcpyAsync(&nbnd, d_nbnd, sizeof(nbnd), cudaMemcpyDeviceToHost, st));
    // stable: rows of equal degree keep their order (structured grids stay contiguous)
    int end_bit = kDegBits;
    while (end_bit < 31 && ((nseg - 1) >> (end_bit - kDegBits)) > 0) ++end_bit;
    if (split) end_bit = 32;
    static_assert(kSortWin >= (1 << 16), "window ids must fit below the boundary bit");
    size_t tb = 0;
    SCHECK(cub::DeviceRadixSort::SortPairs(nullptr, tb, deg, sorted_deg, rows, sorted_rows, m,
                                           0, end_bit, st));
    void *tmp = nullptr;
    SCHECK(cudaMallocAsync(&tmp, tb, st));
    SCHECK(cub::DeviceRadixSort::SortPairs(tmp, tb, deg, sorted_deg, rows, sorted_rows, m, 0,
                                           end_bit, st));
    cudaFreeAsync(tmp, st);
    key_to_deg_kernel<<<grid_of(m), 256, 0, st>>>(m, sorted_deg);
    group_width_kernel<<<grid_of(ngroups), 256, 0, st>>>(ngroups, m, sorted_deg, gslots);
    SCHECK(cudaMemsetAsync(gslots + ngroups, 0, sizeof(unsigned long long), st));
    size_t sb = 0;
    SCHECK(cub::DeviceScan::ExclusiveSum(nullptr, sb, gslots, gbase, ngroups + 1, st));
    SCHECK(cudaMallocAsync(&tmp, sb, st));
    SCHECK(cub::DeviceScan::ExclusiveSum(tmp, sb, gslots, gbase, ngroups + 1, st));
    cudaFreeAsync(tmp, st);
    unsigned long long nslots = 0;
    SCHECK(cudaMemcpyAsync(&nslots, gbase + ngroups, sizeof(nslots), cudaMemcpyDeviceToHost, st));
    SCHECK(cudaStreamSynchronize(st));
    int rc = GABP_OK;
    if (nslots + kSlotPad >= 0xffffffffull) {
        rc = GABP_EINVAL;  // caller keeps the tile layout only
        snprintf(err, errlen, "slice layout needs %llu slots (> 32-bit)", nslots);
    } else if (nslots > 2ull * (unsigned long long)g.E + (1ull << 20)) {
        // a skewed degree distribution pads groups to their widest row: more than twice
        // the edges in slots would stream mostly padding -- the CSR tiles have none
        rc = GABP_EINVAL;
        snprintf(err, errlen, "slice layout would pad %lld edges to %llu slots",
                 (long long)g.E, nslots);
    } else {
        g.nslices = nslices;
        g.nslots = (int64_t)nslots;
        g.npos = npos;
        g.bnd_groups = split ? (int64_t)((nbnd + kStride - 1) / kStride) : 0;
        SCHECK(cudaMallocAsync(&g.slice_info, sizeof(uint2) * nslices, st));
        SCHECK(cudaMallocAsync(&g.pos, sizeof(uint32_t) * (g.n > 0 ? g.n : 1), st));
        SCHECK(cudaMallocAsync(&g.srow, sizeof(uint32_t) * npos, st));
        SCHECK(cudaMallocAsync(&g.sdeg, sizeof(uint32_t) * npos, st));
        SCHECK(cudaMallocAsync(&g.snd, sizeof(double2) * npos, st));
        SCHECK(cudaMallocAsync(&g.srhs, sizeof(double) * npos, st));
        // + kSlotPad: the register-batch kernel loads whole batches past a group's width
        SCHECK(cudaMallocAsync(&g.scol, sizeof(uint32_t) * (nslots + kSlotPad), st));
        SCHECK(cudaMallocAsync(&g.scoef, sizeof(double) * (nslots + kSlotPad), st));
        SCHECK(cudaMemsetAsync(g.scol + nslots, 0, sizeof(uint32_t) * kSlotPad, st));
        SCHECK(cudaMemsetAsync(g.scoef + nslots, 0, sizeof(double) * kSlotPad, st));
        // kernel: the group TMA ring; GABP_SLICE_VARIANT=0/1 selects the register-batch /
        // cp.async kernels (kept as cross-checks, tests/test_gpu_parity.py)
        g.slice_variant = 2;
        if (const char *ev = getenv("GABP_SLICE_VARIANT")) g.slice_variant = atoi(ev);
        if (g.slice_variant < 0 || g.slice_variant > 2) g.slice_variant = 2;
        slice_info_kernel<<<grid_of(nslices), 256, 0, st>>>(nslices, gslots, gbase,
                                                            g.slice_info);
        {  // claim order: (boundary, interior) x width descending, stable
            uint32_t *gk = nullptr, *gk2 = nullptr, *gid = nullptr;
            SCHECK(cudaMallocAsync(&g.gorder, sizeof(uint32_t) * ngroups, st));
            SCHECK(cudaMallocAsync(&gk, sizeof(uint32_t) * ngroups, st));
            SCHECK(cudaMallocAsync(&gk2, sizeof(uint32_t) * ngroups, st));
            SCHECK(cudaMallocAsync(&gid, sizeof(uint32_t) * ngroups, st));
            gorder_key_kernel<<<grid_of(ngroups), 256, 0, st>>>(ngroups, g.bnd_groups,
                                                                g.slice_info, gk, gid);
            size_t ob = 0;
            SCHECK(cub::DeviceRadixSort::SortPairs(nullptr, ob, gk, gk2, gid, g.gorder,
                                                   ngroups, 0, kDegBits + 1, st));
            void *otmp = nullptr;
            SCHECK(cudaMallocAsync(&otmp, ob, st));
            SCHECK(cub::DeviceRadixSort::SortPairs(otmp, ob, gk, gk2, gid, g.gorder, ngroups,
                                                   0, kDegBits + 1, st));
            cudaFreeAsync(otmp, st);
            cudaFreeAsync(gk, st);
            cudaFreeAsync(gk2, st);
            cudaFreeAsync(gid, st);
        }
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
    cudaFreeAsync(gslots, st);
    cudaFreeAsync(gbase, st);
    SCHECK(cudaStreamSynchronize(st));
    return rc;
}

// slot of every swept CSR edge, then the twin slot of every slot (parallel schedule)
__global__ void eslot_kernel(int64_t npos_sw, const uint2 *info, const uint32_t *srow,
                             const uint32_t *sdeg, const uint32_t *row_ptr, uint32_t *eslot) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= npos_sw) return;
    const uint32_t d = sdeg[p];
    if (!d) return;
    const uint2 si = info[p >> 5];
    const uint32_t e0 = row_ptr[srow[p]], l = (uint32_t)(p & 31);
    for (uint32_t q = 0; q < d; ++q) eslot[e0 + q] = si.x + (uint32_t)kStride * q + l;
}
__global__ void stwin_kernel(int64_t npos_sw, const uint2 *info, const uint32_t *srow,
                             const uint32_t *sdeg, const uint32_t *row_ptr, const EdgeRec *er,
                             const uint32_t *eslot, uint32_t *stwin) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= npos_sw) return;
    const uint32_t d = sdeg[p];
    if (!d) return;
    const uint2 si = info[p >> 5];
    const uint32_t e0 = row_ptr[srow[p]], l = (uint32_t)(p & 31);
    for (uint32_t q = 0; q < d; ++q)
        stwin[si.x + (uint32_t)kStride * q + l] = eslot[er[e0 + q].rev];
}

// per-position copies of the node priors and rhs (after every prior computation)
cudaError_t refresh_slice_nodes(const DeviceGraph &g, cudaStream_t st) {
    if (g.nslices == 0) return cudaSuccess;
    slice_nodes_kernel<<<grid_of(g.npos), 256, 0, st>>>(g.npos, g.srow, g.nd, g.rhs, g.snd,
                                                        g.srhs);
    return cudaGetLastError();
}

// out[i] = in[stride * pos[i]] for local rows [lo, lo + cnt): position order -> row order
cudaError_t slice_to_rows(const DeviceGraph &g, int64_t lo, int64_t cnt, const double *in,
                          int stride, double *out, cudaStream_t st) {
    if (cnt <= 0) return cudaSuccess;
    gather_pos_kernel<<<grid_of(cnt), 256, 0, st>>>(lo, cnt, g.pos, in, stride, out);
    return cudaGetLastError();
}

// idx[k] = pos[idx[k]]: a rank's halo lists in position numbering
cudaError_t slice_map_index(const DeviceGraph &g, uint32_t *idx, int64_t cnt, cudaStream_t st) {
    if (cnt <= 0) return cudaSuccess;
    map_pos_kernel<<<grid_of(cnt), 256, 0, st>>>(cnt, g.pos, idx);
    return cudaGetLastError();
}

int build_stwin(DeviceGraph &g, cudaStream_t st, char *err, size_t errlen) {
    if (g.stwin || g.nslices == 0) return GABP_OK;

    if (g.row_lo != 0 || g.row_hi != g.n) {
        snprintf(err, errlen, "the parallel slice kernel runs on whole graphs only");
        return GABP_EINVAL;
    }
    uint32_t *eslot = nullptr;
    SCHECK(cudaMallocAsync(&eslot, sizeof(uint32_t) * (g.E > 0 ? g.E : 1), st));
    SCHECK(cudaMallocAsync(&g.stwin, sizeof(uint32_t) * (g.nslots + kSlotPad), st));
    SCHECK(cudaMemsetAsync(g.stwin, 0, sizeof(uint32_t) * (g.nslots + kSlotPad), st));
    const int64_t npos_sw = g.nslices * 32;
    eslot_kernel<<<grid_of(npos_sw), 256, 0, st>>>(npos_sw, g.slice_info, g.srow, g.sdeg,
                                                   g.row_ptr, eslot);
    stwin_kernel<<<grid_of(npos_sw), 256, 0, st>>>(npos_sw, g.slice_info, g.srow, g.sdeg,
                                                   g.row_ptr, g.er, eslot, g.stwin);
    SCHECK(cudaGetLastError());
    cudaFreeAsync(eslot, st);
    SCHECK(cudaStreamSynchronize(st));
    return GABP_OK;
}

cudaError_t prepare_slice_kernels() {
    int dev = 0, sms = 0, occ = 0;
    cudaError_t e;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess)
        return e;
    if ((e = cudaFuncSetAttribute(slice_kernel_pipe, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)kPipeSmem)) != cudaSuccess)
        return e;
    if ((e = cudaFuncSetAttribute(slice_kernel_pipe,
                                  cudaFuncAttributePreferredSharedMemoryCarveout, 100)) !=
        cudaSuccess)
        return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, slice_kernel_pipe, kPThreads,
                                                           kPipeSmem)) != cudaSuccess)
        return e;
    g_grid_pipe = sms * (occ > 0 ? occ : 1);
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, slice_kernel_ldg<false>,
                                                           kLThreads, 0)) != cudaSuccess)
        return e;
    g_grid_ldg = sms * (occ > 0 ? occ : 1);
    if ((e = cudaFuncSetAttribute(slice_kernel_grp, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)kGrpSmem)) != cudaSuccess)
        return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, slice_kernel_grp, kGThreads,
                                                           kGrpSmem)) != cudaSuccess)
        return e;
    g_grid_grp = sms * (occ > 0 ? occ : 1);
    for (auto k : {slice_kernel_par<false>, slice_kernel_par<true>})
        if ((e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kGrpSmem)) != cudaSuccess)
            return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, slice_kernel_par<false>,
                                                           kGThreads, kGrpSmem)) != cudaSuccess)
        return e;
    g_grid_par = sms * (occ > 0 ? occ : 1);
    return cudaSuccess;
}

// GABP_TWIN_LAUNCH=1 keeps the host-launched exact twin on the group path (A/B timing)
static bool twin_tail_enabled() {
    static const int v = getenv("GABP_TWIN_LAUNCH") ? atoi(getenv("GABP_TWIN_LAUNCH")) : 0;
    return !v;
}

// GABP_NO_PROBE=1 disables the residual probe (A/B timing)
static bool probe_enabled() {
    static const int off = getenv("GABP_NO_PROBE") ? atoi(getenv("GABP_NO_PROBE")) : 0;
    return !off;
}
// GABP_PROBE_FORCE=1: a probe after every launch (tests the mispredicted-probe path)
static int probe_forced() {
    static const int on = getenv("GABP_PROBE_FORCE") ? atoi(getenv("GABP_PROBE_FORCE")) : 0;
    return on ? 1 : 0;
}

// the exact register-batch kernel over [a.sl_lo, a.sl_hi): the twin (runs only when the
// fast launch flagged itself) or, with a.exact_primary, the sweep itself; returns its grid
static int64_t launch_slice_exact(const SweepArgs &a, cudaStream_t st) {
    int64_t gx = g_grid_ldg > 0 ? g_grid_ldg : 148 * 2;
    const int64_t nx = (a.sl_hi - a.sl_lo + kLWarps - 1) / kLWarps;
    if (gx > nx) gx = nx > 0 ? nx : 1;
    slice_kernel_ldg<true><<<(unsigned)gx, kLThreads, 0, st>>>(a);
    return gx;
}

static void launch_slice_fast(const SweepArgs &a, cudaStream_t st) {
    const int64_t nw = a.slice_variant ? kPWarps : kLWarps;
    int64_t grid = a.slice_variant ? g_grid_pipe : g_grid_ldg;
    if (grid <= 0) grid = 148 * 2;
    const int64_t need = (a.nslices + nw - 1) / nw;
    if (grid > need) grid = need > 0 ? need : 1;
    if (a.slice_variant)
        slice_kernel_pipe<<<(unsigned)grid, kPThreads, kPipeSmem, st>>>(a);
    else
        slice_kernel_ldg<false><<<(unsigned)grid, kLThreads, 0, st>>>(a);
}

cudaError_t launch_slice_sweep(const SweepArgs &a, cudaStream_t st) {
    return launch_slice_part(a, 0, st);
}

// One sweep over [a.sl_lo, a.sl_hi) with the fast kernel (reserve_sms SMs left free for a
// concurrent exchange), then the exact twin over every slice: a flagged launch is redone
// whole, so the statistics of an earlier part of the same sweep are re-taken too.
cudaError_t launch_slice_part(const SweepArgs &a0, int reserve_sms, cudaStream_t st) {
    SweepArgs a = a0;
    // residual probe: a residual-only group launch (variant 2), else run by the exact twin
    a.probe = (!a0.dist && probe_enabled()) ? (a0.slice_variant == 2 ? 2 : 1) : 0;
    a.probe_force = probe_forced();
    a.twin_tail = (a.slice_variant == 2 && !a0.dist && a0.sl_lo == 0 &&
                   a0.sl_hi == a0.nslices && twin_tail_enabled()) ? 1 : 0;
    {
        int64_t gx = g_grid_ldg > 0 ? g_grid_ldg : 148 * 2;
        const int64_t nx = (a.nslices + kLWarps - 1) / kLWarps;
        if (gx > nx) gx = nx > 0 ? nx : 1;
        a.twin_grid = (int)gx;
    }
    if (a.slice_variant == 2) {
        int64_t grid = (g_grid_grp > 0 ? g_grid_grp : 148) - reserve_sms;
        const int64_t need = (a.sl_hi - a.sl_lo) / kGroup;
        if (grid > need) grid = need;
        if (grid < 1) grid = 1;
        slice_kernel_grp<<<(unsigned)grid, kGThreads, kGrpSmem, st>>>(a);
    } else {
        launch_slice_fast(a, st);
    }
    // exact twin: exits at once unless the fast launch flagged itself (Ctrl.redo); the
    // whole-graph group launch tail-launches it from the device instead
    if (a.twin_tail) return cudaGetLastError();
    SweepArgs t = a;
    t.sl_lo = 0;
    t.sl_hi = a.nslices;
    t.part_base = 0;
    t.exact_primary = 0;
    launch_slice_exact(t, st);
    return cudaGetLastError();
}

// Parallel schedule: the fast kernel, then its exact twin (exits unless flagged).
cudaError_t launch_slice_parallel(const SweepArgs &a0, cudaStream_t st) {
    SweepArgs a = a0;
    a.probe = (!a0.dist && probe_enabled()) ? 1 : 0;
    a.probe_force = probe_forced();
    int64_t grid = g_grid_par > 0 ? g_grid_par : 148;
    const int64_t need = (a.sl_hi - a.sl_lo) / kGroup;
    if (grid > need) grid = need > 0 ? need : 1;
    slice_kernel_par<false><<<(unsigned)grid, kGThreads, kGrpSmem, st>>>(a);
    SweepArgs t = a;
    t.exact_primary = 0;
    slice_kernel_par<true><<<(unsigned)grid, kGThreads, kGrpSmem, st>>>(t);
    return cudaGetLastError();
}

// The boundary part of a split multi-rank sweep: exact divisions, so its results (sent to
// the peers before the interior part runs) never need the twin.
cudaError_t launch_slice_boundary(const SweepArgs &a, int64_t *grid, cudaStream_t st) {
    SweepArgs b = a;
    b.exact_primary = 1;
    *grid = launch_slice_exact(b, st);
    return cudaGetLastError();
}


}  // namespace gabp
