// small.cu -- the whole broadcast solve of a small graph in ONE launch of one thread-block
// cluster, every operand on chip.
//
// BASELINE config 0 (the reference's own case: Poisson 32x32, 1024 nodes, 3968 directed
// edges) needs 1731 sweeps to ||Ax-b||/||b|| < 1e-8; one kernel launch per sweep plus a
// grid-wide decision costs ~15-20 us per sweep on a graph of 100 KB.  Here the solve loop
// of solver.py:307-346 runs inside a cluster of C <= 8 CTAs (C SMs, distributed shared
// memory); CTA c owns a contiguous block of rows and their incoming message slots:
//
//   shared  I[2][EL]  incoming messages of the owned rows, slot e of row i = m_{dst(e) -> i}
//                     (CSR order), so a row's sums read contiguous local slots; R[2][NL] =
//                     {P_i, x_i} of the owned rows; A[EL]; X[EL] = the cluster address of
//                     x_{dst(e)} in its owner's R (residual rows)
//   regs    per edge: source row, cluster address of the twin slot, -A_ij^2, refined
//                     1/A_ij, the edge's own previous message (the change statistic: the
//                     thread that computes m_ij computed it last sweep too); per node:
//                     A_ii, prior numerator, b_i, row range
//
// Every sweep is two phases separated by cluster barriers (barrier.cluster, ~380 cycles):
//   A(t)  node i: P_i = A_ii + sum_k P_ki, N_i = A_ii mu_ii + sum_k P_ki mu_ki over S_{t-1}
//         in ascending k (np.add.at order, solver.py:239-242), x_i = N_i / P_i -> R[t&1]
//   B(t)  edge e = i -> j: m_ij = (-A_ij^2 / (P_i - P_ji), (P_i x_i - P_ji mu_ji) / A_ij)
//         (solver.py:247-257; sum_p * mu_tilde is P_i x_i) stored into the twin slot of j's
//         owner (st.shared::cluster), the statistics of sweep t; node i: residual row of
//         x^{(t-1)} (A_ii x_i, then + A_ij x_j in ascending j, x_j read from its owner)
// Every warp then publishes its partial statistics to every CTA of the cluster; after the
// barrier a dedicated decision warp per CTA (no row or edge work) reduces them in a fixed
// order and lane 0 takes the decision for sweep t-1 exactly as decide_sweep
// (gabp_internal.cuh) does -- change, blow-up / finiteness, means, epsilon, relative
// residual, sweep cap -- and the singular test of sweep t (solver.py:321-345), identically
// in every CTA, while the compute warps run A(t+1); the stop flag is read after the next
// barrier, and the state it refers to is still intact (two buffers of each).  Bitwise the
// reference: same operations in the same order, IEEE divisions (the compiler's fast path;
// its own slow path when the range test fails).
#include <float.h>
#include <math.h>
#include <stdlib.h>

#include "sweep_common.cuh"

namespace gabp {
namespace {

constexpr int kClMax = kSmallMaxCluster;  // CTAs per cluster (portable limit)
constexpr int kSmMaxWarps = 16;           // compute warps per CTA

struct SmRed {
    // partial statistics of every compute warp of every CTA, [cta][warp]
    double chg[kClMax][kSmMaxWarps];
    double rsq[kClMax][kSmMaxWarps];
    unsigned fl[kClMax][kSmMaxWarps];      // bit 0 out of range, bit 1 NaN change, bit 2 means bad
    unsigned sing[kClMax][kSmMaxWarps];    // first edge with P_excl == 0
    unsigned asing[kClMax][kSmMaxWarps];   // first node with P_i == 0
};
struct SmCtl {
    int stop;
    int64_t T;
};

__device__ __forceinline__ uint32_t su32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t cl_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cl_map(const void *p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(su32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void cl_st(uint32_t addr, double a, double b) {
    asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(a), "d"(b)
                 : "memory");
}
__device__ __forceinline__ void cl_st(uint32_t addr, double a) {
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(a) : "memory");
}
__device__ __forceinline__ void cl_st(uint32_t addr, unsigned a) {
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(a) : "memory");
}
__device__ __forceinline__ double cl_ld(uint32_t addr) {
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ unsigned cl_ld_u32(uint32_t addr) {
    unsigned v;
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
// all threads of all CTAs; remote stores before it are visible after it
__device__ __forceinline__ void cl_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n"
                 "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// owner CTA of edge slot (or row) v: the block c with b[c] <= v < b[c+1]
__device__ __forceinline__ uint32_t owner_of(const uint32_t *b, int C, uint32_t v) {
    uint32_t c = 0;
#pragma unroll
    for (int k = 1; k < kClMax; ++k) c += (k < C && v >= b[k]) ? 1u : 0u;
    return c;
}

// NT compute threads + one decision warp; EPT edge slots and NPT rows per compute thread
// PAR: the parallel schedule (solver.py:146-173) -- B(u) forms every outgoing message from
// the exclusion sum over its row's incoming slots (ascending, own slot skipped) instead of
// aggregate minus twin; the node phase, statistics and decisions are the same (no aggregate
// singular test: _sweep_parallel raises on P_excl only).
template <int NT, int EPT, int NPT, bool PAR>
__global__ void __launch_bounds__(NT + 32, 1) small_solve_kernel(const SweepArgs a,
                                                                const SmallPart part) {
    constexpr int kW = NT / 32;
    constexpr int EL = NT * EPT, NL = NT * NPT;  // local capacities
    static_assert(kW <= kSmMaxWarps, "warp table");
    // (one dynamic block, the same layout in every CTA: a peer's slot is this CTA's offset
    // mapped to the peer's rank)
    extern __shared__ __align__(16) unsigned char sm_raw[];
    double2(*sI)[EL] = reinterpret_cast<double2(*)[EL]>(sm_raw);
    double2(*sR)[NL] = reinterpret_cast<double2(*)[NL]>(sm_raw + 2 * EL * sizeof(double2));  // [3]
    double *sA = reinterpret_cast<double *>(sm_raw + (2 * EL + 3 * NL) * sizeof(double2));
    uint32_t *sX = reinterpret_cast<uint32_t *>(sm_raw + (2 * EL + 3 * NL) * sizeof(double2) +
                                                EL * sizeof(double));
    double2 *sND = reinterpret_cast<double2 *>(sm_raw + (2 * EL + 3 * NL) * sizeof(double2) +
                                               EL * (sizeof(double) + sizeof(uint32_t)));  // [NL]
    __shared__ SmRed red[2];
    __shared__ SmCtl ctl;
    __shared__ uint32_t s_nb[kClMax + 1], s_eb[kClMax + 1];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int C = part.C;
    const uint32_t rank = cl_rank();
    const int n = (int)a.n;
    volatile Ctrl *vc = a.ctrl;
    const double eps = vc->epsilon, rel_tol = vc->rel_tol, bnorm = vc->bnorm;
    const double lim = fmin(vc->blowup, DBL_MAX);
    const int64_t max_iter = vc->max_iter, nglob = vc->n;
    if (tid <= C) {
        s_nb[tid] = part.nb[tid];
        s_eb[tid] = __ldg(a.row_ptr + part.nb[tid]);
    }
    if (tid == 0) {
        ctl.stop = 0;
        ctl.T = 0;
    }
    __syncthreads();
    const uint32_t n0 = s_nb[rank], nloc = s_nb[rank + 1] - n0;
    const uint32_t e0 = s_eb[rank], eloc = s_eb[rank + 1] - e0;
    const bool decider = warp == kW;

    // S_0 = 0, graph records into shared memory and registers
    uint32_t esrc[EPT], etw[EPT];
    uint32_t ers[EPT], ere[EPT];  // (PAR) the source row's slots
    double emcc[EPT], erc[EPT];
    double2 mold[EPT];
    uint32_t ne0[NPT], ne1[NPT];
    double ndg[NPT], npn[NPT], nrh[NPT];
    if (!decider) {
#pragma unroll
        for (int k = 0; k < EPT; ++k) {
            const uint32_t e = tid + k * NT;
            esrc[k] = 0u;
            etw[k] = 0u;
            ers[k] = ere[k] = 0u;
            emcc[k] = -1.0;
            erc[k] = 1.0;
            mold[k] = make_double2(0.0, 0.0);
            if (e < EL) {
                sI[0][e] = make_double2(0.0, 0.0);
                sI[1][e] = make_double2(0.0, 0.0);
            }
            if (e < eloc) {
                const uint32_t ge = e0 + e;
                uint32_t lo = n0, hi = n0 + nloc;  // largest i with row_ptr[i] <= ge
                while (hi - lo > 1) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (__ldg(a.row_ptr + mid) <= ge) lo = mid; else hi = mid;
                }
                const EdgeRec r = a.er[ge];
                esrc[k] = lo - n0;
                if (PAR) {
                    ers[k] = __ldg(a.row_ptr + lo) - e0;
                    ere[k] = __ldg(a.row_ptr + lo + 1) - e0;
                }
                const uint32_t ot = owner_of(s_eb, C, r.rev);
                etw[k] = cl_map(&sI[0][r.rev - s_eb[ot]], ot);
                emcc[k] = -r.coeff * r.coeff;  // (-coeff * coeff, solver.py:256)
                erc[k] = ddiv_rcp(r.coeff);
                sA[e] = r.coeff;
                const uint32_t oc = owner_of(s_nb, C, r.col);
                sX[e] = cl_map(&sR[0][r.col - s_nb[oc]].y, oc);
            }
        }
#pragma unroll
        for (int q = 0; q < NPT; ++q) {
            const uint32_t il = tid + q * NT;
            ne0[q] = ne1[q] = 0u;
            ndg[q] = npn[q] = nrh[q] = 0.0;
            if (il < nloc) {
                const uint32_t i = n0 + il;
                ne0[q] = __ldg(a.row_ptr + i) - e0;
                ne1[q] = __ldg(a.row_ptr + i + 1) - e0;
                ndg[q] = __ldg(&a.nd[i].diag);
                npn[q] = __ldg(&a.nd[i].pnum);
                nrh[q] = __ldg(a.rhs + i);
                if (PAR) sND[il] = make_double2(ndg[q], npn[q]);
            }
        }
    }
    cl_barrier();  // every CTA's buffers are initialised before a remote store can land

    // When the CTA's rows fill at most half of its compute threads, the residual row of node
    // il runs on thread il + NT / 2, beside the thread that sums the node's messages: the
    // node phase is the stretch every other warp waits for at the CTA barrier.
    const bool split = NPT == 1 && nloc <= (uint32_t)(NT / 2);
    uint32_t rr_il = 0xffffffffu, rr_e0 = 0u, rr_e1 = 0u;
    double rr_dg = 0.0, rr_rh = 0.0;
    if (split && !decider && tid >= NT / 2 && (uint32_t)(tid - NT / 2) < nloc) {
        rr_il = (uint32_t)(tid - NT / 2);
        const uint32_t i = n0 + rr_il;
        rr_e0 = __ldg(a.row_ptr + i) - e0;
        rr_e1 = __ldg(a.row_ptr + i + 1) - e0;
        rr_dg = __ldg(&a.nd[i].diag);
        rr_rh = __ldg(a.rhs + i);
    }
    // Iteration u, compute warps:  A(u): marginals of S_{u-1} into R[u % 3] and the residual
    // rows of x^{(u-2)} (R[(u-1) % 3], complete everywhere since the last cluster barrier);
    // CTA barrier; B(u): messages of S_u into the owners' slots, statistics published into
    // table u & 1 of every CTA; ONE cluster barrier.  Decision warp, meanwhile: reduces table
    // (u-1) & 1 and decides sweep u-3 -- its change is two tables old, its means flag one
    // table old, its residual in this table -- then the singular test of sweep u-2; the
    // compute warps read the stop flag after the next cluster barrier, when S_T's marginals
    // (R[(T+1) % 3]) are still intact.
    int64_t T = 0;  // final sweep
    int conv = 0, divg = 0;
    double chg_1 = 0.0, chg_2 = 0.0;      // change of the sweep one / two tables back
    unsigned fl_1 = 0u, fl_2 = 0u;        // message flags of those sweeps
    unsigned mb_1 = 0u;                   // means flag of the table before
    unsigned sg_1 = 0xffffffffu, asg_1 = 0xffffffffu;  // singular indices of the table before
    int64_t u = 1;
    for (;; ++u) {
        if (!decider) {
            const int bo = (int)((u - 1) & 1), bn = (int)(u & 1);
            const int rn = (int)(u % 3), rp = (int)((u + 2) % 3);  // R of S_{u-1}, S_{u-2}
            unsigned asing = 0xffffffffu, mbad = 0u;
            double rsq = 0.0;
            // ---- A(u): aggregates and marginals of S_{u-1}; residual rows of x^{(u-2)} ----
            const double2 *Io = sI[bo];
            double *xh = (a.xhist && u >= 2 && u - 1 <= a.xhist_rows)
                             ? a.xhist + (u - 2) * n : nullptr;
            const uint32_t x_off = (uint32_t)rp * (uint32_t)(NL * sizeof(double2));
#pragma unroll
            for (int q = 0; q < NPT; ++q) {
                const uint32_t il = tid + q * NT;
                if (il < nloc) {
                    double P = ndg[q], N = npn[q];
                    double y = ndg[q] * sR[rp][il].y;
#pragma unroll 4
                    for (uint32_t e = ne0[q]; e < ne1[q]; ++e) {
                        const double2 v = Io[e];
                        P = P + v.x;
                        N = N + v.x * v.y;  // (prec * mean), solver.py:240
                        if (!split && u >= 3) y = y + sA[e] * cl_ld(sX[e] + x_off);
                    }
                    DivRange dr;
                    double x = ddiv_fast_acc(N, P, dr);
                    if (!div_range_ok(dr)) x = div_slow(N, P);  // (rare: out of the fast range)
                    if (!PAR && P == 0.0) asing = min(asing, n0 + il);
                    if (!(fabs(x) <= DBL_MAX)) mbad = 1u;
                    sR[rn][il] = make_double2(P, x);
                    if (xh) xh[n0 + il] = x;
                    if (!split && u >= 3) {
                        const double r = y - nrh[q];
                        rsq += r * r;
                    }
                }
            }
            if (split && u >= 3 && rr_il != 0xffffffffu) {  // residual row of x^{(u-2)}
                double y = rr_dg * sR[rp][rr_il].y;
#pragma unroll 4
                for (uint32_t e = rr_e0; e < rr_e1; ++e) y = y + sA[e] * cl_ld(sX[e] + x_off);
                const double r = y - rr_rh;
                rsq += r * r;
            }
            asm volatile("bar.sync 1, %0;" ::"r"(NT) : "memory");  // the compute warps' R[rn]
            // ---- B(u): messages of S_u, statistics --------------------------------------
            const double2 *Rt = sR[rn];
            const uint32_t tw_off = (uint32_t)bn * (uint32_t)(EL * sizeof(double2));
            double chg = 0.0;
            unsigned fl = 0u, sing = 0xffffffffu;
            DivRange dr;  // fast-path range test of all this thread's divisions, applied once
            double2 mnew[EPT];
            // P_excl and the numerator of edge slot e = (row i, neighbour j): broadcast --
            // aggregate minus the twin message m_ji (solver.py:247-254); parallel -- prior
            // plus the row's incoming terms in ascending order, own slot skipped (:147-150)
            auto edge_in = [&](int k, uint32_t e, double &pe, double &num) {
                if (PAR) {
                    const double2 nd = sND[esrc[k]];
                    pe = nd.x;
                    num = nd.y;
                    for (uint32_t q = ers[k]; q < ere[k]; ++q) {
                        const double2 v = Io[q];
                        if (q != e) {
                            pe = pe + v.x;
                            num = num + v.x * v.y;  // (prec * mean), solver.py:148
                        }
                    }
                } else {
                    const double2 ri = Rt[esrc[k]];
                    const double2 v = Io[e];  // m_ji of S_{u-1}: row i's incoming slot from j
                    pe = ri.x - v.x;
                    num = ri.x * ri.y - v.x * v.y;
                }
            };
#pragma unroll
            for (int k = 0; k < EPT; ++k) {
                const uint32_t e = tid + k * NT;
                mnew[k] = mold[k];
                if (e < eloc) {
                    double pe, num;
                    edge_in(k, e, pe, num);
                    const double np_ = ddiv_fast_acc(emcc[k], pe, dr);
                    const double nm = ddiv_fast_acc_r(num, sA[e], erc[k], dr);
                    if (pe == 0.0) sing = min(sing, e0 + e);
                    mnew[k] = make_double2(np_, nm);
                }
            }
            if (!div_range_ok(dr)) {
                // some division left the fast path's range: this thread's edges again with
                // IEEE division (same inputs, still in the old buffer)
                for (int k = 0; k < EPT; ++k) {
                    const uint32_t e = tid + k * NT;
                    if (e < eloc) {
                        double pe, num;
                        edge_in(k, e, pe, num);
                        mnew[k] = make_double2(div_slow(emcc[k], pe), div_slow(num, sA[e]));
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < EPT; ++k) {
                const uint32_t e = tid + k * NT;
                if (e < eloc) {
                    // mold: m_ij of S_{u-1}, this thread's own result of the last sweep
                    const double d1 = fabs(mnew[k].x - mold[k].x), d2 = fabs(mnew[k].y - mold[k].y);
                    chg = fmax(chg, fmax(d1, d2));
                    if (!(fabs(mnew[k].x) <= lim) || !(fabs(mnew[k].y) <= lim))
                        fl |= (mnew[k].x != mnew[k].x || mnew[k].y != mnew[k].y) ? 3u : 1u;
                    cl_st(etw[k] + tw_off, mnew[k].x, mnew[k].y);
                    mold[k] = mnew[k];
                }
            }
            // warp partials (fixed shapes: run-to-run reproducible), published to every CTA
            chg = warp_max(chg);
            rsq = warp_sum(rsq);
            fl = warp_or(fl | (mbad << 2));
            sing = warp_min(sing);
            asing = warp_min(asing);
            if (lane == 0) {  // into this CTA's own table: the decision warps pull them
                SmRed &Rw = red[bn];
                Rw.chg[rank][warp] = chg;
                Rw.rsq[rank][warp] = rsq;
                Rw.fl[rank][warp] = fl;
                Rw.sing[rank][warp] = sing;
                Rw.asing[rank][warp] = asing;
            }
        } else if (u >= 2) {
            // ---- decision warp: table of iteration u-1 ----------------------------------
            const SmRed &R1 = red[(u - 1) & 1];
            double c_t = 0.0, rsq_p = 0.0;
            unsigned f = 0u, sg = 0xffffffffu, asg = 0xffffffffu;
            // every CTA's warp partials, read from their owners (ld.shared::cluster; this
            // warp is off the sweep's critical path, so the compute warps publish nothing
            // remotely: 280 remote stores per CTA and sweep less before the cluster barrier)
            for (int idx = lane; idx < C * kW; idx += 32) {  // (cta, warp) order per lane
                const int c = idx / kW, w = idx - c * kW;
                c_t = fmax(c_t, cl_ld(cl_map(&R1.chg[c][w], (uint32_t)c)));
                rsq_p += cl_ld(cl_map(&R1.rsq[c][w], (uint32_t)c));
                f |= cl_ld_u32(cl_map(&R1.fl[c][w], (uint32_t)c));
                sg = min(sg, cl_ld_u32(cl_map(&R1.sing[c][w], (uint32_t)c)));
                asg = min(asg, cl_ld_u32(cl_map(&R1.asing[c][w], (uint32_t)c)));
            }
            c_t = warp_max(c_t);
            rsq_p = warp_sum(rsq_p);
            f = warp_or(f);
            sg = warp_min(sg);
            asg = warp_min(asg);
            if (lane == 0) {
                int stop = 0;
                const int64_t tp = u - 3;  // decide sweep u-3 (decide_sweep order)
                if (tp >= 1) {
                    const double change = (fl_2 & 2u) ? NAN : chg_2;
                    const bool means_finite = !(mb_1 & 4u);
                    if (rank == 0) {
                        a.change_hist[tp - 1] = change;
                        a.res_hist[tp - 1] = means_finite ? sqrt(rsq_p) / (double)nglob : INFINITY;
                        a.rsq_hist[tp - 1] = means_finite ? rsq_p : INFINITY;
                    }
                    T = tp;
                    if ((fl_2 & 1u) || !means_finite) {
                        divg = 1;
                        stop = 1;
                    } else if (change < eps) {
                        conv = 1;
                        stop = 1;
                    } else if (rel_tol > 0.0 && sqrt(rsq_p) < rel_tol * bnorm) {
                        conv = 1;
                        stop = 1;
                    } else if (tp >= max_iter) {
                        divg = 1;  // sweep cap (solver.py:344-345)
                        stop = 1;
                    }
                }
                if (!stop && u >= 3 && (sg_1 != 0xffffffffu || asg_1 != 0xffffffffu)) {
                    // SingularSubgraphError in sweep u-2: state not advanced (solver.py:322-326)
                    divg = 1;
                    stop = 1;
                    T = u - 3;
                }
                chg_2 = chg_1;
                fl_2 = fl_1;
                chg_1 = c_t;
                fl_1 = f & 3u;
                mb_1 = f & 4u;
                sg_1 = sg;
                asg_1 = asg;
                if (stop) {
                    ctl.T = T;
                    ctl.stop = 1;  // read by this CTA's warps after the next cluster barrier
                }
            }
        }
        cl_barrier();  // S_u, R of S_{u-1} and the statistics of iteration u are everywhere
        if (ctl.stop) break;
    }
    // the final state S_T: its marginals were formed by A(T+1), in R[(T+1) % 3]; the loop ran
    // at most two sweeps past T + 1
    if (!decider) {
        const double2 *Rf = sR[(ctl.T + 1) % 3];
        for (uint32_t il = tid; il < nloc; il += NT) {
            const double2 r = Rf[il];
            a.x[0][n0 + il] = r.y;
            a.p[0][n0 + il] = r.x;
        }
    } else if (lane == 0 && rank == 0) {
        Ctrl *c = a.ctrl;
        c->iterations = T;
        c->n_hist = T;
        c->final_slot = 0;
        c->converged = conv;
        c->diverged = divg;
        c->next_sweep = u + 1;  // sweeps computed: u
        c->done = 1;
    }
    cl_barrier();  // no CTA leaves while a peer may still read its shared memory
}

struct SmallCfg {
    int nt, ept, npt;
};
constexpr SmallCfg kSmallCfg[2] = {{256, 2, 1}, {480, 4, 2}};

template <int NT, int EPT, int NPT, bool PAR>
cudaError_t launch_small_t(const SweepArgs &a, const SmallPart &p, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)p.C);
    cfg.blockDim = dim3(NT + 32);
    constexpr size_t kSmem = (size_t)NT * (EPT * (2 * 16 + 8 + 4) + NPT * 4 * 16);
    auto k = small_solve_kernel<NT, EPT, NPT, PAR>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kSmem);
    if (e != cudaSuccess) return e;
    cfg.dynamicSmemBytes = kSmem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)p.C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, a, p);
}

}  // namespace

// Plans the cluster of a small graph from its host row offsets: C blocks of rows with
// balanced edge + row counts, the smallest thread configuration whose per-CTA capacities
// hold every block.  false: the graph does not fit (the sweep-per-launch paths run it).
bool small_plan(int64_t n, const uint32_t *row_ptr, SmallPart *out) {
    if (n < 1) return false;
    const int64_t E = row_ptr[n];
    int C = (int)((E + 255) / 256);  // at least ~256 edge slots of work per CTA
    if (C < 1) C = 1;
    // (powers of two: 1, 2, 4, 8)
    int Cp = 1;
    while (Cp < C && Cp < kSmallMaxCluster) Cp *= 2;
    if (const char *f = getenv("GABP_SMALL_C")) {  // probe: force the first cluster size tried
        const int v = atoi(f);
        if (v == 1 || v == 2 || v == 4 || v == 8) Cp = v;
    }
    for (int C2 = Cp; C2 <= kSmallMaxCluster; C2 *= 2) {
        SmallPart p = {};
        p.C = C2;
        p.nb[0] = 0;
        // block c ends at the first row whose weight prefix reaches (c+1)/C of the total
        // (weight of a row: its edges + 1)
        const int64_t total = E + n;
        int64_t i = 0;
        for (int c = 1; c < C2; ++c) {
            const int64_t target = (total * c + C2 - 1) / C2;
            while (i < n && (int64_t)row_ptr[i] + i < target) ++i;
            p.nb[c] = (uint32_t)i;
        }
        p.nb[C2] = (uint32_t)n;
        int64_t emax = 0, nmax = 0;
        for (int c = 0; c < C2; ++c) {
            const int64_t ne = (int64_t)row_ptr[p.nb[c + 1]] - (int64_t)row_ptr[p.nb[c]];
            const int64_t nn = (int64_t)p.nb[c + 1] - (int64_t)p.nb[c];
            if (ne > emax) emax = ne;
            if (nn > nmax) nmax = nn;
        }
        for (int k = 0; k < 2; ++k) {
            const SmallCfg &s = kSmallCfg[k];
            if (emax <= (int64_t)s.nt * s.ept && nmax <= (int64_t)s.nt * s.npt) {
                p.cfg = k;
                *out = p;
                return true;
            }
        }
    }
    return false;
}

void small_capacity(int cfg, int64_t *edges, int64_t *rows) {
    const SmallCfg &s = kSmallCfg[cfg == 0 ? 0 : 1];
    *edges = (int64_t)s.nt * s.ept;
    *rows = (int64_t)s.nt * s.npt;
}

bool small_candidate(int64_t n, int64_t E) {
    const SmallCfg &s = kSmallCfg[1];
    return n >= 1 && n <= (int64_t)kSmallMaxCluster * s.nt * s.npt &&
           E <= (int64_t)kSmallMaxCluster * s.nt * s.ept;
}

cudaError_t launch_small_solve(const SweepArgs &a, const SmallPart &p, bool parallel,
                               cudaStream_t st) {
    if (parallel)
        return p.cfg == 0 ? launch_small_t<256, 2, 1, true>(a, p, st)
                          : launch_small_t<480, 4, 2, true>(a, p, st);
    return p.cfg == 0 ? launch_small_t<256, 2, 1, false>(a, p, st)
                      : launch_small_t<480, 4, 2, false>(a, p, st);
}

}  // namespace gabp
