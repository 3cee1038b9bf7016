// small.cu -- the whole broadcast solve of a small graph in ONE persistent CTA.
//
// BASELINE config 0 (the reference's own case: Poisson 32x32, 1024 nodes, 3968 directed
// edges) needs 1731 sweeps to ||Ax-b||/||b|| < 1e-8; one kernel launch per sweep plus a
// grid-wide decision costs ~15-20 us per sweep on a graph of 100 KB.  Here the solve loop
// of solver.py:307-346 runs inside one CTA of 1024 threads with every operand on chip:
//
//   shared  I[2][E]  incoming messages, slot e of row i = m_{dst(e) -> i} (CSR order), so a
//                    row's sums read contiguous slots and an edge's twin message is its own
//                    slot; R[2][n] = {P_i, x_i}; col[E], A[E] (residual rows)
//   regs    per edge: source, twin slot, -A_ij^2, refined 1/A_ij; per node: A_ii, prior
//                    numerator, b_i, row range
//
// Every sweep is two phases separated by CTA barriers:
//   A(t)  node i: P_i = A_ii + sum_k P_ki, N_i = A_ii mu_ii + sum_k P_ki mu_ki over S_{t-1}
//         in ascending k (np.add.at order, solver.py:239-242), x_i = N_i / P_i -> R[t&1]
//   B(t)  edge e = i -> j: m_ij = (-A_ij^2 / (P_i - P_ji), (P_i x_i - P_ji mu_ji) / A_ij)
//         (solver.py:247-257; sum_p * mu_tilde is P_i x_i) into the twin slot, the
//         statistics of sweep t; node i: residual row of x^{(t-1)} (A_ii x_i, then
//         + A_ij x_j in ascending j)
// Warp 0 then reduces the warp partials and lane 0 takes the decision for sweep t-1 exactly
// as decide_sweep (gabp_internal.cuh) does -- change, blow-up / finiteness, means, epsilon,
// relative residual, sweep cap -- and the singular test of sweep t (solver.py:321-345),
// while the other warps start A(t+1); the stop flag is read after the next barrier, and
// the state it refers to is still intact (two buffers of each).  Bitwise the reference:
// same operations in the same order, IEEE divisions (the compiler's fast path; its own
// slow path when the range test fails).
#include <float.h>
#include <math.h>

#include "sweep_common.cuh"

namespace gabp {
namespace {

constexpr int kSmMaxThreads = 1024;
constexpr int kSmWarps = kSmMaxThreads / 32;  // (reduction slots: the largest CTA)

struct SmRed {
    double chg[kSmWarps];
    double rsq[kSmWarps];
    unsigned fl[kSmWarps];      // bit 0 out of range, bit 1 NaN change, bit 2 means bad
    unsigned sing[kSmWarps];    // first edge with P_excl == 0
    unsigned asing[kSmWarps];   // first node with P_i == 0
    int stop;
};

template <int NT, int EPT, int NPT>
__global__ void __launch_bounds__(NT, 1) small_solve_kernel(const SweepArgs a) {
    constexpr int kSmThreads = NT;
    constexpr int kW = NT / 32;
    extern __shared__ __align__(16) unsigned char sm_raw[];
    __shared__ SmRed red;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = (int)a.n;
    const uint32_t E = __ldg(a.row_ptr + n);
    // (offsets from the __shared__ array, never pointer tables: the compiler must see shared
    // addresses to emit LDS/STS -- a pointer picked from an array becomes generic)
    double2 *sI = reinterpret_cast<double2 *>(sm_raw);  // [2][E]
    double2 *sR = sI + 2 * (size_t)E;                      // [2][n]
    double *sA = reinterpret_cast<double *>(sR + 2 * (size_t)n);
    uint32_t *scol = reinterpret_cast<uint32_t *>(sA + E);
    volatile Ctrl *vc = a.ctrl;
    const double eps = vc->epsilon, rel_tol = vc->rel_tol, bnorm = vc->bnorm;
    const double lim = fmin(vc->blowup, DBL_MAX);
    const int64_t max_iter = vc->max_iter, nglob = vc->n;

    // S_0 = 0, graph records into shared memory and registers
    for (uint32_t e = tid; e < E; e += kSmThreads) {
        const EdgeRec r = a.er[e];
        sI[e] = make_double2(0.0, 0.0);
        sA[e] = r.coeff;
        scol[e] = r.col;
    }
    uint32_t esrc[EPT], erev[EPT];
    double emcc[EPT], erc[EPT];
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
        const uint32_t e = tid + k * kSmThreads;
        esrc[k] = 0u;
        erev[k] = 0u;
        emcc[k] = -1.0;
        erc[k] = 1.0;
        if (e < E) {
            uint32_t lo = 0, hi = (uint32_t)n;  // largest i with row_ptr[i] <= e
            while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) >> 1;
                if (__ldg(a.row_ptr + mid) <= e) lo = mid; else hi = mid;
            }
            const EdgeRec r = a.er[e];
            esrc[k] = lo;
            erev[k] = r.rev;
            emcc[k] = -r.coeff * r.coeff;  // (-coeff * coeff, solver.py:256)
            erc[k] = ddiv_rcp(r.coeff);
        }
    }
    uint32_t ne0[NPT], ne1[NPT];
    double ndg[NPT], npn[NPT], nrh[NPT];
#pragma unroll
    for (int q = 0; q < NPT; ++q) {
        const int i = tid + q * kSmThreads;
        ne0[q] = ne1[q] = 0u;
        ndg[q] = npn[q] = nrh[q] = 0.0;
        if (i < n) {
            ne0[q] = __ldg(a.row_ptr + i);
            ne1[q] = __ldg(a.row_ptr + i + 1);
            ndg[q] = __ldg(&a.nd[i].diag);
            npn[q] = __ldg(&a.nd[i].pnum);
            nrh[q] = __ldg(a.rhs + i);
        }
    }
    if (tid == 0) red.stop = 0;
    // warp 0 lane 0: statistics of the previous sweep, decision state
    double chg_prev = 0.0;
    unsigned fl_prev = 0u;
    int64_t T = 0;  // final sweep
    int conv = 0, divg = 0;
    __syncthreads();

    int64_t t = 1;
    for (;; ++t) {
        const double2 *Io = sI + ((t - 1) & 1) * (size_t)E;
        double2 *In = sI + (t & 1) * (size_t)E;
        double2 *Rt = sR + (t & 1) * (size_t)n;
        // ---- A(t): aggregates and marginals of S_{t-1} ---------------------------------
        unsigned asing = 0xffffffffu, mbad = 0u;
        double *xh = (a.xhist && t >= 2 && t - 1 <= a.xhist_rows) ? a.xhist + (t - 2) * n
                                                                   : nullptr;
#pragma unroll
        for (int q = 0; q < NPT; ++q) {
            const int i = tid + q * kSmThreads;
            if (i < n) {
                double P = ndg[q], N = npn[q];
                for (uint32_t e = ne0[q]; e < ne1[q]; ++e) {
                    const double2 v = Io[e];
                    P = P + v.x;
                    N = N + v.x * v.y;  // (prec * mean), solver.py:240
                }
                DivRange dr;
                double x = ddiv_fast_acc(N, P, dr);
                if (!div_range_ok(dr)) x = div_slow(N, P);  // (rare: out of the fast range)
                if (P == 0.0) asing = min(asing, (unsigned)i);
                if (!(fabs(x) <= DBL_MAX)) mbad = 1u;
                Rt[i] = make_double2(P, x);
                if (xh) xh[i] = x;
            }
        }
        __syncthreads();
        if (red.stop) break;
        // ---- B(t): messages of S_t, statistics; residual rows of x^{(t-1)} -------------
        double chg = 0.0, rsq = 0.0;
        unsigned fl = 0u, sing = 0xffffffffu;
        DivRange dr;  // fast-path range test of all this thread's divisions, applied once
#pragma unroll
        for (int k = 0; k < EPT; ++k) {
            const uint32_t e = tid + k * kSmThreads;
            if (e < E) {
                const double2 ri = Rt[esrc[k]];
                const double2 v = Io[e];  // m_ji of S_{t-1}: row i's incoming slot from j
                const double pe = ri.x - v.x;
                const double num = ri.x * ri.y - v.x * v.y;
                const double np_ = ddiv_fast_acc(emcc[k], pe, dr);
                const double nm = ddiv_fast_acc_r(num, sA[e], erc[k], dr);
                const double2 old = Io[erev[k]];  // m_ij of S_{t-1}
                const double d1 = fabs(np_ - old.x), d2 = fabs(nm - old.y);
                chg = fmax(chg, fmax(d1, d2));
                if (!(fabs(np_) <= lim) || !(fabs(nm) <= lim))
                    fl |= (np_ != np_ || nm != nm) ? 3u : 1u;
                if (pe == 0.0) sing = min(sing, e);
                In[erev[k]] = make_double2(np_, nm);
            }
        }
        if (!div_range_ok(dr)) {
            // some division left the fast path's range: this thread's edges again with IEEE
            // division (same inputs, still in the old buffer), statistics re-taken
            chg = 0.0;
            fl = 0u;
            for (int k = 0; k < EPT; ++k) {
                const uint32_t e = tid + k * kSmThreads;
                if (e < E) {
                    const double2 ri = Rt[esrc[k]];
                    const double2 v = Io[e];
                    const double pe = ri.x - v.x;
                    const double num = ri.x * ri.y - v.x * v.y;
                    const double np_ = div_slow(emcc[k], pe);
                    const double nm = div_slow(num, sA[e]);
                    const double2 old = Io[erev[k]];
                    const double d1 = fabs(np_ - old.x), d2 = fabs(nm - old.y);
                    chg = fmax(chg, fmax(d1, d2));
                    if (!(fabs(np_) <= lim) || !(fabs(nm) <= lim))
                        fl |= (np_ != np_ || nm != nm) ? 3u : 1u;
                    In[erev[k]] = make_double2(np_, nm);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < NPT; ++q) {
            const int i = tid + q * kSmThreads;
            if (i < n) {
                double y = ndg[q] * Rt[i].y;
                for (uint32_t e = ne0[q]; e < ne1[q]; ++e) y = y + sA[e] * Rt[scol[e]].y;
                const double r = y - nrh[q];
                rsq += r * r;
            }
        }
        // CTA reductions (fixed shapes: run-to-run reproducible)
        chg = warp_max(chg);
        rsq = warp_sum(rsq);
        fl = warp_or(fl | (mbad << 2));
        sing = warp_min(sing);
        asing = warp_min(asing);
        if (lane == 0) {
            red.chg[warp] = chg;
            red.rsq[warp] = rsq;
            red.fl[warp] = fl;
            red.sing[warp] = sing;
            red.asing[warp] = asing;
        }
        __syncthreads();
        if (warp == 0) {
            const bool lv = lane < kW;
            const double c_t = warp_max(lv ? red.chg[lane] : 0.0);
            const double rsq_p = warp_sum(lv ? red.rsq[lane] : 0.0);
            const unsigned f = warp_or(lv ? red.fl[lane] : 0u);
            const unsigned sg = warp_min(lv ? red.sing[lane] : 0xffffffffu);
            const unsigned asg = warp_min(lv ? red.asing[lane] : 0xffffffffu);
            if (lane == 0) {
                int stop = 0;
                const int64_t tp = t - 1;  // decide sweep t-1 (decide_sweep order)
                if (tp >= 1) {
                    const double change = (fl_prev & 2u) ? NAN : chg_prev;
                    const bool means_finite = !(f & 4u);
                    a.change_hist[tp - 1] = change;
                    a.res_hist[tp - 1] = means_finite ? sqrt(rsq_p) / (double)nglob : INFINITY;
                    a.rsq_hist[tp - 1] = means_finite ? rsq_p : INFINITY;
                    T = tp;
                    if ((fl_prev & 1u) || !means_finite) {
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
                if (!stop && (sg != 0xffffffffu || asg != 0xffffffffu)) {
                    // SingularSubgraphError in sweep t: state not advanced (solver.py:322-326)
                    divg = 1;
                    stop = 1;
                    T = t - 1;
                }
                chg_prev = c_t;
                fl_prev = f & 3u;
                red.stop = stop;
            }
        }
        // (no barrier: A(t+1) writes the other node buffer; the stop flag is read after
        // the next barrier, before B(t+1) overwrites the state it refers to)
    }
    // the final state S_T: the decision was taken in iteration t-1 (T = t-2, or T = t-2 for
    // a singular sweep t-1) and its marginals were formed by A(t-1), in R[(t-1) & 1]
    const double2 *Rf = sR + ((t - 1) & 1) * (size_t)n;
    for (int i = tid; i < n; i += kSmThreads) {
        const double2 r = Rf[i];
        a.x[0][i] = r.y;
        a.p[0][i] = r.x;
    }
    if (tid == 0) {
        Ctrl *c = a.ctrl;
        c->iterations = T;
        c->n_hist = T;
        c->final_slot = 0;
        c->converged = conv;
        c->diverged = divg;
        c->next_sweep = t;  // sweeps computed: t - 1
        c->done = 1;
    }
}

constexpr size_t kSmMaxDyn = 227 * 1024 - sizeof(SmRed) - 256;

}  // namespace

// shared bytes: messages 2 x 16 E, node states 2 x 16 n, coefficients 8 E, columns 4 E
size_t small_smem_bytes(int64_t n, int64_t E) { return 44u * (size_t)E + 32u * (size_t)n; }

bool small_fits(int64_t n, int64_t E) {
    return n >= 1 && n <= 2 * kSmMaxThreads && E <= 5 * kSmMaxThreads &&
           small_smem_bytes(n, E) <= kSmMaxDyn;
}

#ifndef GABP_SMALL_NT
#define GABP_SMALL_NT 512
#endif
template <int NT, int EPT, int NPT>
cudaError_t launch_small_t(const SweepArgs &a, size_t smem, cudaStream_t st) {
    auto k = small_solve_kernel<NT, EPT, NPT>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kSmMaxDyn);
    if (e != cudaSuccess) return e;
    k<<<1, NT, smem, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_small_solve(const SweepArgs &a, int64_t E, cudaStream_t st) {
    const size_t smem = small_smem_bytes(a.n, E);
#if GABP_SMALL_NT == 512
    if (a.n <= 1024 && E <= 8 * 512) return launch_small_t<512, 8, 2>(a, smem, st);
#else
    if (a.n <= 1024 && E <= 4 * 1024) return launch_small_t<1024, 4, 1>(a, smem, st);
#endif
    return launch_small_t<1024, 5, 2>(a, smem, st);
}

}  // namespace gabp
