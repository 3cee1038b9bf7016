// dia.cu -- the broadcast solve on a diagonal (stencil) layout: graphs whose edges all lie
// on a few diagonals j - i = o_k (the Poisson grids of BASELINE configs 0, 2 and 4: 4 or 6
// diagonals at +-1, +-p, +-p^2).
//
// Layout (HBM, all arrays indexed by the local node i, natural order -- no permutation):
//   coef [D][nl]   A_{i, i+o_k}; 0 where row i has no neighbour on diagonal k
//   msg  [2][D][nl] {P, mu}: slot (k, i) holds row i's INCOMING message from j = i + o_k,
//                  m_{j -> i}; a double buffer (S_{s-1} read, S_s written)
//   p, x [3][nl]   P_i and the marginal x_i of the state S_t in ring slot t % 3
// The twin of slot (k, i) is slot (opp(k), j): a shifted, coalesced read of the same array,
// so the broadcast update (solver.py:232-272)
//   m_{j -> i} = (-A_ij^2 / (P_j - P_ij), (P_j x_j - P_ij mu_ij) / A_ij),   m_ij = slot (opp k, j)
// reads each old message once from DRAM (its second touch, one grid row / plane later, hits
// L2), and a row sums its new incoming messages straight away: launch s computes S_s, the
// aggregates and marginal x^{(s)}, the residual row of x^{(s-1)} and the statistics, and
// decides sweep s-1 -- per slot 16 B read + 16 B written + 8 B of coefficient, against 60 B
// on the recompute slice layout (slice.cu), which must rebuild every twin from an older
// message because a random graph has no such locality.
//
// Bitwise the reference: ascending diagonals are ascending neighbours (np.add.at order), IEEE
// divisions (fast path, range test deferred per node; a node whose test fails is redone with
// '/'), no FMA contraction.
#include <cub/device/device_reduce.cuh>
#include <float.h>
#include <math.h>
#include <stdio.h>

#include "sweep_common.cuh"

namespace gabp {
namespace {


// ---- sweep kernel ------------------------------------------------------------------------------
// A thread per row, every load of the row issued before any use; an empty slot (no neighbour
// on that diagonal: grid boundary, a missing edge) computes on harmless operands and adds
// -0.0 -- the identity of IEEE addition in round-to-nearest, for +-0 too -- so the row needs
// no branch per diagonal.  UNIFORM: every off-diagonal of the matrix has one value c (the
// Poisson grids: -1), so a row carries a byte of diagonal-occupancy bits instead of D
// coefficients (8 B per slot less traffic), and -c^2 and the refined 1/c are constants.
// EXACT: IEEE '/' everywhere -- the twin a fast launch tail-launches when one of its
// divisions left the fast path's range (the fast launch then discards its statistics).
// Tiles of kDRows rows, static and in the blocked order (dia_tile_row): per-CTA residual
// partials in CTA order, run-to-run reproducible.
#ifndef GABP_DIA_MINB
#define GABP_DIA_MINB 2
#endif
constexpr int kDRows = 256;

// first row of tile t (tile order: identity, or chunks of W rows of every O-row plane, so
// the second touch of a twin message or neighbour state is W rows -- a few MB -- after the
// first and hits L2, instead of a whole plane (~80 MB at 512^3) later)
__device__ __forceinline__ int64_t dia_tile_row(const SweepArgs &a, int64_t r0e, int64_t t) {
    if (a.dia_W <= 0) return r0e + t * kDRows;
    const int64_t tw = a.dia_W / kDRows;                            // tiles per chunk-plane
    const int64_t Z = (a.dia_r1 - r0e + a.dia_O - 1) / a.dia_O;     // planes
    const int64_t c = t / (Z * tw), rem = t % (Z * tw);
    return r0e + (rem / tw) * a.dia_O + c * a.dia_W + (rem % tw) * kDRows;
}
__host__ __device__ __forceinline__ int64_t dia_ntiles(const SweepArgs &a) {
    const int64_t r0e = a.dia_r0 & ~1ll;
    if (a.dia_W <= 0) return (a.dia_r1 - r0e + kDRows - 1) / kDRows;
    const int64_t Z = (a.dia_r1 - r0e + a.dia_O - 1) / a.dia_O;
    return (a.dia_O / a.dia_W) * Z * (a.dia_W / kDRows);
}

template <int D, bool UNIFORM, bool EXACT>
__global__ void __launch_bounds__(kDRows, GABP_DIA_MINB) dia_sweep_kernel(const SweepArgs a) {
    __shared__ TailSmem<kDRows / 32> T;
    __shared__ double srsq[kDRows / 32];
    __shared__ unsigned sasing[kDRows / 32];
    __shared__ int64_t s_sweep;
    __shared__ int s_skip;
    const int tid = threadIdx.x;
    if (tid == 0) {
        volatile Ctrl *vc = a.ctrl;
        const int64_t s = vc->next_sweep;
        s_sweep = s;
        s_skip = vc->done || s > vc->max_iter + 1;
        if (EXACT && blockIdx.x == 0) atomicAdd(&a.ctrl->twin_launches, 1);
    }
    __syncthreads();
    if (s_skip) return;
    const int64_t s = s_sweep;
    const int64_t nl = a.dia_nl, nlc = a.dia_nlc;
    const double2 *mo = a.msg[(s - 1) & 1];
    double2 *mn = a.msg[s & 1];
    const double *po = a.p[(s - 1) % 3], *xo = a.x[(s - 1) % 3];
    double *pn = a.p[s % 3], *xn = a.x[s % 3];
    double *xh = (a.xhist && s >= 1 && s <= a.xhist_rows) ? a.xhist + (s - 1) * a.n : nullptr;
    const double lim = fmin(a.ctrl->blowup, DBL_MAX);
    const bool resid = s >= 2;
    // per-diagonal constants in registers
    int64_t off[D], tws[D];
#pragma unroll
    for (int k = 0; k < D; ++k) {
        off[k] = a.dia_off[k];
        tws[k] = (int64_t)a.dia_opp[k] * nl + off[k];  // twin slot of (k, i): tws[k] + i
    }
    const double cu = a.dia_cu, mccu = -cu * cu;  // (-coeff * coeff, solver.py:256)
    const double rcu = UNIFORM && !EXACT ? ddiv_rcp(cu) : 1.0;
    double chg = 0.0, rsq = 0.0;
    unsigned fl = 0u, sing = 0xffffffffu, asing = 0xffffffffu, mbad = 0u;
    DivRange dr;
    const int64_t r0 = a.dia_r0, r1 = a.dia_r1, r0e = r0 & ~1ll;
    const int64_t nt = dia_ntiles(a);
    for (int64_t t = blockIdx.x; t < nt; t += gridDim.x) {
        const int64_t i = dia_tile_row(a, r0e, t) + tid;
        if (i < r0 || i >= r1) continue;
        // ---- loads
        double c[D], Pj[D], xj[D];
        double2 tw[D], old[D];
        unsigned mask = 0u;
        if (UNIFORM) mask = a.dia_mask[i];
#pragma unroll
        for (int k = 0; k < D; ++k) {
            if (!UNIFORM) c[k] = __ldcs(a.dia_coef + k * nlc + i);
            const int64_t j = i + off[k];  // (in the padded arrays for every i: never used
                                            //  when the slot is empty)
            // L2 policy by touch order: a message of a positive-offset diagonal is read first
            // as the row's own old message and a row or plane later as a twin; one of a
            // negative-offset diagonal the other way round -- only the second touch streams
            if (off[k] > 0) {
                tw[k] = __ldcg(mo + tws[k] + i);  // m_ij of S_{s-1}
                old[k] = __ldcg(mo + k * nl + i);
            } else {
                tw[k] = __ldcs(mo + tws[k] + i);
                old[k] = __ldcs(mo + k * nl + i);
            }
            Pj[k] = __ldcg(po + j);
            xj[k] = __ldcg(xo + j);
        }
        const NodeRec nd = a.nd[i];
        const double xi = __ldcg(xo + i), bi = __ldcs(a.rhs + i);
        // ---- the row
        double P = nd.diag, N = nd.pnum;
        double y = nd.diag * xi;  // residual row of x^{(s-1)}: A_ii x_i, then + A_ij x_j
#pragma unroll
        for (int k = 0; k < D; ++k) {
            const bool v = UNIFORM ? ((mask >> k) & 1u) != 0u : c[k] != 0.0;
            const double ck = UNIFORM ? cu : (v ? c[k] : 1.0);
            const double pe = v ? Pj[k] - tw[k].x : 1.0;
            // (sum_p * mu_tilde) - (prec * mean)
            // (an empty slot divides 1 by 1: in the fast path's range, result unused)
            const double num = v ? Pj[k] * xj[k] - tw[k].x * tw[k].y : 1.0;
            const double mcc = UNIFORM ? mccu : -ck * ck;
            double np_, nm;
            if (EXACT) {
                np_ = mcc / pe;
                nm = num / ck;
            } else {
                np_ = ddiv_fast_acc(mcc, pe, dr);
                nm = UNIFORM ? ddiv_fast_acc_r(num, ck, rcu, dr) : ddiv_fast_acc(num, ck, dr);
            }
            __stcs(mn + k * nl + i, make_double2(np_, nm));
            if (v) {
                const double d1 = fabs(np_ - old[k].x), d2 = fabs(nm - old[k].y);
                chg = fmax(chg, fmax(d1, d2));
                if (!(fabs(np_) <= lim) || !(fabs(nm) <= lim))
                    fl |= (np_ != np_ || nm != nm) ? 3u : 1u;
                if (pe == 0.0) sing = min(sing, (unsigned)i);
            }
            P = P + (v ? np_ : -0.0);
            N = N + (v ? np_ * nm : -0.0);  // (prec * mean), solver.py:240
            y = y + (v ? ck * xj[k] : -0.0);
        }
        double x;
        if (EXACT) {
            x = N / P;
        } else {
            x = ddiv_fast_acc(N, P, dr);
        }
        if (P == 0.0) asing = min(asing, (unsigned)i);  // (singular for sweep s + 1)
        if (!(fabs(x) <= DBL_MAX)) mbad = 1u;
        __stcg(pn + i, P);
        __stcg(xn + i, x);
        if (xh) xh[i] = x;
        if (resid) {
            const double r = y - bi;
            rsq += r * r;
        }
    }
    Stats st;
    st.chg = chg;
    st.rsq = rsq;
    st.out_of_range = fl;
    st.sing = sing;
    st.means_bad = mbad;
    const unsigned redo = EXACT ? 0u : (div_range_ok(dr) ? 0u : 1u);
    const bool twin = dia_epilogue<kDRows, EXACT>(T, srsq, sasing, a, s, st, asing, redo, tid);
    if constexpr (!EXACT) {
        if (twin && tid == 0) {
            // a fast division left its range: the exact twin redoes this sweep, launched into
            // the tail of this grid (after it, before the next launch of the stream)
            dia_sweep_kernel<D, UNIFORM, true><<<gridDim.x, kDRows, 0, cudaStreamTailLaunch>>>(a);
        }
    }
}

// ---- parallel schedule on the diagonal layout ----------------------------------------------
// solver.py:146-173: every outgoing message from the exclusion sum over the row's incoming
// slots (prior first, ascending neighbours, own slot skipped).  A row's incoming slots are
// its own D slots (coalesced); its outgoing message to j = i + o_k goes into j's slot
// (opp k, j) -- a shifted, coalesced WRITE of the same array, and the old outgoing message
// (the change statistic) is the shifted read the broadcast kernel makes for its twin.  So the
// reference's default schedule streams a stencil graph like the broadcast one: per slot 16 B
// read + 16 B written, the second touch of every old message from L2.  Launch protocol of
// the CSR kernels (sweep_epilogue, LAG 0): launch s reads S_{s-1}, writes S_s, forms the
// marginals x^{(s-1)} of the state it read and the residual row of x^{(s-2)}, decides sweep
// s-2.  Divisions: the fast path with its range test per division, IEEE '/' when it fails.
// CTAs per SM: three for up to 4 diagonals (80 registers; Poisson 4096^2 0.718 -> 0.633 ms),
// two for the wider stencils (three spill: 320^3 1.74 -> 2.32 ms)
constexpr int dia_par_minb(int D) { return D <= 4 ? 3 : 2; }
template <int D, bool UNIFORM>
__global__ void __launch_bounds__(kDRows, dia_par_minb(D)) dia_par_kernel(const SweepArgs a) {
    __shared__ TailSmem<kDRows / 32> T;
    __shared__ int64_t s_sweep;
    __shared__ int s_skip;
    const int tid = threadIdx.x;
    if (tid == 0) {
        volatile Ctrl *vc = a.ctrl;
        const int64_t s = vc->next_sweep;
        s_sweep = s;
        s_skip = vc->done || s > vc->max_iter + 2;
    }
    __syncthreads();
    if (s_skip) return;
    const int64_t s = s_sweep;
    const int64_t nl = a.dia_nl, nlc = a.dia_nlc;
    const double2 *mo = a.msg[(s - 1) % 3];
    double2 *mn = a.msg[s % 3];
    const bool resid = s >= 3;
    const double *xp = a.x[(s + 1) % 3];  // x^{(s-2)} (residual), read when resid
    double *xc = a.x[(s - 1) % 3], *pc = a.p[(s - 1) % 3];
    double *xh = (a.xhist && s >= 2 && s - 1 <= a.xhist_rows) ? a.xhist + (s - 2) * a.n : nullptr;
    Stats st;
    st.lim = fmin(a.ctrl->blowup, DBL_MAX);
    int64_t off[D], tws[D];
#pragma unroll
    for (int k = 0; k < D; ++k) {
        off[k] = a.dia_off[k];
        tws[k] = (int64_t)a.dia_opp[k] * nl + off[k];  // slot (opp k, i + o_k): tws[k] + i
    }
    const double cu = a.dia_cu, mccu = -cu * cu;  // (-coeff * coeff, solver.py:156)
    const double rcu = UNIFORM ? ddiv_rcp(cu) : 1.0;
    const int64_t r0 = a.dia_r0, r1 = a.dia_r1, r0e = r0 & ~1ll;
    const int64_t nt = dia_ntiles(a);
    for (int64_t t = blockIdx.x; t < nt; t += gridDim.x) {
        const int64_t i = dia_tile_row(a, r0e, t) + tid;
        if (i < r0 || i >= r1) continue;
        // ---- loads
        double c[D], xj[D];
        double2 in[D], old[D];
        unsigned mask = 0u;
        if (UNIFORM) mask = a.dia_mask[i];
#pragma unroll
        for (int k = 0; k < D; ++k) {
            if (!UNIFORM) c[k] = __ldcs(a.dia_coef + k * nlc + i);
            // (touch order as in the broadcast kernel: only the second touch streams)
            if (off[k] > 0) {
                old[k] = __ldcg(mo + tws[k] + i);  // m_ij of S_{s-1}: j's slot from i
                in[k] = __ldcg(mo + k * nl + i);   // m_ji of S_{s-1}
            } else {
                old[k] = __ldcs(mo + tws[k] + i);
                in[k] = __ldcs(mo + k * nl + i);
            }
            xj[k] = resid ? __ldcg(xp + i + off[k]) : 0.0;
        }
        const NodeRec nd = a.nd[i];
        const double xi = resid ? __ldcg(xp + i) : 0.0, bi = __ldcs(a.rhs + i);
        // ---- incoming terms (an empty slot adds -0.0: the identity of IEEE addition)
        bool v[D];
        double tp[D], tn[D];
#pragma unroll
        for (int k = 0; k < D; ++k) {
            v[k] = UNIFORM ? ((mask >> k) & 1u) != 0u : c[k] != 0.0;
            tp[k] = v[k] ? in[k].x : -0.0;
            tn[k] = v[k] ? in[k].x * in[k].y : -0.0;  // (prec * mean), solver.py:148
        }
        // marginals of S_{s-1} (infer_marginals, solver.py:275-287) and the residual row
        double P = nd.diag, N = nd.pnum, y = nd.diag * xi;
#pragma unroll
        for (int k = 0; k < D; ++k) {
            P = P + tp[k];
            N = N + tn[k];
            const double ck = UNIFORM ? cu : c[k];
            y = y + (v[k] ? ck * xj[k] : -0.0);
        }
        bool okx;
        double x = ddiv_fast(N, P, okx);
        if (!okx) x = div_slow(N, P);
        if (!(fabs(x) <= DBL_MAX)) st.means_bad = 1u;
        __stcg(pc + i, P);
        __stcg(xc + i, x);
        if (xh) xh[i] = x;
        if (resid) {
            const double r = y - bi;
            st.rsq += r * r;
        }
        // ---- the D outgoing messages
#pragma unroll
        for (int k = 0; k < D; ++k) {
            double pe = nd.diag, num = nd.pnum;
#pragma unroll
            for (int q = 0; q < D; ++q) {
                if (q != k) {
                    pe = pe + tp[q];
                    num = num + tn[q];
                }
            }
            if (v[k]) {
                const double ck = UNIFORM ? cu : c[k];
                const double mcc = UNIFORM ? mccu : -ck * ck;
                bool okp, okm;
                double np_ = ddiv_fast(mcc, pe, okp);
                double nm = UNIFORM ? ddiv_fast_r(num, ck, rcu, okm) : ddiv_fast(num, ck, okm);
                if (!okp) np_ = div_slow(mcc, pe);
                if (!okm) nm = div_slow(num, ck);
                __stcs(mn + tws[k] + i, make_double2(np_, nm));
                const double d1 = fabs(np_ - old[k].x), d2 = fabs(nm - old[k].y);
                st.chg = fmax(st.chg, fmax(d1, d2));
                if (!(fabs(np_) <= st.lim) || !(fabs(nm) <= st.lim))
                    st.out_of_range |= (np_ != np_ || nm != nm) ? 3u : 1u;
                if (pe == 0.0) {  // the CSR id of edge i -> j (solver.py:150-154)
                    const unsigned before = UNIFORM ? __popc(mask & ((1u << k) - 1u)) : [&] {
                        unsigned b = 0u;
                        for (int q = 0; q < k; ++q) b += v[q] ? 1u : 0u;
                        return b;
                    }();
                    st.sing = min(st.sing, a.row_ptr[i] + before);
                }
            }
        }
    }
    __syncthreads();
    sweep_epilogue<kDRows, kModeSolve, 0>(T, a, s, resid, st, tid);
}

// Aggregates and marginals of S_0 (all messages +0) into ring slot 0: the same sums as a
// sweep forms them, so the +0 terms leave exactly the bits a sum over zero messages has.
template <int D>
__global__ void dia_init_kernel(const SweepArgs a) {
    const int64_t nl = a.dia_nl;
    for (int64_t i = a.dia_r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.dia_r1;
         i += (int64_t)gridDim.x * blockDim.x) {
        const NodeRec nd = a.nd[i];
        double P = nd.diag, N = nd.pnum;
#pragma unroll
        for (int k = 0; k < D; ++k)
            if (a.dia_mask ? ((a.dia_mask[i] >> k) & 1u) != 0u
                           : a.dia_coef[k * a.dia_nlc + i] != 0.0) {
                P = P + 0.0;
                N = N + 0.0 * 0.0;
            }
        a.p[0][i] = P;
        a.x[0][i] = N / P;
    }
}

// ---- build --------------------------------------------------------------------------------
// first swept row of the largest degree (its offsets are the candidate diagonals)
__global__ void dia_pick_kernel(int64_t r0, int64_t r1, const uint32_t *row_ptr, uint32_t dmax,
                                unsigned long long *row) {
    const int64_t i = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    // (a grid has millions of widest rows: only a row below the current minimum goes to the
    // atomic -- 16.8 M atomics on one word cost 5.5 ms of the 4096^2 build)
    const bool hit = i < r1 && row_ptr[i + 1] - row_ptr[i] == dmax;
    const unsigned long long cand = hit ? (unsigned long long)i : ~0ull;
    const unsigned lo = __reduce_min_sync(~0u, (unsigned)(cand & 0xffffffffull) |
                                                   (hit ? 0u : 0xffffffffu));
    // (rows of one warp are consecutive: the lowest hit lane carries the warp's minimum)
    if (hit && (unsigned)(cand & 0xffffffffull) == lo &&
        cand < *(volatile unsigned long long *)row)
        atomicMin(row, cand);
}
// every swept edge on a candidate diagonal: coef[k][i] = A_ij, else a failure flag
__global__ void dia_fill_kernel(int64_t r0, int64_t r1, int64_t nl, const uint32_t *row_ptr,
                                const EdgeRec *er, int D, DiaOffsets off, double *coef,
                                int *bad) {
    const int64_t i = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= r1) return;
    for (uint32_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
        const EdgeRec r = er[e];
        const int64_t o = (int64_t)r.col - i;
        int k = 0;
        while (k < D && off.v[k] != o) ++k;
        if (k == D) {
            *bad = 1;
            return;
        }
        coef[k * nl + i] = r.coeff;
    }
}

// every stored off-diagonal equal to the first (one value: a mask replaces the coefficients)
__global__ void dia_uniform_kernel(int64_t E, const EdgeRec *er, int *nonuniform) {
    const double c0 = er[0].coeff;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E;
         e += (int64_t)gridDim.x * blockDim.x)
        if (er[e].coeff != c0 || __double_as_longlong(er[e].coeff) != __double_as_longlong(c0)) {
            *nonuniform = 1;
            return;
        }
}
__global__ void dia_mask_kernel(int64_t r0, int64_t r1, int64_t nlc, int D, const double *coef,
                                uint8_t *mask) {
    const int64_t i = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= r1) return;
    unsigned m = 0u;
    for (int k = 0; k < D; ++k)
        if (coef[k * nlc + i] != 0.0) m |= 1u << k;
    mask[i] = (uint8_t)m;
}

inline unsigned grid_of(int64_t n) { return (unsigned)((n + 255) / 256 > 0 ? (n + 255) / 256 : 1); }

int g_dia_grid = 0;


}  // namespace

#define DCHECK(call)                                                                        \
    do {                                                                                    \
        cudaError_t _e = (call);                                                            \
        if (_e != cudaSuccess) {                                                            \
            snprintf(err, errlen, "%s: %s", #call, cudaGetErrorString(_e));                 \
            return _e == cudaErrorMemoryAllocation ? GABP_ENOMEM : GABP_ECUDA;              \
        }                                                                                   \
    } while (0)

int build_dia(DeviceGraph &g, cudaStream_t st, char *err, size_t errlen) {
    g.dia_D = 0;
    const int64_t r0 = g.row_lo, r1 = g.row_hi, nl = g.n;
    if (r1 <= r0 || g.max_degree < 1 || g.max_degree > kDiaMaxD || g.E == 0) return GABP_OK;
    if (getenv("GABP_NO_DIA")) return GABP_OK;
    // the candidate diagonals: the columns of the first widest row
    unsigned long long *d_row = nullptr;
    DCHECK(cudaMallocAsync(&d_row, sizeof(unsigned long long), st));
    DCHECK(cudaMemsetAsync(d_row, 0xff, sizeof(unsigned long long), st));
    dia_pick_kernel<<<grid_of(r1 - r0), 256, 0, st>>>(r0, r1, g.row_ptr, (uint32_t)g.max_degree,
                                                      d_row);
    unsigned long long row = 0;
    DCHECK(cudaMemcpyAsync(&row, d_row, sizeof(row), cudaMemcpyDeviceToHost, st));
    DCHECK(cudaStreamSynchronize(st));
    cudaFreeAsync(d_row, st);
    if (row == ~0ull) return GABP_OK;  // (the widest row is a halo row)
    uint32_t rp[2];
    DCHECK(cudaMemcpy(rp, g.row_ptr + row, sizeof(rp), cudaMemcpyDeviceToHost));
    const int D = (int)(rp[1] - rp[0]);
    EdgeRec rec[kDiaMaxD];
    DCHECK(cudaMemcpy(rec, g.er + rp[0], sizeof(EdgeRec) * D, cudaMemcpyDeviceToHost));
    DiaOffsets off{};
    for (int k = 0; k < D; ++k) off.v[k] = (int64_t)rec[k].col - (int64_t)row;  // ascending
    // symmetric stencil: every diagonal has its opposite; D even, at most kDiaMaxD
    int opp[kDiaMaxD];
    for (int k = 0; k < D; ++k) {
        opp[k] = -1;
        for (int q = 0; q < D; ++q)
            if (off.v[q] == -off.v[k]) opp[k] = q;
        if (opp[k] < 0) return GABP_OK;
    }
    // dense enough: padding slots cost bandwidth like edges
    const int64_t m = r1 - r0;
    if ((double)g.E < 0.6 * (double)D * (double)m) return GABP_OK;
    double *coef = nullptr;
    int *d_bad = nullptr;
    const int64_t nlc = (nl + 1) & ~1ll;  // 16-byte aligned rows for the bulk copies
    const size_t cbytes = sizeof(double) * (D * nlc + 2 * kDRows);
    DCHECK(cudaMallocAsync(&coef, cbytes, st));
    DCHECK(cudaMemsetAsync(coef, 0, cbytes, st));
    DCHECK(cudaMallocAsync(&d_bad, sizeof(int), st));
    DCHECK(cudaMemsetAsync(d_bad, 0, sizeof(int), st));
    dia_fill_kernel<<<grid_of(m), 256, 0, st>>>(r0, r1, nlc, g.row_ptr, g.er, D, off, coef, d_bad);
    DCHECK(cudaGetLastError());
    int bad = 0;
    DCHECK(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    DCHECK(cudaStreamSynchronize(st));
    cudaFreeAsync(d_bad, st);
    if (bad) {
        cudaFreeAsync(coef, st);
        return GABP_OK;
    }
    // one off-diagonal value (the Poisson grids): occupancy bits instead of coefficients
    int *d_nu = nullptr;
    DCHECK(cudaMallocAsync(&d_nu, sizeof(int), st));
    DCHECK(cudaMemsetAsync(d_nu, 0, sizeof(int), st));
    dia_uniform_kernel<<<148 * 8, 256, 0, st>>>(g.E, g.er, d_nu);
    int nonuniform = 1;
    DCHECK(cudaMemcpyAsync(&nonuniform, d_nu, sizeof(int), cudaMemcpyDeviceToHost, st));
    DCHECK(cudaStreamSynchronize(st));
    cudaFreeAsync(d_nu, st);
    if (!nonuniform) {
        const size_t mb = (size_t)nl + 2 * 256 + 16;
        DCHECK(cudaMallocAsync(&g.dia_mask, mb, st));
        DCHECK(cudaMemsetAsync(g.dia_mask, 0, mb, st));
        dia_mask_kernel<<<grid_of(m), 256, 0, st>>>(r0, r1, nlc, D, coef, g.dia_mask);
        DCHECK(cudaGetLastError());
        DCHECK(cudaMemcpy(&g.dia_cu, &g.er[0].coeff, sizeof(double), cudaMemcpyDeviceToHost));
        cudaFreeAsync(coef, st);
        coef = nullptr;
    }
    g.dia_D = D;
    g.dia_coef = coef;
    g.dia_nlc = nlc;
    int64_t O = 0;
    for (int k = 0; k < D; ++k) O = off.v[k] > O ? off.v[k] : O;
    g.dia_O = O;
    // blocked tile order for wide stencils (3-D grids): chunks of W rows of every plane
    constexpr int64_t kChunk = 16384;
    g.dia_W = (O >= 4 * kChunk && O % kChunk == 0 && m >= 2 * O) ? kChunk : 0;
    g.dia_off = off;
    for (int k = 0; k < D; ++k) g.dia_opp[k] = opp[k];
    return GABP_OK;
}

cudaError_t prepare_dia_kernels() {
    int dev = 0, sms = 0, occ = 0;
    cudaError_t e;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess)
        return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
             &occ, dia_sweep_kernel<6, false, false>, kDRows, 0)) != cudaSuccess)
        return e;
    g_dia_grid = sms * (occ > 0 ? occ : 1);
    return cudaSuccess;
}

// (a multiple of 32 elements: the padded arrays keep the 256-byte alignment other kernels'
// vector loads rely on)
int64_t dia_pad(int64_t max_off) { return (max_off + 2 * kDRows + 16 + 31) & ~31ll; }

cudaError_t launch_dia_init(const SweepArgs &a, cudaStream_t st) {
    const unsigned grid = 148 * 8;
    switch (a.dia_D) {
        case 2: dia_init_kernel<2><<<grid, 256, 0, st>>>(a); break;
        case 4: dia_init_kernel<4><<<grid, 256, 0, st>>>(a); break;
        case 6: dia_init_kernel<6><<<grid, 256, 0, st>>>(a); break;
        case 8: dia_init_kernel<8><<<grid, 256, 0, st>>>(a); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

template <int D>
void dia_launch_t(const SweepArgs &a, cudaStream_t st) {
    const int64_t nt = dia_ntiles(a);
    int64_t grid = g_dia_grid > 0 ? g_dia_grid : 148 * 2;
    if (grid > nt) grid = nt > 0 ? nt : 1;
    if (a.dia_mask)
        dia_sweep_kernel<D, true, false><<<(unsigned)grid, kDRows, 0, st>>>(a);
    else
        dia_sweep_kernel<D, false, false><<<(unsigned)grid, kDRows, 0, st>>>(a);
}

template <int D>
void dia_par_launch_t(const SweepArgs &a, cudaStream_t st) {
    const int64_t nt = dia_ntiles(a);
    int64_t grid = (g_dia_grid > 0 ? g_dia_grid : 148 * 2) / GABP_DIA_MINB * dia_par_minb(D);
    if (grid > nt) grid = nt > 0 ? nt : 1;
    if (a.dia_mask)
        dia_par_kernel<D, true><<<(unsigned)grid, kDRows, 0, st>>>(a);
    else
        dia_par_kernel<D, false><<<(unsigned)grid, kDRows, 0, st>>>(a);
}

cudaError_t launch_dia_par_sweep(const SweepArgs &a, cudaStream_t st) {
    switch (a.dia_D) {
        case 2: dia_par_launch_t<2>(a, st); break;
        case 4: dia_par_launch_t<4>(a, st); break;
        case 6: dia_par_launch_t<6>(a, st); break;
        case 8: dia_par_launch_t<8>(a, st); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_dia_sweep(const SweepArgs &a, cudaStream_t st) {
    switch (a.dia_D) {
        case 2: dia_launch_t<2>(a, st); break;
        case 4: dia_launch_t<4>(a, st); break;
        case 6: dia_launch_t<6>(a, st); break;
        case 8: dia_launch_t<8>(a, st); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace gabp
