// dense.cu -- broadcast sweep for a dense A (linear detection, BASELINE config 3).
//
// Storage: A is Kp x Kp row-major (Kp = K rounded up to 32, padding zero); messages are a
// Kp x Kp matrix M[k][j] = m_{k->j} (sender-major: the out-slot layout of the sparse path).
// The diagonal, the padding and the exact zeros of A -- non-edges in the reference
// (linalg.py:81-82) -- hold the message (P, mu) = (-0, +0): P and P mu are then -0, and
// x + (-0) == x for every x in round-to-nearest (-0 included), so the column walk adds
// every entry without an edge test and gets the reference's sums over edges bit for bit.
// (Edges start at (+0, +0), the reference's initial messages; launch_dense_init.)
// One launch s = two kernels:
//
//   column walk  one CTA per 32 columns: lane l of the summing warp walks column i0 + l in
//                ascending row order -- the incoming messages of node i in ascending sender
//                order, exactly the order of the reference's np.add.at (solver.py:242-243).
//                -- and A's column for the residual row of x^{(s-2)}.  One producer lane
//                streams the 32 x 32 blocks of A and M^{(s-1)} as 2-D tensor copies
//                (cp.async.bulk.tensor, tensor maps over the padded matrices) and the
//                x^{(s-2)} block as a 1-D bulk copy into a kColStages-deep mbarrier ring;
//                the sums are plain dependent adds (non-edges add -0, no edge test).
//                Writes P_i, P_i mu~_i, x^{(s-1)}, residual partials.
//   pair tiles   a CTA takes the tile pair (I, J), I <= J: M^{(s-1)}[I][J], M^{(s-1)}[J][I]
//                and A[I][J] (A is symmetric) are staged once, and both directions are
//                updated from them -- m_ij = f(P_i, N_i, m_ji, A_ij) and
//                m_ji = f(P_j, N_j, m_ij, A_ij) (broadcast_sweep, solver.py:249-257) -- so
//                each old message is read once, serving as one edge's previous value (the
//                change statistic) and as its twin's input; the transposed result goes out
//                through shared memory.  Max change / blowup / singular statistics; the last
//                CTA runs the solve decision for sweep s-2 (the sparse kernel's protocol).
//                (Moving the residual rows here -- the A tile is staged anyway -- cost the
//                issue-bound pair kernel 44 us per sweep at K = 4096 against 20 us of extra
//                A stream in the walk, so they stay in the walk.)
// Per edge and sweep: 24 B in the walk, 16 + 4 + 16 B in the pair tiles (was 80 B with
// one-direction tiles and a column walk without bulk copies).
#include <cuda.h>  // CUtensorMap (the encoder is fetched at run time: no libcuda link)
#include <cudaTypedefs.h>
#include <float.h>
#include <math.h>

#include "sweep_common.cuh"

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
__device__ __forceinline__ uint32_t s_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// ---- column walk -----------------------------------------------------------------------------
constexpr int kColRows = 32;     // rows of M per ring stage
constexpr int kColStages = 8;
constexpr int kColCta = 64;      // warp 0 sums, warp 1 produces

struct __align__(128) ColStage {
    double2 M[kColRows][32];
    double A[kColRows][32];
    double X[kColRows];
};
struct ColSmem {
    ColStage st[kColStages];
    uint64_t full[kColStages];
    uint64_t empty[kColStages];
    int64_t sweep;
    int skip;
};

__device__ __forceinline__ void mb_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(s_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mb_expect_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(s_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(s_u32(bar)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t *bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "DW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        " @!p bra DW_%=;\n}\n" ::"r"(s_u32(bar)),
        "r"(parity), "r"(0x989680u)
        : "memory");
}
__device__ __forceinline__ void bulk(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
        ::"r"(s_u32(dst)), "l"(src), "r"(bytes), "r"(s_u32(bar))
        : "memory");
}

struct __align__(64) DenseMaps {
    CUtensorMap A;     // Kp x Kp doubles, box 32 x 32
    CUtensorMap M[3];  // Kp x 2Kp doubles (one double2 = two columns), box 32 x 64
};

__device__ __forceinline__ void tensor2d(void *dst, const CUtensorMap *map, int x, int y,
                                         uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(s_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(s_u32(bar))
        : "memory");
}

// Column walk of launch s (solve mode).
__global__ void __launch_bounds__(kColCta, 1) dense_column_kernel(
    const SweepArgs a, const DenseArgs d, const __grid_constant__ DenseMaps maps) {
    extern __shared__ __align__(128) unsigned char col_raw[];
    ColSmem &S = *reinterpret_cast<ColSmem *>(col_raw);
    const int tid = threadIdx.x, lane = tid & 31;
    if (tid == 0) {
        volatile Ctrl *vc = a.ctrl;
        const int64_t s = vc->next_sweep;
        S.skip = vc->done || s > vc->max_iter + 2;
        S.sweep = s;
    }
    if (tid < kColStages) {
        mb_init(&S.full[tid], 1u);
        mb_init(&S.empty[tid], 1u);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    __syncthreads();
    if (S.skip) return;
    const int64_t s = S.sweep;
    const bool resid = s >= 3;
    const int64_t K = d.K;
    const CUtensorMap *mmap = &maps.M[(s - 1) % 3];
    const double *xprev = resid ? a.x[(s - 2) % 3] : nullptr;
    const int64_t i0 = (int64_t)blockIdx.x * 32;
    const int64_t nstage = d.ld / kColRows;  // padding rows hold (-0, +0) messages, A = 0
    (void)i0;

    if (tid >= 32) {  // ---- producer lane: one 2-D copy each of A and M, the x block ----
        if (lane == 0) {
            for (int64_t t = 0; t < nstage; ++t) {
                const int st = (int)(t % kColStages);
                if (t >= kColStages)
                    mb_wait(&S.empty[st], (unsigned)((t / kColStages) - 1) & 1u);
                const int64_t k0 = t * kColRows;
                const int rows = (int)((K - k0) < kColRows ? (K - k0) : kColRows);
                // x block: whole 16-byte units (x arrays carry kNodePad >= 2 doubles of padding)
                const unsigned xb = resid && rows > 0 ? (unsigned)(((rows + 1) & ~1) * 8) : 0u;
                mb_expect_tx(&S.full[st],
                             (unsigned)(sizeof(double2) * 32 * kColRows) +
                                 (resid ? (unsigned)(sizeof(double) * 32 * kColRows) + xb : 0u));
                tensor2d(&S.st[st].M[0][0], mmap, (int)(2 * i0), (int)k0, &S.full[st]);
                if (resid) {  // (no residual before launch 3)
                    tensor2d(&S.st[st].A[0][0], &maps.A, (int)i0, (int)k0, &S.full[st]);
                    if (xb) bulk(&S.st[st].X[0], xprev + k0, xb, &S.full[st]);
                }
            }
        }
        return;
    }
    // ---- summing warp: lane = column ----
    const int64_t i = i0 + lane;
    const bool col = i < K;
    double sp = 0.0, sn = 0.0, y = 0.0;
    if (col) {
        const NodeRec nd = a.nd[i];
        sp = nd.diag;
        sn = nd.pnum;
    }
    for (int64_t t = 0; t < nstage; ++t) {
        const int st = (int)(t % kColStages);
        mb_wait(&S.full[st], (unsigned)(t / kColStages) & 1u);
        const ColStage &C = S.st[st];
        const int64_t k0 = t * kColRows;
        if (resid) {
            const int rows = (int)((K - k0) < kColRows ? (K - k0) : kColRows);
#pragma unroll 16
            for (int r = 0; r < kColRows; ++r) {  // ascending k: the reference's order
                const double2 m = C.M[r][lane];  // (non-edges: -0, -0 * +0 = -0: identities)
                sp = sp + m.x;
                sn = sn + m.x * m.y;
                // residual row: sum_k A_ki x_k (A symmetric), the diagonal included; rows
                // past K have A = 0 and an unfilled x slot
                y = y + C.A[r][lane] * (r < rows ? C.X[r] : 0.0);
            }
        } else {
#pragma unroll 16
            for (int r = 0; r < kColRows; ++r) {
                const double2 m = C.M[r][lane];
                sp = sp + m.x;
                sn = sn + m.x * m.y;
            }
        }
        __syncwarp();
        if (lane == 0) mb_arrive(&S.empty[st]);
    }
    double rsq = 0.0;
    unsigned bad = 0u, agg_sing = 0xffffffffu;
    if (col) {
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

// S_0 of the dense ring: (+0, +0) on edges, (-0, +0) elsewhere.
__global__ void dense_init_kernel(const uint32_t *emask, int64_t ld, double2 *msg) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // q = k * ld + j
    if (q >= ld * ld) return;
    const int64_t k = q / ld, j = q % ld;
    const bool edge = (emask[(j >> 5) * ld + k] >> (j & 31)) & 1u;
    msg[q] = make_double2(edge ? 0.0 : -0.0, 0.0);
}

// Edge bitmask of a padded dense A: word (cb, k) bit l = A[k][32 cb + l] != 0 and k != 32 cb + l.
__global__ void dense_mask_kernel(const double *A, int64_t ld, uint32_t *emask) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // q = cb * ld + k
    const int64_t nb = ld / 32;
    if (q >= nb * ld) return;
    const int64_t cb = q / ld, k = q % ld;
    uint32_t w = 0u;
    for (int l = 0; l < 32; ++l) {
        const int64_t j = cb * 32 + l;
        if (A[k * ld + j] != 0.0 && j != k) w |= 1u << l;
    }
    emask[q] = w;
}

// ---- pair tiles -------------------------------------------------------------------------
#ifndef GABP_PAIR_CTA
#define GABP_PAIR_CTA 256
#endif
#ifndef GABP_PAIR_BUFS
#define GABP_PAIR_BUFS 2
#endif
constexpr int kPairCta = GABP_PAIR_CTA;    // 32 x kPairWarps threads
constexpr int kPairWarps = kPairCta / 32;
constexpr int kPairBufs = GABP_PAIR_BUFS;  // staged pairs: kPairBufs - 1 in flight ahead
static_assert(kPairCta % 256 == 0 && kPairCta <= 1024, "tile rows split evenly over warps");

struct __align__(16) PairBuf {
    double2 mij[kTile][kTile + 1];  // M^{(s-1)}[I][J]
    double2 mji[kTile][kTile + 1];  // M^{(s-1)}[J][I]
    double aij[kTile][kTile];       // A[I][J]
    double2 ni[kTile], nj[kTile];   // {P, N} of the rows of I and J
    uint2 ij;                       // the staged pair (I, J)
};
struct PairSmem {
    PairBuf b[kPairBufs];
    double2 out[kTile][kTile + 1];  // new M[J][I], staged for the coalesced store
    double red_d[kPairWarps];
    unsigned red_u[kPairWarps];
    uint2 next_ij[kPairBufs];       // tile pairs of the coming stagings (thread 0 writes)
    int64_t sweep;
    int skip;
    int last;
};

__device__ __forceinline__ void cpa16(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s_u32(dst)), "l"(src));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cpa_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// stage the pair (I, J) (tile indices) into buffer B
__device__ __forceinline__ void pair_stage(PairBuf &B, int64_t I, int64_t J, const DenseArgs &d,
                                           const double2 *M, int tid) {
    const int64_t ld = d.ld, i0 = I * kTile, j0 = J * kTile;
    {  // one double2 per copy: rows tid/32 + kPairWarps m, column tid % 32
        const int r0 = tid >> 5, c = tid & 31;
        const double2 *gij = M + (i0 + r0) * ld + j0 + c, *gji = M + (j0 + r0) * ld + i0 + c;
        const int64_t step = (int64_t)kPairWarps * ld;
#pragma unroll
        for (int m = 0; m < kTile / kPairWarps; ++m) {
            cpa16(&B.mij[r0 + m * kPairWarps][c], gij + m * step);
            cpa16(&B.mji[r0 + m * kPairWarps][c], gji + m * step);
        }
    }
    {  // two doubles per copy
        constexpr int RPP = kPairCta / 16;  // rows per pass
        const int r0 = tid >> 4, c = (tid & 15) * 2;
        const double *ga = d.A + (i0 + r0) * ld + j0 + c;
#pragma unroll
        for (int m = 0; m < kTile / RPP; ++m)
            cpa16(&B.aij[r0 + m * RPP][c], ga + (int64_t)m * RPP * ld);
    }
    if (tid < kTile) {
        cpa16(&B.ni[tid], d.node + i0 + tid);
        cpa16(&B.nj[tid], d.node + j0 + tid);
    }
    if (tid == 0) B.ij = make_uint2((unsigned)I, (unsigned)J);
}

struct PairStats {
    double chg = 0.0;
    unsigned oor = 0u;
    unsigned long long sing = ~0ull;
};

// Tile pair p of the upper triangle (I <= J) in row-major order: row I holds nt - I pairs,
// so pairs before row I number I nt - I (I - 1) / 2.  Computed, not loaded: a pair-list load
// sat on the critical path of every staging (10 % of the stall samples).
__device__ __forceinline__ uint2 pair_of(int64_t p, int64_t nt) {
    const double b = 2.0 * (double)nt + 1.0;
    int64_t I = (int64_t)((b - sqrt(b * b - 8.0 * (double)p)) * 0.5);
    if (I < 0) I = 0;
    auto before = [nt](int64_t i) { return i * nt - i * (i - 1) / 2; };
    while (I > 0 && before(I) > p) --I;
    while (before(I + 1) <= p) ++I;
    return make_uint2((unsigned)I, (unsigned)(I + (p - before(I))));
}

// statistics of one new message against its previous value
template <bool EXACT>
__device__ __forceinline__ void pair_stat(double2 nw, double2 old, double pe, int64_t i,
                                          int64_t j, int64_t K, double lim, PairStats &ps) {
    if (EXACT && pe == 0.0) {  // (exact pass only: the edge id is formed only here)
        const uint64_t e = (uint64_t)(i * K + j);
        if (e < ps.sing) ps.sing = e;
    }
    const double d1 = fabs(nw.x - old.x), d2 = fabs(nw.y - old.y);
    ps.chg = fmax(ps.chg, fmax(d1, d2));
    if (!(fabs(nw.x) <= lim) || !(fabs(nw.y) <= lim))
        ps.oor |= (nw.x != nw.x || nw.y != nw.y) ? 3u : 1u;  // bit 1: a NaN change
}

// The tile pair's 32 x 32 elements of one thread column (rows ty + kPairWarps m): both
// directions' new messages, stored (m_ij to global, m_ji to the transpose buffer), with
// their statistics in ps.  EXACT = false: the divisions' range tests are deferred into dr
// (no branch per element); a pair whose test fails anywhere is redone with EXACT = true,
// which also reports a zero exclusion precision (the fast path turns it into a NaN
// quotient, which fails the range test).
template <bool EXACT>
__device__ __forceinline__ void pair_elems(const PairBuf &B, PairSmem &S, double2 *Mo,
                                           int64_t ld, int64_t K, int64_t i0, int64_t j0,
                                           bool diag, int tx, int ty, double lim,
                                           PairStats &ps, DivRange &dr) {
    const int rmax = (int)(K - i0 < kTile ? K - i0 : kTile);  // rows / columns < K
    const bool jin = j0 + tx < K;
    const double2 ndj = B.nj[tx];
    double2 *orow = Mo + (i0 + ty) * ld + j0 + tx;
#pragma unroll
    for (int m = 0; m < kTile / kPairWarps; ++m) {
        const int r = ty + m * kPairWarps;
        const double c = B.aij[r][tx];
        double2 nij = make_double2(-0.0, 0.0), nji = make_double2(-0.0, 0.0);
        if (c != 0.0 && (!diag || r != tx) && r < rmax && jin) {
            // m = f(node, twin message, A) = (-c^2 / pe, (N - P_t mu_t) / c) for both
            // directions (solver.py:249-257); the two divisions by A_ij share its reciprocal
            const double2 oij = B.mij[r][tx], oji = B.mji[tx][r];
            const double2 ndi = B.ni[r];
            const double pe1 = ndi.x - oji.x, num1 = ndi.y - oji.x * oji.y;
            const double pe2 = ndj.x - oij.x, num2 = ndj.y - oij.x * oij.y;
            const double cc = -c * c;
            if (EXACT) {
                nij = make_double2(cc / pe1, num1 / c);
                nji = make_double2(cc / pe2, num2 / c);
            } else {
                const double rc = ddiv_rcp(c);
                nij = make_double2(ddiv_fast_acc(cc, pe1, dr), ddiv_fast_acc_r(num1, c, rc, dr));
                nji = make_double2(ddiv_fast_acc(cc, pe2, dr), ddiv_fast_acc_r(num2, c, rc, dr));
            }
            pair_stat<EXACT>(nij, oij, pe1, i0 + r, j0 + tx, K, lim, ps);
            if (diag)
                nji = make_double2(-0.0, 0.0);  // (the (j, i) element of the tile does it)
            else
                pair_stat<EXACT>(nji, oji, pe2, j0 + tx, i0 + r, K, lim, ps);
        }
        __stcs(orow + (int64_t)m * kPairWarps * ld, nij);
        S.out[tx][r] = nji;
    }
}

__global__ void __launch_bounds__(kPairCta) dense_pair_kernel(const SweepArgs a,
                                                              const DenseArgs d,
                                                              int64_t col_blocks) {
    extern __shared__ __align__(16) unsigned char pair_raw[];
    PairSmem &S = *reinterpret_cast<PairSmem *>(pair_raw);
    const int tid = threadIdx.x;
    Ctrl *ctrl = a.ctrl;
    const int64_t npairs = d.npairs, nt = d.ld / kTile;
    if (tid == 0) {
        volatile Ctrl *vc = ctrl;
        const int64_t s = vc->next_sweep;
        S.skip = vc->done || s > vc->max_iter + 2;
        S.sweep = s;
        // tile pairs of the first stagings (thread 0 computes, the barriers publish)
        for (int q = 0; q < kPairBufs; ++q) {
            const int64_t pq = (int64_t)blockIdx.x + (int64_t)q * gridDim.x;
            S.next_ij[q] = pq < npairs ? pair_of(pq, nt) : make_uint2(0u, 0u);
        }
    }
    __syncthreads();
    if (S.skip) return;
    const int64_t s = S.sweep;
    const int64_t K = d.K, ld = d.ld;
    const double2 *M = d.msg[(s - 1) % 3];
    double2 *Mo = d.msg[s % 3];
    const double lim = fmin(ctrl->blowup, DBL_MAX);
    PairStats ps;
    const int tx = tid & 31, ty = tid >> 5;
    int64_t p = blockIdx.x;
#pragma unroll
    for (int q = 0; q < kPairBufs - 1; ++q) {  // kPairBufs - 1 pairs in flight
        const int64_t pq = p + (int64_t)q * gridDim.x;
        if (pq < npairs) pair_stage(S.b[q], S.next_ij[q].x, S.next_ij[q].y, d, M, tid);
        cpa_commit();
    }
    for (int k = 0; p < npairs; p += gridDim.x, ++k) {
        // buffer (k-1) % kPairBufs was released by the barrier ending iteration k-1; its
        // pair indices were published by that barrier (slot (k-1) % kPairBufs of next_ij)
        const int64_t pn = p + (int64_t)(kPairBufs - 1) * gridDim.x;
        const int nb = (k + kPairBufs - 1) % kPairBufs;
        if (pn < npairs) pair_stage(S.b[nb], S.next_ij[nb].x, S.next_ij[nb].y, d, M, tid);
        cpa_commit();
        cpa_wait<kPairBufs - 1>();
        __syncthreads();  // pair p landed for every thread; next_ij[nb] read by all
        if (tid == 0) {   // indices of the pair staged next iteration into buffer nb + 1
            const int64_t pq = pn + gridDim.x;
            S.next_ij[(nb + 1) % kPairBufs] = pq < npairs ? pair_of(pq, nt) : make_uint2(0u, 0u);
        }
        const PairBuf &B = S.b[k % kPairBufs];
        const uint2 ij = B.ij;
        const int64_t I = ij.x, J = ij.y, i0 = I * kTile, j0 = J * kTile;
        const bool diag = I == J;
        PairStats pt;
        DivRange dr;
        pair_elems<false>(B, S, Mo, ld, K, i0, j0, diag, tx, ty, lim, pt, dr);
        // out complete; buffer k % kPairBufs free for the staging kPairBufs - 1 pairs ahead
        if (__syncthreads_or(!div_range_ok(dr))) {
            PairStats pe;
            DivRange dx;
            pair_elems<true>(B, S, Mo, ld, K, i0, j0, diag, tx, ty, lim, pe, dx);
            pt = pe;
            __syncthreads();
        }
        ps.chg = fmax(ps.chg, pt.chg);
        ps.oor |= pt.oor;
        ps.sing = pt.sing < ps.sing ? pt.sing : ps.sing;
        if (!diag) {
            double2 *trow = Mo + (j0 + ty) * ld + i0 + tx;
#pragma unroll
            for (int m = 0; m < kTile / kPairWarps; ++m)
                __stcs(trow + (int64_t)m * kPairWarps * ld, S.out[ty + m * kPairWarps][tx]);
        }
    }
    cpa_wait<0>();
    // CTA reductions + last-CTA decision (the sparse kernel's protocol)
    const int warp = tid >> 5, lane = tid & 31;
    double chg = warp_max_d(ps.chg);
    const unsigned oor = __reduce_or_sync(~0u, ps.oor);
    const unsigned sl = (unsigned)(ps.sing & 0xffffffffu), sh = (unsigned)(ps.sing >> 32);
    const unsigned msh = __reduce_min_sync(~0u, sh);
    const unsigned msl = __reduce_min_sync(~0u, sh == msh ? sl : 0xffffffffu);
    __syncthreads();  // (the last pair's transposed store read S.out)
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
        for (int w = 0; w < kPairWarps; ++w) {
            bc = fmax(bc, S.red_d[w]);
            f |= S.red_u[w];
        }
        const int slot = (int)(s % kStatSlots);
        if (bc > 0.0)
            atomicMax(&ctrl->change_bits[slot], (unsigned long long)__double_as_longlong(bc));
        if (f) atomicOr(&ctrl->msg_nonfinite[slot], (f & 2u) ? 3 : 1);
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
        for (int64_t b = tid; b < col_blocks; b += kPairCta) part += rp[b];
    }
    part = warp_sum_d(part);
    if (lane == 0) S.red_d[warp] = part;
    __syncthreads();
    if (tid == 0) {
        double rsq_t = 0.0;
        for (int w = 0; w < kPairWarps; ++w) rsq_t += S.red_d[w];
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

// ---- fused dense sweep: one kernel per sweep -----------------------------------------------
// The column walk and the pair tiles read every old message twice and A twice (970 MB of DRAM
// per sweep at K = 4096 against 798 MB algorithmic) in two launches.  Here one CTA owns a
// block J of 32 receivers and walks the sender blocks I = 0, 1, ... in ascending order; for
// the tile (I, J) it forms the NEW incoming messages of its receivers,
//   m_{k -> j} = (-A_kj^2 / (P_k - P_jk), (P_k x_k - P_jk mu_jk) / A_kj)     (solver.py:247-257)
// from the sender's aggregate {P_k, x_k} of S_{s-1} and the twin message m_{j -> k} -- the
// tile (J, I) read transposed -- writes them, takes the change statistic against the old tile
// (I, J), and hands them to a summing warp that adds them to the receivers' sums in ascending
// sender order (np.add.at order) together with the residual row terms A_kj x_k.  So a launch
// computes S_s, its aggregates and marginals x^{(s)}, the residual of x^{(s-1)} and decides
// sweep s-1 (the diagonal layout's protocol, dia_epilogue): per edge 16 B written, A once,
// and the old message twice -- as tile (I, J) by block J and as tile (J, I) by block I, which
// walk towards each other's tile at the same pace, so part of the second touches hit L2.
//   warps 0..7   message warps: rows 4 w .. 4 w + 3 of the tile, lane = receiver; tiles
//                staged by cp.async (L1 bypass), three tiles in flight
//   warp 8       summing warp, one tile behind: lane = receiver, 32 dependent adds per tile
constexpr int kFusedMsgWarps = 16;
constexpr int kFusedThreads = 32 * (kFusedMsgWarps + 1);
constexpr int kFusedStages = 4;
struct __align__(16) FusedStage {
    double2 own[kTile][kTile];      // M^{(s-1)}[I][J]: the old messages k -> j
    double2 twin[kTile][kTile + 1]; // M^{(s-1)}[J][I]: the twin messages j -> k (read [j][k])
    double A[kTile][kTile];         // A[I][J]
    double P[kTile], X[kTile];      // aggregates of the senders: P_k, x_k of S_{s-1}
};
struct __align__(16) FusedOut {
    double2 pn[kTile][kTile];       // new message as {P, P mu} (the sums' terms)
    double ax[kTile][kTile];        // A_kj x_k (residual row terms)
};
struct FusedSmem {
    FusedStage st[kFusedStages];
    FusedOut out[2];
    TailSmem<kFusedThreads / 32> tail;
    double srsq[kFusedThreads / 32];
    unsigned sasing[kFusedThreads / 32];
    int64_t sweep;
    int skip;
};

__device__ __forceinline__ void cpa8(void *dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s_u32(dst)), "l"(src));
}

// Per-thread source pointers of the tile copies, advanced tile by tile (the sender block
// moves down the rows of the own and A tiles and along the columns of the twin tile).
struct FusedSrc {
    const double2 *own, *twin;
    const double *A, *P, *X;
    int64_t k0;  // first sender row of the next tile to stage
};
__device__ __forceinline__ void fused_stage(FusedStage &F, FusedSrc &g, int64_t ld, int64_t K,
                                            int tid) {
    {  // one double2 per copy: rows tid / 32 + kFusedMsgWarps m, column tid % 32
        const int r0 = tid >> 5, c = tid & 31;
        const int64_t step = (int64_t)kFusedMsgWarps * ld;
#pragma unroll
        for (int m = 0; m < kTile / kFusedMsgWarps; ++m) {
            cpa16(&F.own[r0 + m * kFusedMsgWarps][c], g.own + m * step);
            cpa16(&F.twin[r0 + m * kFusedMsgWarps][c], g.twin + m * step);
        }
    }
    {  // two doubles per copy
        constexpr int RPP = 32 * kFusedMsgWarps / 16;  // rows per pass
        const int r0 = tid >> 4, c = (tid & 15) * 2;
        if (RPP >= kTile) {
            if (r0 < kTile) cpa16(&F.A[r0][c], g.A);
        } else {
#pragma unroll
            for (int m = 0; m < (kTile / RPP > 0 ? kTile / RPP : 1); ++m)
                cpa16(&F.A[r0 + m * RPP][c], g.A + (int64_t)m * RPP * ld);
        }
    }
    if (tid < kTile) {  // (rows past K: padding, their A is zero)
        if (g.k0 + tid < K) {
            cpa8(&F.P[tid], g.P);
            cpa8(&F.X[tid], g.X);
        } else {
            F.P[tid] = 0.0;
            F.X[tid] = 0.0;
        }
    }
    g.own += (int64_t)kTile * ld;
    g.twin += kTile;
    g.A += (int64_t)kTile * ld;
    g.P += kTile;
    g.X += kTile;
    g.k0 += kTile;
}

__global__ void __launch_bounds__(kFusedThreads, 1) dense_fused_kernel(const SweepArgs a,
                                                                      const DenseArgs d) {
    extern __shared__ __align__(16) unsigned char fused_raw[];
    FusedSmem &S = *reinterpret_cast<FusedSmem *>(fused_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    Ctrl *ctrl = a.ctrl;
    if (tid == 0) {
        volatile Ctrl *vc = ctrl;
        const int64_t s = vc->next_sweep;
        S.skip = vc->done || s > vc->max_iter + 1;
        S.sweep = s;
    }
    __syncthreads();
    if (S.skip) return;
    const int64_t s = S.sweep;
    const int64_t K = d.K, ld = d.ld, nt = ld / kTile;
    const double2 *M = d.msg[(s - 1) % 3];
    double2 *Mo = d.msg[s % 3];
    const double *Po = a.p[(s - 1) % 3], *Xo = a.x[(s - 1) % 3];
    const bool resid = s >= 2;
    const int64_t J = blockIdx.x, j0 = J * kTile;
    const int64_t j = j0 + lane;
    const bool msgw = warp < kFusedMsgWarps;
    Stats st;
    st.lim = fmin(ctrl->blowup, DBL_MAX);
    unsigned asing = 0xffffffffu;
    // summing warp: the receiver's running sums (prior first, solver.py:239-243)
    double sp = 0.0, sn = 0.0, y = 0.0;
    if (!msgw && j < K) {
        const NodeRec nd = a.nd[j];
        sp = nd.diag;
        sn = nd.pnum;
    }
    FusedSrc src;
    src.own = M + (int64_t)(tid >> 5) * ld + j0 + (tid & 31);
    src.twin = M + (j0 + (tid >> 5)) * ld + (tid & 31);
    src.A = d.A + (int64_t)(tid >> 4) * ld + j0 + (tid & 15) * 2;
    src.P = Po + (tid & 31);
    src.X = Xo + (tid & 31);
    src.k0 = 0;
    const bool jin = j < K;
    if (msgw) {
#pragma unroll
        for (int q = 0; q < kFusedStages - 1; ++q) {
            if (q < nt) fused_stage(S.st[q], src, ld, K, tid);
            cpa_commit();
        }
    }
    for (int64_t t = 0; t <= nt; ++t) {
        if (msgw) cpa_wait<kFusedStages - 2>();  // tile t has landed (this thread's copies)
        __syncthreads();  // ... everybody's; out[(t-1) & 1] complete; out[t & 1] and the
                          // stage of tile t - 1 are free
        if (msgw) {
            if (t + kFusedStages - 1 < nt)
                fused_stage(S.st[(t + kFusedStages - 1) % kFusedStages], src, ld, K, tid);
            cpa_commit();
            if (t < nt) {
                const FusedStage &F = S.st[t % kFusedStages];
                FusedOut &O = S.out[t & 1];
                const int64_t i0 = t * kTile;
                const bool diag = t == J;  // (the tile holds the non-edges k == j)
                const int rmax = (int)(K - i0 < kTile ? K - i0 : kTile);  // sender rows < K
                double2 *orow = Mo + (i0 + warp * (kTile / kFusedMsgWarps)) * ld + j;
#pragma unroll
                for (int r = 0; r < kTile / kFusedMsgWarps; ++r) {
                    const int k = warp * (kTile / kFusedMsgWarps) + r;
                    const double c = F.A[k][lane];
                    const double pk = F.P[k], xk = F.X[k];
                    const bool edge = c != 0.0 && jin && k < rmax && !(diag && k == lane);
                    double2 nw = make_double2(-0.0, 0.0);  // non-edges keep (-0, +0)
                    if (edge) {
                        const double2 tw = F.twin[lane][k], old = F.own[k][lane];
                        const double pe = pk - tw.x;
                        const double num = pk * xk - tw.x * tw.y;  // (sum_p * mu_tilde) - ...
                        const double cc = -c * c;                  // (-coeff * coeff)
                        bool okp, okm;
                        double np_ = ddiv_fast(cc, pe, okp);
                        double nm = ddiv_fast(num, c, okm);
                        if (!(okp && okm)) {  // (rare: a quotient outside the fast path's range)
                            np_ = div_slow(cc, pe);
                            nm = div_slow(num, c);
                        }
                        nw = make_double2(np_, nm);
                        const double d1 = fabs(np_ - old.x), d2 = fabs(nm - old.y);
                        st.chg = fmax(st.chg, fmax(d1, d2));
                        if (!(fabs(np_) <= st.lim) || !(fabs(nm) <= st.lim))
                            st.out_of_range |= (np_ != np_ || nm != nm) ? 3u : 1u;
                        if (pe == 0.0) st.sing = min(st.sing, (unsigned)((i0 + k) * K + j));
                    }
                    __stcs(orow + (int64_t)r * ld, nw);
                    O.pn[k][lane] = make_double2(nw.x, nw.x * nw.y);  // (prec * mean)
                    O.ax[k][lane] = c * xk;  // (the diagonal term included; padding: 0 * 0)
                }
            }
        } else if (t >= 1) {  // summing warp: tile t - 1, ascending senders
            const FusedOut &O = S.out[(t - 1) & 1];
#pragma unroll 8
            for (int k = 0; k < kTile; ++k) {
                const double2 v = O.pn[k][lane];
                sp = sp + v.x;
                sn = sn + v.y;
                y = y + O.ax[k][lane];
            }
        }
    }
    if (!msgw && j < K) {  // aggregates and marginal of S_s, residual row of x^{(s-1)}
        bool ok;
        double x = ddiv_fast(sn, sp, ok);
        if (!ok) x = div_slow(sn, sp);
        if (sp == 0.0) asing = (unsigned)j;  // (singular for sweep s + 1)
        if (!(fabs(x) <= DBL_MAX)) st.means_bad = 1u;
        a.p[s % 3][j] = sp;
        a.x[s % 3][j] = x;
        if (a.xhist && s >= 1 && s <= a.xhist_rows) a.xhist[(s - 1) * a.n + j] = x;
        if (resid) {
            const double r = y - a.rhs[j];
            st.rsq = r * r;
        }
    }
    if (msgw) cpa_wait<0>();
    __syncthreads();
    dia_epilogue<kFusedThreads, true>(S.tail, S.srsq, S.sasing, a, s, st, asing, 0u, tid);
}

// aggregates and marginals of S_0 (all messages zero): P_i = A_ii, x_i = A_ii mu_ii / A_ii
__global__ void dense_fused_init_kernel(const SweepArgs a, int64_t K) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= K) return;
    const NodeRec nd = a.nd[i];
    // (the sums over S_0's +0 messages leave the prior: x + (+0) == x unless x is -0)
    const double P = nd.diag + 0.0, N = nd.pnum + 0.0;
    a.p[0][i] = P;
    a.x[0][i] = N / P;
}

int g_pair_grid = 0;

// Tensor maps of the current dense buffers (re-encoded when the buffers change).
DenseMaps g_maps;
const void *g_maps_key[4] = {nullptr, nullptr, nullptr, nullptr};

cudaError_t encode_maps(const DenseArgs &d) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
        if (e != cudaSuccess || !fn) return e != cudaSuccess ? e : cudaErrorNotSupported;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint32_t elem[2] = {1, 1};
    {
        const cuuint64_t dim[2] = {(cuuint64_t)d.ld, (cuuint64_t)d.ld};
        const cuuint64_t stride[1] = {(cuuint64_t)d.ld * sizeof(double)};
        const cuuint32_t box[2] = {32, 32};
        if (encode(&g_maps.A, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(d.A), dim,
                   stride, box, elem, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
            CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    for (int b = 0; b < 3; ++b) {
        const cuuint64_t dim[2] = {(cuuint64_t)(2 * d.ld), (cuuint64_t)d.ld};
        const cuuint64_t stride[1] = {(cuuint64_t)d.ld * sizeof(double2)};
        const cuuint32_t box[2] = {64, 32};
        if (encode(&g_maps.M[b], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d.msg[b], dim, stride, box,
                   elem, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
            CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    g_maps_key[0] = d.A;
    for (int b = 0; b < 3; ++b) g_maps_key[b + 1] = d.msg[b];
    return cudaSuccess;
}

}  // namespace

cudaError_t launch_dense_mask(const double *A, int64_t ld, uint32_t *emask, cudaStream_t st) {
    const int64_t n = (ld / 32) * ld;
    dense_mask_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(A, ld, emask);
    return cudaGetLastError();
}

cudaError_t launch_dense_init(const uint32_t *emask, int64_t ld, double2 *msg, cudaStream_t st) {
    const int64_t n = ld * ld;
    dense_init_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(emask, ld, msg);
    return cudaGetLastError();
}

cudaError_t launch_dense_fused_init(const SweepArgs &a, const DenseArgs &d, cudaStream_t st) {
    dense_fused_init_kernel<<<(unsigned)((d.K + 255) / 256), 256, 0, st>>>(a, d.K);
    return cudaGetLastError();
}

cudaError_t launch_dense_fused_sweep(const SweepArgs &a, const DenseArgs &d, cudaStream_t st) {
    static bool ready = false;
    if (!ready) {
        cudaError_t e = cudaFuncSetAttribute(dense_fused_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)sizeof(FusedSmem));
        if (e != cudaSuccess) return e;
        ready = true;
    }
    dense_fused_kernel<<<(unsigned)(d.ld / kTile), kFusedThreads, sizeof(FusedSmem), st>>>(a, d);
    return cudaGetLastError();
}

cudaError_t launch_dense_sweep(const SweepArgs &a, const DenseArgs &d, cudaStream_t st) {
    if (g_maps_key[0] != d.A || g_maps_key[1] != d.msg[0] || g_maps_key[2] != d.msg[1] ||
        g_maps_key[3] != d.msg[2]) {
        cudaError_t e = encode_maps(d);
        if (e != cudaSuccess) return e;
    }
    if (g_pair_grid == 0) {
        cudaError_t e = cudaFuncSetAttribute(
            dense_column_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(ColSmem));
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(dense_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sizeof(PairSmem));
        if (e != cudaSuccess) return e;
        int dev = 0, sms = 0, occ = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, dense_pair_kernel, kPairCta,
                                                      sizeof(PairSmem));
        g_pair_grid = sms * (occ > 0 ? occ : 1);
    }
    const int64_t cb = d.ld / 32;
    dense_column_kernel<<<(unsigned)cb, kColCta, sizeof(ColSmem), st>>>(a, d, g_maps);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    int64_t grid = g_pair_grid;
    if (grid > d.npairs) grid = d.npairs;
    dense_pair_kernel<<<(unsigned)grid, kPairCta, sizeof(PairSmem), st>>>(a, d, cb);
    return cudaGetLastError();
}

}  // namespace gabp
