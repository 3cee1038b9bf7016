// gabp_internal.cuh -- device data layout and kernel interfaces of libgabp_b200.
//
// HBM layout of a built graph:
//   row_ptr   u32[n+1]   CSR offsets, edges grouped by source, neighbours ascending
//                        (= reference edge ids, graph.py:84-91)
//   er        EdgeRec[E] {rev, col, coeff}: twin edge id (graph.py:95-97), destination,
//                        A_ij -- one 16-byte record, one bulk copy per tile
//   nd        NodeRec[n] {A_ii, prior_num}: prior precision (graph.py:73) and
//                        A_ii * (b_i / A_ii) (solver.py:147)
//   diag, prior_num f64[n] the same node values as plain arrays (auxiliary kernels)
//   rhs       f64[n]
//   tile_start u32[T+1]  row tiles: <= kTileRows rows, edges bounded by kBucket + deg
// Message state: msg[3] f64x2[E] = {P, mu} per directed edge (out-slot layout:
// message i->j lives at edge id of (i->j), i.e. in row i), a ring of three sweeps.
// agg[3] f64x2[n] = {P_i, P_i * mu~_i}: node aggregates of the last states, used by the
// aggregate-recompute gathers (sweep.cu, slice.cu).
#pragma once

#include <cuda_runtime.h>
#include <float.h>
#include <stdint.h>

#include "../../include/gabp_b200.h"

namespace gabp {

#ifndef GABP_EPT
#define GABP_EPT 2
#endif
#ifndef GABP_CTAS_PER_SM
#define GABP_CTAS_PER_SM 4
#endif
#ifndef GABP_THREADS
#define GABP_THREADS 128
#endif
constexpr int kThreads = GABP_THREADS;  // threads per sweep CTA
constexpr int kTileRows = kThreads;  // max rows per tile (thread per row)
constexpr int kEPT = GABP_EPT;  // staged edges per thread per tile
constexpr int kChunk = kTileRows * kEPT;  // edges a tile may stage (fast path)
constexpr int kBucket = kChunk * 3 / 4;  // tile boundaries every kBucket edge ids (build.cu)
constexpr int kCtasPerSm = GABP_CTAS_PER_SM;
#ifndef GABP_STAGES
#define GABP_STAGES 3
#endif
constexpr int kStages = GABP_STAGES;    // contiguous-stream stage ring depth
constexpr int kNodePad = 4;     // node arrays are padded so 16-byte staging may overrun
constexpr int kStatSlots = 4;   // ring of per-sweep statistic slots
constexpr unsigned long long kNoIndex = ~0ull;  // "no singular edge/node" sentinel

enum Mode { kModeSolve = 0, kModeSingle = 1 };

// diagonal (stencil) layout, dia.cu: at most kDiaMaxD diagonals j - i = o_k, ascending
constexpr int kDiaMaxD = 8;
struct DiaOffsets {
    int64_t v[kDiaMaxD];
};

struct __align__(16) EdgeRec {
    uint32_t rev;   // id of the twin edge j -> i
    uint32_t col;   // destination node j
    double coeff;   // A_ij
};

// Per-sweep state of a node on the slice path: the aggregate precision P_i of S_t and the
// marginal x_i^{(t)} = mu~_i.  The aggregate numerator the messages use is the reference's
// rounded product (sum_p * mu_tilde) (solver.py:254): one multiplication of the two stored
// values, formed where it is used.  One node per 32-byte sector (one 256-bit gather).
// GABP_NODE16 packs two nodes per sector: measured on config 1 it halves the gather working
// set (L2 gather misses 10.4 M -> 2.5 M sectors, DRAM 2.23 -> 2.05 GB per launch) and is
// still 4 % slower (0.381 vs 0.365 ms/sweep; profiles/r02_evidence.md), so it stays a probe.
#ifdef GABP_NODE16
struct __align__(16) NodeState {
    double P, x;
};
#else
struct __align__(32) NodeState {
    double P;   // P_i = A_ii + sum_k P_ki
    double x;   // x_i = N_i / P_i (the marginal mean, mu~_i of the next sweep)
    double pad[2];
};
#endif

struct __align__(16) NodeRec {
    double diag;    // A_ii
    double pnum;    // A_ii * (b_i / A_ii)
};

// Device-resident solve controller.  One kernel launch == one sweep s (1-based).
// Launch s reads messages S_{s-1}, writes S_s, computes the marginals x^{(s-1)} of the
// state it read, and the residual of x^{(s-2)} (needs every x^{(s-2)}_j, complete only
// after launch s-1).  The decision for sweep t = s-2 is taken by the last block of
// launch s, once change_t, blowup/finiteness of S_t, finiteness of x^{(t)} and the
// residual of x^{(t)} are all known -- the reference loop body of solver.py:321-343.
struct Ctrl {
    int64_t next_sweep;  // s of the next launch
    int32_t done;
    int32_t converged;
    int32_t diverged;
    int32_t redo;        // slice path: 1 = a fast launch met a slow-path division, 2 = the
                         // exact relaunch of that sweep is pending (slice.cu)
    uint32_t ticket;     // finished-block counter of the current launch
    int64_t iterations;
    int64_t n_hist;
    int64_t final_slot;  // x/p ring slot holding the returned marginals
    double epsilon, blowup, rel_tol, bnorm;
    int64_t max_iter;
    int64_t n;
    // per-sweep statistics, slot = sweep % kStatSlots
    unsigned long long change_bits[kStatSlots];   // max |dP|,|dmu| (non-negative -> bit order)
    int32_t msg_nonfinite[kStatSlots];            // bit 0: some |message| > blowup or not
                                                  // finite; bit 1: some change is NaN
    int32_t means_nonfinite[kStatSlots];
    unsigned long long agg_singular[kStatSlots];   // broadcast: first node with P_i == 0
    unsigned long long singular_min[kStatSlots];   // first edge with P_excl == 0
    uint32_t work_twin;         // claims of an exact group twin (zeroed when redo becomes 2)
    uint32_t work[kStatSlots];  // slice TMA kernel: next work unit of launch s (slot s % 4);
                                // the last CTA of launch s zeroes slot (s + 2) % 4
    int64_t probe_t;            // slice path: sweep T whose residual the exact twin after
                                // launch T+1 computes, deciding T a launch early (0: none)
    int32_t probes;             // residual probes run (diagnostics)
    int32_t twin_launches;      // exact-twin kernels launched, host- or tail-launched (each
                                // counts itself)
    double2 *serial_msg;        // serial sweep: the message buffer the levels update in place
                                // (set per sweep, so one captured graph serves every buffer)
    uint32_t bar_count, bar_gen;  // serial sweep: grid barrier between levels
};

// A fresh controller: every "first index" slot at the kNoIndex sentinel.
inline Ctrl fresh_ctrl() {
    Ctrl c{};
    for (int k = 0; k < kStatSlots; ++k) {
        c.agg_singular[k] = kNoIndex;
        c.singular_min[k] = kNoIndex;
    }
    return c;
}

struct SweepArgs {
    int64_t n;
    int64_t ntiles;
    const uint32_t *row_ptr;
    const uint32_t *tile_start;
    const uint4 *tile_info;
    const EdgeRec *er;
    const NodeRec *nd;
    const double *diag;
    const double *prior_num;
    const double *rhs;
    double2 *msg[3];
    double2 *agg[3];
    double *x[3];
    double *p[3];
    double *rsq_part;   // [>= persistent grid] per-CTA residual partials
    double *rsq_grp;    // [groups] residual partial of each slice group (kernels that claim
                        // groups dynamically: the sum must not depend on which CTA ran one)
    Ctrl *ctrl;
    double *change_hist;
    double *res_hist;
    double *rsq_hist;
    double *xhist;        // optional [xhist_rows x n] tentative means per sweep
    int64_t xhist_rows;
    // multi-rank mode: the last CTA publishes this rank's statistics of the launch into
    // dstats ([0..4] reduced with max across ranks, [5] with sum) instead of deciding;
    // finish_kernel decides once the reduction is done (dist.cu)
    int dist;
    double *dstats;
    int msg_lag;        // message statistics of a launch refer to sweep s - msg_lag
    NodeState *rec[3];  // slice path: node state of S_t in rec[t % 3] (position order)
    int slice_variant;  // slice kernel: 0 register batches, 1 cp.async ring, 2 group TMA ring
    // slice range of this launch (whole groups; multi-rank split: boundary / interior) and
    // the offset of its CTAs' residual partials (a sweep split over launches sums the
    // partials of all of them, in CTA order)
    int64_t sl_lo, sl_hi;
    int64_t part_base;
    int exact_primary;  // the exact kernel runs as the sweep itself, not as a twin
    int slice_path;     // this launch family is the slice path (halo records)
    // slice layout (slice.cu): lane-per-row broadcast solve, nodes in position order
    int64_t nslices;
    const uint2 *slice_info;   // {slot base, width} per slice of 32 rows (group width)
    const uint32_t *gorder;    // claim order of the groups: widest first inside the boundary
                               // and the interior range (null: ascending group ids)
    const uint32_t *sdeg;      // degree per position
    const uint32_t *srow;      // local row per position (~0: padding / halo)
    const double2 *snd;        // {A_ii, A_ii mu_ii} per position
    const double *srhs;        // b_i per position
    const uint32_t *scol;      // position of the destination, per slot
    const double *scoef;       // A_ij per slot
    const uint32_t *stwin;     // slot of the twin message (parallel schedule), per slot
    // binned message order of the four-rows-per-warp parallel kernel (rowpar.cu:
    // build_bins; null: messages in CSR order)
    const uint2 *gidx;         // per edge {position of the twin message, column}
    const double *gcoef;       // per edge A_ij (a stream of its own: the kernel keeps only
                               // the two indices in registers)
    const uint32_t *gout;      // position of the edge's own message
    int quad_slots;            // rowquad_kernel: slots per lane that cover the graph's rows
                               // (2, 4, 6 or 8; rows past 8 x slots take the long-row path)
    int probe;                 // residual probe: 0 off, 1 run by the exact twin, 2 as a
                               // residual-only group launch (probe_next)
    int probe_force;           // test hook (GABP_PROBE_FORCE=1): request a probe after every
                               // launch, so every mispredicted probe path runs
    // diagonal layout (dia.cu; dia_D == 0: not built)
    int dia_D;
    int64_t dia_nl, dia_r0, dia_r1;  // node array length, swept rows
    int64_t dia_nlc;                 // coefficient row stride (nl rounded up to even)
    int64_t dia_O, dia_W;            // widest offset; blocked tile order chunk (0: identity)
    const double *dia_coef;          // [D][nlc] (non-uniform coefficients)
    const uint8_t *dia_mask;         // [nl] occupied diagonals of a row (uniform coefficient)
    double dia_cu;                   // the one off-diagonal value when dia_mask is set
    int64_t dia_off[kDiaMaxD];       // o_k, ascending
    int dia_opp[kDiaMaxD];           // diagonal of -o_k
    double2 *strip;            // serial tasks longer than kRowParMaxDegree: per-warp global
    int64_t strip_stride;      // strips of strip_stride terms (else unused)
    int twin_tail;             // group launch: the exact twin is tail-launched from the
    int twin_grid;             // device only when the launch flags itself (slice.cu)
};

// kernels (sweep.cu); prepare_sweep_kernels() must run once per device before launches
cudaError_t prepare_sweep_kernels();
int read_timeline(long long *out, int n);  // GABP_TIMELINE builds only
// gather: kGatherMessage (twin message msg_old[rev]) or kGatherRecompute (node aggregate of
// the previous state + recomputation, broadcast schedule in solve mode only)
enum Gather { kGatherMessage = 0, kGatherRecompute = 1, kGatherSlice = 2,
              kGatherSliceParallel = 3, kGatherRowParallel = 4 };
cudaError_t launch_sweep(const SweepArgs &a, int schedule, int mode, int gather, cudaStream_t st);
// parallel schedule, warp per row over the CSR order (rowpar.cu); rows of at most
// kRowParMaxDegree edges (the per-warp strip of incoming terms)
constexpr int kRowParMaxDegree = 256;
// serial tasks of more than kRowParMaxDegree edges: warps of the serial kernels (either
// launch form) that may need a global strip of SweepArgs::strip_stride terms each
int64_t serial_strip_warps();
cudaError_t prepare_rowpar_kernels();
cudaError_t launch_rowpar(const SweepArgs &a, int mode, cudaStream_t st);
// serial schedule: one dependency level of tasks {node, order position}, in place on the
// buffer a.ctrl->serial_msg
cudaError_t launch_serial_level(const SweepArgs &a, const uint2 *tasks, int64_t cnt, double lim,
                                cudaStream_t st);
cudaError_t launch_edge_col(int64_t E, const EdgeRec *er, uint32_t *col, cudaStream_t st);
// the whole serial sweep as one cooperative launch (grid barrier between levels); lvl =
// device level offsets [nlev + 1], max_cnt = the widest level
cudaError_t launch_serial_sweep(const SweepArgs &a, const uint2 *tasks, const int64_t *lvl,
                                int nlev, int64_t max_cnt, double lim, cudaStream_t st);
cudaError_t launch_marginals(int64_t n, const uint32_t *row_ptr, const EdgeRec *er,
                             const double *diag, const double *prior_num, const double2 *msg,
                             double *means, double *precs, cudaStream_t st);
cudaError_t launch_residual_sq(int64_t n, const uint32_t *row_ptr, const EdgeRec *er,
                               const double *diag, const double *rhs, const double *x,
                               double *part, int64_t nparts, double *out, cudaStream_t st);

// Controller fields a decision reads, loaded together from L2 (ld.global.cg, independent
// loads the compiler issues back to back): the decision sits on the critical path between
// two launches, where a chain of volatile loads costs ~0.3 us each.
struct CtrlSnap {
    int32_t done, msg_nonfinite, means_nonfinite;
    int64_t max_iter, n;
    unsigned long long change_bits, singular_min, agg_singular;
    double epsilon, rel_tol, bnorm;
};
__device__ __forceinline__ CtrlSnap ctrl_snap(volatile Ctrl *vc, int slot) {
    const Ctrl *c = const_cast<const Ctrl *>(vc);
    CtrlSnap r;
    r.done = __ldcg(&c->done);
    r.msg_nonfinite = __ldcg(&c->msg_nonfinite[slot]);
    r.means_nonfinite = __ldcg(&c->means_nonfinite[slot]);
    r.max_iter = (int64_t)__ldcg(reinterpret_cast<const long long *>(&c->max_iter));
    r.n = (int64_t)__ldcg(reinterpret_cast<const long long *>(&c->n));
    r.change_bits = __ldcg(&c->change_bits[slot]);
    r.singular_min = __ldcg(&c->singular_min[slot]);
    r.agg_singular = __ldcg(&c->agg_singular[slot]);
    r.epsilon = __ldcg(&c->epsilon);
    r.rel_tol = __ldcg(&c->rel_tol);
    r.bnorm = __ldcg(&c->bnorm);
    return r;
}

// Decision for sweep t (solver.py:321-345), executed by one thread of the last CTA (or of
// finish_kernel in multi-rank mode).
__device__ __forceinline__ void decide_sweep(volatile Ctrl *c, SweepArgs const &a, int64_t t, double rsq_t) {
    if (t < 1) return;
    const int slot = (int)(t % kStatSlots);
    const CtrlSnap k = ctrl_snap(c, slot);
    if (k.done || t > k.max_iter) return;
    if (k.singular_min != kNoIndex || k.agg_singular != kNoIndex) {
        // SingularSubgraphError: state not advanced, no history row (solver.py:322-326)
        c->diverged = 1;
        c->iterations = t - 1;
        c->n_hist = t - 1;
        c->final_slot = (t - 1) % 3;
        c->done = 1;
        return;
    }
    // max change; NaN when a new message is NaN, as np.max propagates it (solver.py:161-165,
    // 262-266) -- the old messages are finite in every sweep the loop still accepts
    const double change =
        (k.msg_nonfinite & 2) ? NAN : __longlong_as_double((long long)k.change_bits);
    const bool means_finite = !k.means_nonfinite;
    const double res = means_finite ? sqrt(rsq_t) / (double)k.n : INFINITY;
    a.change_hist[t - 1] = change;
    a.res_hist[t - 1] = res;
    a.rsq_hist[t - 1] = means_finite ? rsq_t : INFINITY;
    c->n_hist = t;
    c->iterations = t;
    c->final_slot = t % 3;
    if (k.msg_nonfinite || !means_finite) {  // not finite or biggest > blowup
        c->diverged = 1;
        c->done = 1;
    } else if (change < k.epsilon) {
        c->converged = 1;
        c->done = 1;
    } else if (k.rel_tol > 0.0 && sqrt(rsq_t) < k.rel_tol * k.bnorm) {
        c->converged = 1;
        c->done = 1;
    } else if (t >= k.max_iter) {
        c->diverged = 1;  // sweep cap (solver.py:344-345)
        c->done = 1;
    }
}

// Residual probe (slice path, slice.cu): at the end of launch T+1 -- after the decision
// for T-1 -- the statistics of sweep T and of x^{(T)} are complete; only the residual of
// x^{(T)} is missing, and launch T+2 would compute it alongside a whole sweep T+1 that is
// thrown away when T ends the solve.  Returns T when that decision is certain (divergence,
// singular, epsilon test, sweep cap) or when the residual test is predicted to pass
// (geometric extrapolation of the last two residuals, margin shrinking to 1 as the
// contraction rate approaches 1, where a missed prediction costs a negligible fraction of
// the solve); the next launch then computes only the residual of x^{(T)} and decides T.
// rsq_prev is the squared residual of x^{(T-1)} decided just now.
__device__ __forceinline__ int64_t probe_next(volatile Ctrl *c, SweepArgs const &a, int64_t T,
                                              double rsq_prev) {
    if (T < 1) return 0;
    const int slot = (int)(T % kStatSlots);
    const CtrlSnap k = ctrl_snap(c, slot);
    const double r2 = T >= 3 ? a.rsq_hist[T - 3] : 0.0;  // x^{(T-2)}
    if (k.done || T > k.max_iter) return 0;
    if (a.probe_force) return T;
    if (k.singular_min != kNoIndex || k.agg_singular != kNoIndex || k.msg_nonfinite ||
        k.means_nonfinite || T >= k.max_iter)
        return T;
    if (__longlong_as_double((long long)k.change_bits) < k.epsilon) return T;
    if (k.rel_tol > 0.0 && T >= 3) {
        const double r1 = rsq_prev;  // x^{(T-1)}
        if (r2 > 0.0 && r1 <= DBL_MAX && r2 <= DBL_MAX) {
            const double rho2 = fmin(r1 / r2, 1.0);  // squared contraction per sweep
            const double m = 1.0 + 0.5 * (1.0 - sqrt(rho2));
            const double lim = k.rel_tol * k.bnorm;
            if (r1 * rho2 < lim * lim * m * m) return T;
        }
    }
    return 0;
}

// dense variant (dense.cu): A row-major K x K, messages a padded K x K matrix ring
struct DenseArgs {
    int64_t K;
    int64_t ld;      // leading dimension: K rounded up to 32 (A, msg and node are padded)
    const double *A;
    double2 *msg[3];
    double2 *node;   // {P_i, P_i mu~_i} of the state read by the launch
    const uint2 *pairs;  // upper-triangle tile pairs (I <= J) of the pair-tile kernel
    int64_t npairs;
    const uint32_t *emask;  // [ld/32][ld]: bit l of word (cb, k) = A[k][32 cb + l] is an edge
};
cudaError_t launch_dense_sweep(const SweepArgs &a, const DenseArgs &d, cudaStream_t st);
// one kernel per sweep (dense_fused_kernel): launch protocol of the diagonal layout
cudaError_t launch_dense_fused_init(const SweepArgs &a, const DenseArgs &d, cudaStream_t st);
cudaError_t launch_dense_fused_sweep(const SweepArgs &a, const DenseArgs &d, cudaStream_t st);
cudaError_t launch_dense_mask(const double *A, int64_t ld, uint32_t *emask, cudaStream_t st);
cudaError_t launch_dense_init(const uint32_t *emask, int64_t ld, double2 *msg, cudaStream_t st);

// |message| maximum of a state as an ordered bit pattern (NaN > +inf > finite), state.cu
cudaError_t launch_absmax(int64_t E, const double2 *a, unsigned long long *d_out,
                          cudaStream_t st);
cudaError_t launch_gather(int64_t cnt, const int64_t *idx, const double2 *m, double2 *out,
                          cudaStream_t st);

// the broadcast solve on the diagonal layout (dia.cu): build_dia after the CSR (a no-op
// unless every edge lies on one of <= kDiaMaxD symmetric diagonals); launch_dia_init forms
// the aggregates of S_0 in ring slot 0, then one launch_dia_sweep per sweep
cudaError_t prepare_dia_kernels();
cudaError_t launch_dia_init(const SweepArgs &a, cudaStream_t st);
cudaError_t launch_dia_sweep(const SweepArgs &a, cudaStream_t st);
// the parallel schedule on the diagonal layout (launch protocol of the CSR kernels: no init,
// max_iter + 2 launches, decision of sweep s-2 in launch s)
cudaError_t launch_dia_par_sweep(const SweepArgs &a, cudaStream_t st);
// elements of padding the diagonal kernel needs on both sides of the message and node-state
// arrays (every staged range in bounds)
int64_t dia_pad(int64_t max_off);

// the whole broadcast solve of a small graph in one launch of one thread-block cluster
// (small.cu): messages and node states in the distributed shared memory of <= 8 CTAs
constexpr int kSmallMaxCluster = 8;
struct SmallPart {
    int C;                              // CTAs in the cluster
    int cfg;                            // thread configuration (small.cu: kSmallCfg)
    uint32_t nb[kSmallMaxCluster + 1];  // CTA c owns rows [nb[c], nb[c+1])
};
bool small_candidate(int64_t n, int64_t E);  // sizes a cluster could hold at all
bool small_plan(int64_t n, const uint32_t *row_ptr, SmallPart *out);
void small_capacity(int cfg, int64_t *edges, int64_t *rows);
cudaError_t launch_small_solve(const SweepArgs &a, const SmallPart &p, bool parallel,
                               cudaStream_t st);

// multi-rank helpers (dist.cu)
cudaError_t launch_finish(const SweepArgs &a, cudaStream_t st);
// diagonal layout across ranks: the decision for sweep s-1 after launch s, and the halo of
// {P, x} plus the incoming messages on the diagonals that cross to a peer
struct DiaHalo {
    int nd;                 // diagonals exchanged with this peer
    int diag[kDiaMaxD];
};
cudaError_t launch_dia_finish(const SweepArgs &a, cudaStream_t st);
cudaError_t launch_dia_pack(const SweepArgs &a, const uint32_t *idx, int64_t cnt, double *buf,
                            const DiaHalo &h, int64_t s_fix, int post_finish, cudaStream_t st);
cudaError_t launch_dia_unpack(const SweepArgs &a, const uint32_t *idx, int64_t cnt,
                              const double *buf, const DiaHalo &h, int64_t s_fix,
                              int post_finish, cudaStream_t st);
// pre_finish = 1: called between the sweep launch and its finish_kernel (split sweep)
cudaError_t launch_halo_pack(const SweepArgs &a, const uint32_t *idx, int64_t cnt, double *buf,
                             cudaStream_t st, int pre_finish);
cudaError_t launch_halo_unpack(const SweepArgs &a, const uint32_t *idx, int64_t cnt,
                               const double *buf, cudaStream_t st, int pre_finish);

// graph build (build.cu)
struct DeviceGraph {
    int64_t n = 0, E = 0, npairs = 0, ntiles = 0, max_degree = 0;
    int device = 0;
    uint32_t *row_ptr = nullptr;
    uint32_t *tile_start = nullptr;
    uint4 *tile_info = nullptr;   // {r0, r1, e0, e1} per tile
    EdgeRec *er = nullptr;
    NodeRec *nd = nullptr;
    double *diag = nullptr;
    double *prior_num = nullptr;
    double *rhs = nullptr;
    double rhs_norm = 0.0;
    double build_ms = 0.0;
    double twin_span = 0.0;  // mean |rev(e) - e| in edges: locality of the twin gather
    int64_t row_lo = 0, row_hi = 0;  // swept rows
    // slice layout (build_slices, slice.cu); nslices == 0 when not built
    int64_t nslices = 0, nslots = 0, npos = 0;
    int64_t bnd_groups = 0;     // multi-rank: leading groups holding the boundary rows
    int slice_variant = 2;      // 0: register batches, 1: cp.async ring, 2: group TMA ring
    uint2 *slice_info = nullptr;
    uint32_t *gorder = nullptr; // groups by width, descending (claim order of the TMA kernels)
    uint32_t *pos = nullptr;    // local row -> position
    uint32_t *srow = nullptr, *sdeg = nullptr;
    double2 *snd = nullptr;
    double *srhs = nullptr;
    uint32_t *scol = nullptr;
    double *scoef = nullptr;
    uint32_t *stwin = nullptr;  // built on the first parallel-schedule solve (build_stwin)
    // binned message order (rowpar.cu: build_bins), built on the first solve that uses it
    uint2 *gidx = nullptr;
    double *gcoef = nullptr;
    uint32_t *gout = nullptr;
    int bins = 0;               // 0: not tried, -1: not worth it (messages fit L2), else count
    int64_t rows_gt16 = 0, rows_gt32 = 0, rows_gt48 = 0;  // rows of more than 16 / 32 / 48
                                                          // edges (rowquad_kernel)
    // diagonal layout (build_dia, dia.cu); dia_D == 0 when the graph is not a stencil
    int dia_D = 0;
    int64_t dia_nlc = 0, dia_O = 0, dia_W = 0;
    double *dia_coef = nullptr;
    uint8_t *dia_mask = nullptr;  // uniform coefficient dia_cu: occupancy bits per row
    double dia_cu = 0.0;
    DiaOffsets dia_off{};
    int dia_opp[kDiaMaxD] = {};
};

// Builds CSR + twin index + tiles from device-resident inputs.  Returns a GABP_* code
// and fills *err with a message on failure.
// Only rows [row_lo, row_hi) are swept (a rank's owned block; the rest are halo rows).
int build_graph_device(DeviceGraph &g, int64_t n, int64_t npairs, const double *d_diag,
                       const double *d_rhs, const int64_t *d_pi, const int64_t *d_pj,
                       const double *d_pv, int64_t row_lo, int64_t row_hi, cudaStream_t st,
                       char *err, size_t errlen, cudaEvent_t idx_ready = nullptr,
                       cudaEvent_t val_ready = nullptr);
void free_graph(DeviceGraph &g, cudaStream_t st);
// slice layout of the swept rows (slice.cu); GABP_OK or an error (the tile layout stays)
int build_slices(DeviceGraph &g, cudaStream_t st, char *err, size_t errlen);
int build_dia(DeviceGraph &g, cudaStream_t st, char *err, size_t errlen);
cudaError_t prepare_slice_kernels();
cudaError_t launch_slice_sweep(const SweepArgs &a, cudaStream_t st);
cudaError_t launch_slice_part(const SweepArgs &a, int reserve_sms, cudaStream_t st);
cudaError_t launch_slice_boundary(const SweepArgs &a, int64_t *grid, cudaStream_t st);
// parallel schedule over the slice groups (slice.cu); build_stwin first
cudaError_t launch_slice_parallel(const SweepArgs &a, cudaStream_t st);
int build_stwin(DeviceGraph &g, cudaStream_t st, char *err, size_t errlen);
// binned message order for rowquad_kernel (rowpar.cu); g.bins < 0 afterwards: not used
int build_bins(DeviceGraph &g, cudaStream_t st, char *err, size_t errlen);
cudaError_t refresh_slice_nodes(const DeviceGraph &g, cudaStream_t st);
cudaError_t slice_to_rows(const DeviceGraph &g, int64_t lo, int64_t cnt, const double *in,
                          int stride, double *out, cudaStream_t st);
cudaError_t slice_map_index(const DeviceGraph &g, uint32_t *idx, int64_t cnt, cudaStream_t st);
constexpr int64_t kSliceMaxDegree = 4096;  // rows longer than this: tile layout only
constexpr int64_t kSlotPad = 4096;         // slot arrays are padded by 8 group columns
int compute_priors(DeviceGraph &g, cudaStream_t st, char *err, size_t errlen);

}  // namespace gabp
