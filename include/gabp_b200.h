/*
 * gabp_b200.h -- C ABI of the B200-native Gaussian BP sweep library (libgabp_b200.so).
 *
 * Plain pointers and sizes only; no torch types.  Every entry point replaces one
 * function of the reference Python package (/root/reference/pkg/src/gabp); the
 * reference file:line it stands in for is cited on each declaration.  The
 * ctypes binding a maintainer of the reference would add is in INTEGRATION.md; the
 * in-tree binding is paper_0810_1119_b200/_lib.py.
 *
 * Conventions
 *   - Return value: GABP_OK (0) or a negative GABP_E* code; gabp_last_error() gives
 *     the message of the last failure on the calling thread.
 *   - Pointers named h_* are host memory, d_* are device (HBM) memory on the graph's
 *     device.  Host pointers may be pageable or pinned.
 *   - Edge ids follow the reference numbering (graph.py:84-91): directed edges grouped
 *     by source node, neighbours ascending; message arrays are indexed by edge id, so
 *     they compare element-for-element with GaussianGraph/MessageState arrays.
 *   - fp64 throughout; message updates are computed with the reference's exact
 *     operation order (no FMA contraction), so results are bitwise reproducible and
 *     match the CPU oracle bitwise.
 */
#ifndef GABP_B200_H
#define GABP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GABP_OK 0
#define GABP_EINVAL (-1)     /* bad argument / malformed system (ValueError) */
#define GABP_ECUDA (-2)      /* CUDA runtime failure */
#define GABP_ENOMEM (-3)     /* device allocation failed */
#define GABP_EZERODIAG (-4)  /* zero diagonal entry (graph.py:64-69 ZeroDiagonalError) */
#define GABP_ESINGULAR (-5)  /* P_excl == 0 in a single sweep (solver.py:34 SingularSubgraphError) */
#define GABP_EDUP (-6)       /* duplicate off-diagonal pair */

#define GABP_SCHED_PARALLEL 0  /* solver.py:146 _sweep_parallel (exclusion sums) */
#define GABP_SCHED_BROADCAST 2 /* solver.py:232 broadcast_sweep (aggregate + subtract) */

#define GABP_GATHER_AUTO 0      /* slice layout when built, else by twin-message locality */
#define GABP_GATHER_MESSAGE 1   /* row tiles, gather the twin message m_ji itself */
#define GABP_GATHER_RECOMPUTE 2 /* row tiles, broadcast only: gather node j's aggregate and
                                   recompute m_ji */
#define GABP_GATHER_SLICE 3     /* slice layout (lane per row): broadcast solve recomputes
                                   m_ji as GABP_GATHER_RECOMPUTE; parallel solve sums the
                                   row's incoming slots and stores to the twin slots */
#define GABP_GATHER_ROWS 4      /* parallel schedule: four rows per warp over the CSR order,
                                   the rows' incoming terms in a shared-memory strip, the
                                   exclusion sums from a carried prefix (rows <= 256 edges;
                                   AUTO takes it on whole graphs of mean degree >= 7).
                                   A solve whose messages exceed L2 keeps them in a binned
                                   order (built once per graph, report.message_bins; window
                                   size GABP_BIN_WINDOW_MB, default 48; GABP_ROW_NO_BIN=1
                                   keeps the CSR order).  The broadcast schedule treats this
                                   mode as GABP_GATHER_AUTO */

typedef struct gabp_graph gabp_graph_t;  /* device-resident GaussianGraph */
typedef struct gabp_state gabp_state_t;  /* device-resident MessageState  */

typedef struct {
    int64_t n;            /* unknowns */
    int64_t num_edges;    /* directed edges = 2 * off-diagonal nonzeros */
    int64_t num_tiles;    /* row tiles of the sweep kernel */
    int64_t max_degree;
    int32_t device;
    int32_t is_dense;     /* 1 for graphs made by gabp_graph_create_dense */
    double rhs_norm;      /* ||b||_2 */
    double build_ms;      /* device time of the last build (CUDA events) */
    double twin_span;     /* mean |rev(e) - e| over edges (twin-gather locality) */
    int64_t num_slices;   /* 32-row slices of the slice layout (0: not built) */
    int64_t num_slots;    /* edge slots of the slice layout, padding included */
    int32_t slice_variant;/* slice kernel: 0 register batches, 1 cp.async ring, 2 TMA ring (default) */
    int32_t dia_diagonals;/* diagonals of the stencil layout (0: not a stencil graph) */
} gabp_graph_info_t;

/* SolveOptions (solver.py:38-54) + extensions after the first four fields. */
typedef struct {
    double epsilon;           /* message-change threshold (default 1e-6) */
    int64_t max_iter;         /* sweep cap (default 10000) */
    double blowup;            /* |message| divergence bound (default 1e10) */
    int32_t schedule;         /* GABP_SCHED_PARALLEL | GABP_SCHED_BROADCAST */
    int32_t sweeps_per_poll;  /* sweeps launched (one CUDA graph) between host polls; 0 = auto */
    double rel_residual_tol;  /* extension: also stop when ||Ax-b||/||b|| < tol; <= 0 = off */
    double *h_means_history;  /* optional host [rows x n]: tentative means per sweep
                                 (SolveReport.means_history, solver.py:327-332); NULL = off */
    int64_t means_history_rows;
    int32_t gather_mode;      /* GABP_GATHER_* (results are bitwise identical in every mode) */
    int32_t reserved;
} gabp_options_t;

/* SolveReport (solver.py:77-89) scalar part; histories go to caller arrays. */
typedef struct {
    int32_t converged;
    int32_t diverged;
    int64_t iterations;       /* sweeps counted as the reference counts them */
    int64_t n_hist;           /* entries written to change/residual histories */
    int64_t sweeps_launched;  /* including speculative look-ahead sweeps */
    int64_t messages_sent;    /* MessageState.messages_sent of the final state */
    double device_ms;         /* CUDA-event time of the sweep loop */
    double final_rel_residual;/* ||Ax-b||/||b|| of the returned means */
    int64_t residual_probes;  /* residual-only launches / twin probes that decided a sweep
                                 one launch early */
    int64_t kernel_launches;  /* kernels the solve loop enqueued (incl. launches that exit at
                                 once after the decision); 0 for multi-rank solves */
    int64_t split_sweeps;     /* multi-rank: sweeps run split (boundary rows first, halo
                                 exchange under the interior rows) */
    int64_t dist_layout;      /* multi-rank kernel family agreed by the ranks: 0 none (one
                                 rank), 1 slice layout (node-state halo), 2 row tiles,
                                 3 diagonal layout (message + node-state halo) */
    int64_t message_bins;     /* parallel schedule, four-rows-per-warp kernel: bins of the binned
                                 message order the solve ran in (0: CSR order; DESIGN.md
                                 "rowquad_kernel") */
} gabp_report_t;

const char *gabp_last_error(void);
/* Gives the device memory the library keeps for reuse (released solve workspaces and
 * staging buffers of earlier graphs) back to the device; an allocation that fails does this
 * once by itself before it reports GABP_ENOMEM. */
int gabp_release_cached(int32_t device);
int gabp_version(void);
int gabp_device_count(int32_t *count);

/* ---- graph (graph.py:53-163) ------------------------------------------------------ */

/* build_graph(system) (graph.py:161; GaussianGraph.__init__ graph.py:63-120).
 * System = diag[n], rhs[n] and the upper-triangle off-diagonal pairs
 * (pair_i[p] < pair_j[p], pair_v[p] != 0) in any order (linalg.py:34-62 SymSystem).
 * Copies host arrays to the device and builds CSR + twin index there. */
int gabp_graph_create(int64_t n, int64_t npairs, const double *h_diag, const double *h_rhs,
                      const int64_t *h_pair_i, const int64_t *h_pair_j, const double *h_pair_v,
                      int32_t device, gabp_graph_t **out);

/* Same, inputs already resident in HBM (int64 pair indices). */
int gabp_graph_create_device(int64_t n, int64_t npairs, const double *d_diag,
                             const double *d_rhs, const int64_t *d_pair_i,
                             const int64_t *d_pair_j, const double *d_pair_v, int32_t device,
                             gabp_graph_t **out);

/* Same as gabp_graph_create, but only rows [row_lo, row_hi) are swept: the graph of one
 * rank's row block plus its halo rows (paper_0810_1119_b200/dist.py). */
int gabp_graph_create_ex(int64_t n, int64_t npairs, const double *h_diag, const double *h_rhs,
                         const int64_t *h_pair_i, const int64_t *h_pair_j,
                         const double *h_pair_v, int64_t row_lo, int64_t row_hi,
                         int32_t device, gabp_graph_t **out);

/* Same as gabp_graph_create_ex, inputs already resident in HBM: a rank that generates
 * or receives only its own row block (and halo) never stages the global system. */
int gabp_graph_create_device_ex(int64_t n, int64_t npairs, const double *d_diag,
                                const double *d_rhs, const int64_t *d_pair_i,
                                const int64_t *d_pair_j, const double *d_pair_v,
                                int64_t row_lo, int64_t row_hi, int32_t device,
                                gabp_graph_t **out);

/* Dense variant (linear detection, BASELINE config 3): A given as a row-major n x n
 * symmetric matrix; exact zeros off the diagonal are non-edges (linalg.py:81-82). */
int gabp_graph_create_dense(int64_t n, const double *h_a, const double *h_rhs, int32_t device,
                            gabp_graph_t **out);

void gabp_graph_destroy(gabp_graph_t *g);
int gabp_graph_info(const gabp_graph_t *g, gabp_graph_info_t *info);

/* Host copies of the graph arrays (graph.py:92-97 src/dst/coeff/rev). row_ptr[n+1],
 * col[E] (= dst), rev[E], coeff[E]; any pointer may be NULL. */
int gabp_graph_export(const gabp_graph_t *g, int64_t *h_row_ptr, int64_t *h_col,
                      int64_t *h_rev, double *h_coeff);

/* SymSystem.with_rhs (linalg.py:92-93) on a built graph. */
int gabp_graph_set_rhs(gabp_graph_t *g, const double *h_rhs);

/* The CUDA stream (cudaStream_t) all work of this graph is issued on. */
void *gabp_graph_stream(const gabp_graph_t *g);

/* ---- message state (solver.py:57-97) ---------------------------------------------- */

/* initial_state(graph) (solver.py:92-97): all messages exactly zero. */
int gabp_state_create(const gabp_graph_t *g, gabp_state_t **out);
/* MessageState.copy() (solver.py:67-74): independent device copy. */
int gabp_state_clone(const gabp_state_t *s, gabp_state_t **out);
void gabp_state_destroy(gabp_state_t *s);
int gabp_state_reset(gabp_state_t *s);
/* MessageState.prec / .mean (host copies, length num_edges); NULL skips. */
int gabp_state_read(const gabp_state_t *s, double *h_prec, double *h_mean);
int gabp_state_write(gabp_state_t *s, const double *h_prec, const double *h_mean);
int gabp_state_counters(const gabp_state_t *s, int64_t *iteration, int64_t *messages_sent);

/* sweep(graph, state, options) (solver.py:220-229) for the synchronous schedules:
 * GABP_SCHED_PARALLEL = _sweep_parallel (solver.py:146-173),
 * GABP_SCHED_BROADCAST = broadcast_sweep (solver.py:232-272).
 * On success the state advances one sweep and *max_change receives
 * max(|dP|, |dmu|).  If an exclusion (or, for broadcast, aggregate) precision is
 * exactly zero the state is left unchanged, GABP_ESINGULAR is returned and
 * *singular_index receives the first offending edge id (or node id when
 * *singular_is_node is set). */
int gabp_sweep(const gabp_graph_t *g, gabp_state_t *s, int32_t schedule, double *max_change,
               int64_t *singular_index, int32_t *singular_is_node);

/* infer_marginals(graph, state) (solver.py:275-287): means = num / prec_tot
 * (non-finite where prec_tot == 0), precisions = prec_tot. Host outputs, length n. */
/* One serial sweep (solver.py:176-217 _sweep_serial; replaces the reference's pure-Python
 * loop): in place on s, nodes in `order` (norder host int64 entries, repeats allowed; NULL =
 * ascending 0..n-1), each recomputing all its outgoing messages from its current incoming
 * ones.  Run as dependency levels (tasks on non-adjacent nodes in parallel), bitwise the
 * sequential loop.  out_of_range = some updated message is non-finite or |v| > blowup;
 * GABP_ESINGULAR with *singular_edge = the first P_excl == 0 edge in loop order, the state
 * left unchanged.  Whole graphs only; tasks of more than 256 edges keep
 * their terms in a global scratch strip instead of shared memory. */
int gabp_sweep_serial(const gabp_graph_t *g, gabp_state_t *s, const int64_t *order,
                      int64_t norder, double blowup, double *max_change, int32_t *out_of_range,
                      int64_t *singular_edge, int32_t *num_levels);
int gabp_infer_marginals(const gabp_graph_t *g, const gabp_state_t *s, double *h_means,
                         double *h_precs);

/* ---- whole-state checks and point reads ------------------------------------------ */

/* The divergence test of the solve loop on a state (solver.py:333-338): *blown = 1 when a
 * message is not finite or max |message| > blowup. */
int gabp_state_blown(const gabp_state_t *s, double blowup, int32_t *blown);
/* Messages of `count` edge ids (host list) into host arrays (either may be NULL): the
 * buffer reads of compute_message / compute_message_max_product (solver.py:100-143). */
int gabp_state_gather(const gabp_state_t *s, const int64_t *h_edges, int64_t count,
                      double *h_prec, double *h_mean);

/* ---- solve (solver.py:307-346) ---------------------------------------------------- */

/* solve(system, options) on a built graph.  Runs the sweep loop on the device with a
 * device-side convergence test (max message change, blowup, finiteness, singular
 * exclusion sums, sweep cap, optional relative residual), recording per-sweep
 * max_change and residual_norm_per_eq (linalg.py:285-288) histories.  Output arrays
 * (host) may be NULL: means/precs length n, histories length max_iter. */
int gabp_solve(gabp_graph_t *g, const gabp_options_t *opt, double *h_means, double *h_precs,
               double *h_change_hist, double *h_res_hist, gabp_report_t *rep);

/* Same, results left in device memory (d_means/d_precs length n, may be NULL). */
int gabp_solve_device(gabp_graph_t *g, const gabp_options_t *opt, double *d_means,
                      double *d_precs, gabp_report_t *rep);

/* The whole drop-in call: build_graph + solve + free, host buffers in and out. */
int gabp_solve_system(int64_t n, int64_t npairs, const double *h_diag, const double *h_rhs,
                      const int64_t *h_pair_i, const int64_t *h_pair_j,
                      const double *h_pair_v, int32_t device, const gabp_options_t *opt,
                      double *h_means, double *h_precs, double *h_change_hist,
                      double *h_res_hist, gabp_report_t *rep);

/* residual_norm_per_eq(system, x) (linalg.py:285-288): sqrt(sum (Ax-b)^2) / n. */
int gabp_residual_norm_per_eq(const gabp_graph_t *g, const double *h_x, double *out);

/* ---- multi-rank (row blocks) -------------------------------- */

/* 128-byte ncclUniqueId for gabp_dist_attach (rank 0 creates, the caller broadcasts). */
int gabp_nccl_unique_id(void *out128);

/* Make a graph built with gabp_graph_create_ex one rank of a multi-rank broadcast solve.
 * Per peer q: send_counts[q] owned local node ids (concatenated in send_idx) whose
 * aggregates and marginals the peer needs, recv_counts[q] halo local ids filled from it.
 * nccl_id == NULL: in-process partitions on one device (gabp_dist_solve_local).
 * gabp_solve on an attached graph then runs the NCCL loop and returns the owned rows. */
int gabp_dist_attach(gabp_graph_t *g, const void *nccl_id, int32_t rank, int32_t world,
                     int64_t n_global, double bnorm_global, int32_t npeers,
                     const int32_t *peers, const int64_t *send_counts, const int64_t *send_idx,
                     const int64_t *recv_counts, const int64_t *recv_idx);

/* Runs the multi-rank loop over nparts in-process partitions (rank p = parts[p]). */
int gabp_dist_solve_local(int32_t nparts, gabp_graph_t **parts, const gabp_options_t *opt,
                          double *device_ms);

/* Outputs of the last solve of a partition: owned rows of means/precs, histories. */
int gabp_dist_results(gabp_graph_t *g, const gabp_options_t *opt, double *h_means,
                      double *h_precs, double *h_change_hist, double *h_res_hist,
                      gabp_report_t *rep);

/* Sweep-kernel timing hook for bench.py: from zero messages, runs 3 untimed launches
 * (the first launches stream less than a full sweep), then `sweeps` launches of the solve
 * kernel, and returns their average device time per sweep (CUDA events on the graph
 * stream; exact twins included when a launch flags itself). */
int gabp_bench_sweeps(gabp_graph_t *g, int32_t schedule, int32_t gather_mode, int64_t sweeps,
                      double *ms_per_sweep);

/* Host-only planning hook of the one-launch cluster solve of small graphs (small.cu; no
 * device call): cuts the rows [0, n) of a CSR with host offsets row_ptr[n+1] into the row
 * blocks of the cluster's CTAs.  Returns the number of CTAs (1, 2, 4 or 8; 0 when the graph
 * does not fit a cluster and takes the launch-per-sweep kernels), block c = rows
 * [bounds[c], bounds[c+1]) in bounds[9], and the per-CTA capacities of the chosen thread
 * configuration in cap_edges / cap_rows. */
int gabp_small_plan(int64_t n, const uint32_t *row_ptr, int64_t *bounds, int64_t *cap_edges,
                    int64_t *cap_rows);

#ifdef __cplusplus
}
#endif
#endif /* GABP_B200_H */
