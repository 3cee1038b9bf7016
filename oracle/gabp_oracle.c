/*
 * gabp_oracle.c -- CPU ORACLE for the GaBP sweep hot path.  TEST INFRASTRUCTURE.
 *
 * This file is the checker, never the product: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The product path
 * (paper_0810_1119_b200/) runs on the CUDA library and fails loudly without it.
 *
 * It is a plain-C restatement of the reference Python package
 * (/root/reference/pkg/src/gabp, numpy-based) for the synchronous sweep path:
 *
 *   graph build   graph.py:63-120   GaussianGraph.__init__: CSR grouped by source,
 *                                  neighbours ascending, rev[] twin index, coeff[]
 *   parallel      solver.py:146-173 _sweep_parallel: exclusion sums accumulated in
 *                                  ascending-k order (np.add.at over excl_edge)
 *   broadcast     solver.py:232-272 broadcast_sweep: node aggregate then subtraction
 *   serial        solver.py:176-217 _sweep_serial: in place, node by node in the given
 *                                  order (sequential; single thread)
 *   marginals     solver.py:275-287 infer_marginals
 *   residual      linalg.py:285-288 residual_norm_per_eq (row-wise summation order;
 *                                  the reference sums in dict order -> differs in
 *                                  the last bits only; tests compare with tolerance)
 *   solve loop    solver.py:307-346 solve(), plus one extension: an optional relative
 *                                  residual stop ||Ax-b||/||b|| < rel_residual_tol
 *
 * Floating point: every message is computed with the same operation sequence as the
 * numpy reference (no FMA contraction: build with -ffp-contract=off), so message
 * buffers, marginals and max_change agree BITWISE with the reference; this is pinned
 * against the tests/golden fixtures produced by running the reference itself
 * (tests/golden/make_golden.py).
 *
 * OpenMP parallelises over nodes/edges.  Every per-edge/per-node value is computed
 * by one thread in a fixed order, and the residual sum uses fixed 4096-row chunks
 * summed in chunk order, so results do not depend on the thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_EINVAL 1
#define ORC_ENOMEM 2

/* ------------------------------------------------------------------------- */
/* graph build (graph.py:63-120)                                             */
/* ------------------------------------------------------------------------- */

typedef struct {
    int64_t key_col;
    int64_t payload; /* 2*pair + direction */
} orc_slot;

static int cmp_slot(const void *a, const void *b) {
    const orc_slot *x = (const orc_slot *)a, *y = (const orc_slot *)b;
    return (x->key_col > y->key_col) - (x->key_col < y->key_col);
}

/* Upper-triangle pairs (pi[p] < pj[p], value pv[p]) in any order -> directed CSR:
 * row_ptr[n+1], col[E], rev[E], coeff[E] with E = 2*npairs.  Edge ids grouped by
 * source node, neighbours ascending (graph.py:84-91); rev[e] = id of (j -> i)
 * (graph.py:95-97).  Returns ORC_EINVAL on a bad or duplicated pair. */
int oracle_build_graph(int64_t n, int64_t npairs, const int64_t *pi, const int64_t *pj,
                       const double *pv, int64_t *row_ptr, int64_t *col, int64_t *rev,
                       double *coeff) {
    int64_t E = 2 * npairs;
    memset(row_ptr, 0, sizeof(int64_t) * (size_t)(n + 1));
    for (int64_t p = 0; p < npairs; ++p) {
        if (!(0 <= pi[p] && pi[p] < pj[p] && pj[p] < n)) return ORC_EINVAL;
        if (pv[p] == 0.0) return ORC_EINVAL;
        row_ptr[pi[p] + 1]++;
        row_ptr[pj[p] + 1]++;
    }
    for (int64_t i = 0; i < n; ++i) row_ptr[i + 1] += row_ptr[i];
    int64_t *cursor = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    orc_slot *slots = (orc_slot *)malloc(sizeof(orc_slot) * (size_t)(E > 0 ? E : 1));
    int64_t *pos = (int64_t *)malloc(sizeof(int64_t) * (size_t)(E > 0 ? E : 1));
    if (!cursor || !slots || !pos) {
        free(cursor); free(slots); free(pos);
        return ORC_ENOMEM;
    }
    memcpy(cursor, row_ptr, sizeof(int64_t) * (size_t)n);
    for (int64_t p = 0; p < npairs; ++p) {
        int64_t a = cursor[pi[p]]++;
        slots[a].key_col = pj[p];
        slots[a].payload = 2 * p;       /* i -> j */
        int64_t b = cursor[pj[p]]++;
        slots[b].key_col = pi[p];
        slots[b].payload = 2 * p + 1;   /* j -> i */
    }
    int bad = 0;
#pragma omp parallel for schedule(dynamic, 1024) reduction(| : bad)
    for (int64_t i = 0; i < n; ++i) {
        int64_t s = row_ptr[i], e = row_ptr[i + 1];
        qsort(slots + s, (size_t)(e - s), sizeof(orc_slot), cmp_slot);
        for (int64_t q = s + 1; q < e; ++q)
            if (slots[q].key_col == slots[q - 1].key_col) bad = 1; /* duplicate pair */
    }
    if (bad) {
        free(cursor); free(slots); free(pos);
        return ORC_EINVAL;
    }
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < E; ++e) {
        col[e] = slots[e].key_col;
        pos[slots[e].payload] = e;
    }
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < E; ++e) {
        int64_t pl = slots[e].payload;
        rev[e] = pos[pl ^ 1];
        coeff[e] = pv[pl >> 1];
    }
    free(cursor); free(slots); free(pos);
    return ORC_OK;
}

/* prior_num = prior_prec * prior_mean with prior_mean = rhs / diag (graph.py:73-74,
 * solver.py:147). */
void oracle_priors(int64_t n, const double *diag, const double *rhs, double *prior_num) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        double pm = rhs[i] / diag[i];
        prior_num[i] = diag[i] * pm;
    }
}

/* ------------------------------------------------------------------------- */
/* sweeps                                                                    */
/* ------------------------------------------------------------------------- */

typedef struct {
    double max_change;   /* max(|dP|, |dmu|) as solver.py:160-163 (NaN propagates) */
    int64_t singular;    /* first offending edge (parallel/broadcast) or node (agg), -1 */
    int singular_is_node;
} orc_sweep_out;

static inline double nanmax(double a, double b) {
    if (a != a) return a;
    if (b != b) return b;
    return a > b ? a : b;
}

/* _sweep_parallel (solver.py:146-173): P_ij = -A_ij^2 / P_i\j, mu_ij = num_i\j / A_ij,
 * exclusion sums accumulated in ascending-k order over N(i) \ j. */
void oracle_sweep_parallel(int64_t n, const int64_t *row_ptr, const int64_t *col,
                           const int64_t *rev, const double *coeff, const double *prior_prec,
                           const double *prior_num, const double *prec, const double *mean,
                           double *prec_out, double *mean_out, orc_sweep_out *out) {
    double mc = 0.0;
    int64_t sing = INT64_MAX;
    (void)col;
#pragma omp parallel
    {
        double lmc = 0.0;
        int64_t lsing = INT64_MAX;
#pragma omp for schedule(dynamic, 256)
        for (int64_t i = 0; i < n; ++i) {
            int64_t s = row_ptr[i], t = row_ptr[i + 1];
            for (int64_t e = s; e < t; ++e) {
                double p_excl = prior_prec[i];
                double num = prior_num[i];
                for (int64_t q = s; q < t; ++q) {
                    if (q == e) continue;
                    int64_t r = rev[q]; /* incoming edge (k -> i) */
                    p_excl += prec[r];
                    num += prec[r] * mean[r];
                }
                if (p_excl == 0.0 && e < lsing) lsing = e;
                double c = coeff[e];
                double np_ = -c * c / p_excl;
                double nm = num / c;
                prec_out[e] = np_;
                mean_out[e] = nm;
                lmc = nanmax(lmc, fabs(np_ - prec[e]));
                lmc = nanmax(lmc, fabs(nm - mean[e]));
            }
        }
#pragma omp critical
        {
            mc = nanmax(mc, lmc);
            if (lsing < sing) sing = lsing;
        }
    }
    out->max_change = mc;
    out->singular = sing == INT64_MAX ? -1 : sing;
    out->singular_is_node = 0;
}

/* _sweep_serial (solver.py:176-217): in place, nodes in `order` (NULL = 0..n-1); node i
 * recomputes every outgoing message from its current incoming ones (exclusion sums in
 * ascending neighbour order, solver.py:188-197).  Stops at the first P_excl == 0 edge in
 * loop order (the reference raises there) and reports it. */
void oracle_sweep_serial(int64_t n, const int64_t *row_ptr, const int64_t *rev,
                         const double *coeff, const double *prior_prec, const double *prior_num,
                         double *prec, double *mean, const int64_t *order, int64_t norder,
                         orc_sweep_out *out) {
    double mc = 0.0;
    out->singular = -1;
    out->singular_is_node = 0;
    if (!order) norder = n;
    for (int64_t t = 0; t < norder; ++t) {
        const int64_t i = order ? order[t] : t;
        const int64_t s = row_ptr[i], u = row_ptr[i + 1];
        for (int64_t e = s; e < u; ++e) {
            double acc_p = prior_prec[i];
            double acc_num = prior_num[i];
            for (int64_t q = s; q < u; ++q) {
                if (q == e) continue;
                const int64_t r = rev[q]; /* incoming edge (k -> i), current value */
                acc_p += prec[r];
                acc_num += prec[r] * mean[r];
            }
            if (acc_p == 0.0) {
                out->singular = e;
                out->max_change = mc;
                return;
            }
            const double c = coeff[e];
            const double np_ = -c * c / acc_p;
            const double nm = acc_num / c;
            const double dp = fabs(np_ - prec[e]), dm = fabs(nm - mean[e]);
            if (dp > mc) mc = dp; /* solver.py:204-207: plain '>' (NaN never wins) */
            if (dm > mc) mc = dm;
            prec[e] = np_;
            mean[e] = nm;
        }
    }
    out->max_change = mc;
}

/* node aggregates shared by broadcast_sweep (solver.py:240-243) and infer_marginals
 * (solver.py:281-284): sum_p = P_ii + sum_k P_ki, sum_num = P_ii mu_ii + sum_k P_ki mu_ki,
 * incoming edges in edge-id order == ascending source k. */
static inline void node_aggregate(int64_t i, const int64_t *row_ptr, const int64_t *rev,
                                  const double *prior_prec, const double *prior_num,
                                  const double *prec, const double *mean, double *sp,
                                  double *sn) {
    double p = prior_prec[i], m = prior_num[i];
    for (int64_t q = row_ptr[i]; q < row_ptr[i + 1]; ++q) {
        int64_t r = rev[q];
        p += prec[r];
        m += prec[r] * mean[r];
    }
    *sp = p;
    *sn = m;
}

/* broadcast_sweep (solver.py:232-272). node_p/node_n are scratch of length n. */
void oracle_sweep_broadcast(int64_t n, const int64_t *row_ptr, const int64_t *col,
                            const int64_t *rev, const double *coeff, const double *prior_prec,
                            const double *prior_num, const double *prec, const double *mean,
                            double *prec_out, double *mean_out, double *node_p, double *node_n,
                            orc_sweep_out *out) {
    int64_t sing_node = INT64_MAX;
    (void)col;
#pragma omp parallel for schedule(static) reduction(min : sing_node)
    for (int64_t i = 0; i < n; ++i) {
        double sp, sn;
        node_aggregate(i, row_ptr, rev, prior_prec, prior_num, prec, mean, &sp, &sn);
        if (sp == 0.0 && i < sing_node) sing_node = i;
        double mu_tilde = sn / sp;
        node_p[i] = sp;
        node_n[i] = sp * mu_tilde;
    }
    if (sing_node != INT64_MAX) {
        out->max_change = 0.0;
        out->singular = sing_node;
        out->singular_is_node = 1;
        return;
    }
    double mc = 0.0;
    int64_t sing = INT64_MAX;
#pragma omp parallel
    {
        double lmc = 0.0;
        int64_t lsing = INT64_MAX;
#pragma omp for schedule(static)
        for (int64_t i = 0; i < n; ++i) {
            for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
                int64_t r = rev[e];
                double p_excl = node_p[i] - prec[r];
                if (p_excl == 0.0 && e < lsing) lsing = e;
                double num = node_n[i] - prec[r] * mean[r];
                double c = coeff[e];
                double np_ = -c * c / p_excl;
                double nm = num / c;
                prec_out[e] = np_;
                mean_out[e] = nm;
                lmc = nanmax(lmc, fabs(np_ - prec[e]));
                lmc = nanmax(lmc, fabs(nm - mean[e]));
            }
        }
#pragma omp critical
        {
            mc = nanmax(mc, lmc);
            if (lsing < sing) sing = lsing;
        }
    }
    out->max_change = mc;
    out->singular = sing == INT64_MAX ? -1 : sing;
    out->singular_is_node = 0;
}

/* infer_marginals (solver.py:275-287): means = num / prec_tot (may be non-finite). */
void oracle_marginals(int64_t n, const int64_t *row_ptr, const int64_t *rev,
                      const double *prior_prec, const double *prior_num, const double *prec,
                      const double *mean, double *means, double *precs) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        double sp, sn;
        node_aggregate(i, row_ptr, rev, prior_prec, prior_num, prec, mean, &sp, &sn);
        means[i] = sn / sp;
        precs[i] = sp;
    }
}

/* sum_i (A x - b)_i^2, rows in CSR order, fixed 4096-row chunks summed in order. */
double oracle_residual_sq(int64_t n, const int64_t *row_ptr, const int64_t *col,
                          const double *coeff, const double *diag, const double *rhs,
                          const double *x) {
    int64_t nchunk = (n + 4095) / 4096;
    double *part = (double *)calloc((size_t)(nchunk > 0 ? nchunk : 1), sizeof(double));
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < nchunk; ++c) {
        double acc = 0.0;
        int64_t hi = (c + 1) * 4096 < n ? (c + 1) * 4096 : n;
        for (int64_t i = c * 4096; i < hi; ++i) {
            double y = diag[i] * x[i];
            for (int64_t q = row_ptr[i]; q < row_ptr[i + 1]; ++q) y += coeff[q] * x[col[q]];
            double r = y - rhs[i];
            acc += r * r;
        }
        part[c] = acc;
    }
    double s = 0.0;
    for (int64_t c = 0; c < nchunk; ++c) s += part[c];
    free(part);
    return s;
}

/* ------------------------------------------------------------------------- */
/* solve loop (solver.py:307-346)                                            */
/* ------------------------------------------------------------------------- */

typedef struct {
    double epsilon;
    int64_t max_iter;
    double blowup;
    int schedule;            /* 0 = parallel, 2 = broadcast */
    double rel_residual_tol; /* <= 0: off (reference behaviour) */
} orc_options;

typedef struct {
    int converged, diverged;
    int64_t iterations;
    int64_t n_hist;          /* rows written to the history arrays */
} orc_report;

/* Runs the reference solve loop.  means/precs (n) receive the marginals of the final
 * state; change_hist/res_hist (max_iter) receive per-sweep max_change and
 * residual_norm_per_eq (sqrt(sum r^2) / n, linalg.py:285-288). */
int oracle_solve(int64_t n, const int64_t *row_ptr, const int64_t *col, const int64_t *rev,
                 const double *coeff, const double *diag, const double *rhs,
                 const orc_options *opt, double *means, double *precs, double *change_hist,
                 double *res_hist, orc_report *rep) {
    int64_t E = row_ptr[n];
    size_t eb = sizeof(double) * (size_t)(E > 0 ? E : 1);
    size_t nb = sizeof(double) * (size_t)(n > 0 ? n : 1);
    double *p0 = (double *)calloc(1, eb), *m0 = (double *)calloc(1, eb);
    double *p1 = (double *)malloc(eb), *m1 = (double *)malloc(eb);
    double *prior_num = (double *)malloc(nb), *node_p = (double *)malloc(nb),
           *node_n = (double *)malloc(nb), *xs = (double *)malloc(nb), *ps = (double *)malloc(nb);
    if (!p0 || !m0 || !p1 || !m1 || !prior_num || !node_p || !node_n || !xs || !ps) {
        free(p0); free(m0); free(p1); free(m1); free(prior_num); free(node_p);
        free(node_n); free(xs); free(ps);
        return ORC_ENOMEM;
    }
    oracle_priors(n, diag, rhs, prior_num);
    double bnorm = 0.0;
    for (int64_t i = 0; i < n; ++i) bnorm += rhs[i] * rhs[i];
    bnorm = sqrt(bnorm);
    int converged = 0, diverged = 0;
    int64_t iters = 0, nh = 0;
    for (int64_t it = 0; it < opt->max_iter; ++it) {
        orc_sweep_out so;
        if (opt->schedule == 2)
            oracle_sweep_broadcast(n, row_ptr, col, rev, coeff, diag, prior_num, p0, m0, p1, m1,
                                   node_p, node_n, &so);
        else
            oracle_sweep_parallel(n, row_ptr, col, rev, coeff, diag, prior_num, p0, m0, p1, m1,
                                  &so);
        if (so.singular >= 0) { /* SingularSubgraphError: state not advanced */
            diverged = 1;
            break;
        }
        double *t;
        t = p0; p0 = p1; p1 = t;
        t = m0; m0 = m1; m1 = t;
        iters++;
        oracle_marginals(n, row_ptr, rev, diag, prior_num, p0, m0, xs, ps);
        int means_finite = 1, finite = 1;
        double biggest = 0.0;
        for (int64_t i = 0; i < n; ++i)
            if (!isfinite(xs[i])) { means_finite = 0; break; }
        for (int64_t e = 0; e < E; ++e) {
            if (!isfinite(p0[e]) || !isfinite(m0[e])) finite = 0;
            double a = fabs(p0[e]), b = fabs(m0[e]);
            if (a > biggest) biggest = a;
            if (b > biggest) biggest = b;
        }
        double rsq = means_finite ? oracle_residual_sq(n, row_ptr, col, coeff, diag, rhs, xs)
                                  : INFINITY;
        change_hist[nh] = so.max_change;
        res_hist[nh] = means_finite ? sqrt(rsq) / (double)n : INFINITY;
        nh++;
        if (!finite || biggest > opt->blowup || !means_finite) {
            diverged = 1;
            break;
        }
        if (so.max_change < opt->epsilon) {
            converged = 1;
            break;
        }
        if (opt->rel_residual_tol > 0.0 && sqrt(rsq) < opt->rel_residual_tol * bnorm) {
            converged = 1;
            break;
        }
    }
    if (!converged && !diverged) diverged = 1;
    oracle_marginals(n, row_ptr, rev, diag, prior_num, p0, m0, means, precs);
    rep->converged = converged;
    rep->diverged = diverged;
    rep->iterations = iters;
    rep->n_hist = nh;
    free(p0); free(m0); free(p1); free(m1); free(prior_num); free(node_p);
    free(node_n); free(xs); free(ps);
    return ORC_OK;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_threads(int t) {
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}
