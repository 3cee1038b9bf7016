"""Generate the golden fixtures by running the REFERENCE package itself.

Run in the build container (the reference is importable only there):

    python tests/golden/make_golden.py

For each case it imports ``gabp`` from /root/reference/pkg/src, builds the reference
GaussianGraph, runs the first sweeps of both synchronous schedules and a full
``solve`` and stores everything as ``tests/golden/<case>.npz``.  The fixtures pin the
C oracle (tests/test_oracle_golden.py, bitwise) and the CUDA path
(tests/test_gpu_parity.py) to the reference's own outputs.  The GPU box never reads
/root/reference; it only reads these files.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import gabp  # noqa: E402  (the reference)

from paper_0810_1119_b200 import problems as P  # noqa: E402  (seeded generators only)

TRACE_SWEEPS = 6


def ref_system(pi, pj, pv, diag, rhs):
    off = {(int(i), int(j)): float(v) for i, j, v in zip(pi, pj, pv)}
    return gabp.SymSystem(diag=np.asarray(diag, float), offdiag=off, rhs=np.asarray(rhs, float))


def cases():
    out = {}
    for name in ("toy3", "cdma3", "cdma4", "nonpsd3", "poisson:3", "poisson:10"):
        s = P.load_instance(name).system
        out[name.replace(":", "")] = (s, {})
    out["poisson2d_32"] = (P.gen_poisson2d(32, 0).system, {"rel_residual_tol": 1e-8})
    out["tree25"] = (P.gen_random("tree", 25, 3).system, {})
    out["strict20"] = (P.gen_random("strict_dominant", 20, 7001).system, {})
    out["spd10"] = (P.gen_random("spd", 10, 17).system, {})
    sing = P.SymSystem(diag=np.ones(3), offdiag={(0, 1): 1.0, (1, 2): 1.0}, rhs=np.ones(3))
    out["singular_path"] = (sing, {})
    div = P.SymSystem(diag=np.ones(3), offdiag={(0, 1): 4.0, (1, 2): 4.0, (0, 2): 4.0},
                      rhs=np.ones(3))
    out["divergent3"] = (div, {"max_iter": 500})
    out["identity3"] = (P.SymSystem(diag=np.ones(3), offdiag={}, rhs=np.array([1.0, 2.0, 3.0])),
                        {})
    out["random300"] = (P.gen_random_sparse(300, 16, 1).system, {"rel_residual_tol": 1e-8})
    out["cdma_32x64"] = (P.gen_cdma_detection(64, 32, 0.5, 2)[0].system, {})
    out["poisson3d_6"] = (P.gen_poisson3d(6, 4).system, {"rel_residual_tol": 1e-8})
    return out


def ref_solve(system, schedule, epsilon, max_iter, rel_tol):
    """solver.py:307-346 verbatim through the reference's own functions, plus the
    relative-residual stop when rel_tol is given."""
    if rel_tol is None:
        r = gabp.solve(system, gabp.SolveOptions(schedule=schedule, epsilon=epsilon,
                                                 max_iter=max_iter))
        return (r.converged, r.diverged, r.iterations, r.means, r.precisions,
                np.array(r.max_change_history), np.array(r.residual_history))
    opts = gabp.SolveOptions(schedule=schedule, epsilon=epsilon, max_iter=max_iter)
    g = gabp.build_graph(system)
    state = gabp.initial_state(g, schedule)
    bnorm = float(np.linalg.norm(system.rhs))
    ch, rh = [], []
    converged = diverged = False
    for _ in range(max_iter):
        try:
            state, change = gabp.sweep(g, state, opts)
        except gabp.solver.SingularSubgraphError:
            diverged = True
            break
        means, _ = gabp.infer_marginals(g, state)
        res = gabp.residual_norm_per_eq(system, means)
        ch.append(change)
        rh.append(res)
        if change < epsilon:
            converged = True
            break
        if res * system.n < rel_tol * bnorm:
            converged = True
            break
    if not converged and not diverged:
        diverged = True
    means, precs = gabp.infer_marginals(g, state)
    return converged, diverged, state.iteration, means, precs, np.array(ch), np.array(rh)


def main():
    for case, (s, extra) in cases().items():
        system = ref_system(s.pair_i, s.pair_j, s.pair_v, s.diag, s.rhs)
        g = gabp.build_graph(system)
        rec = dict(diag=s.diag, rhs=s.rhs, pair_i=s.pair_i, pair_j=s.pair_j, pair_v=s.pair_v,
                   src=g.src, dst=g.dst, rev=g.rev, coeff=g.coeff)
        max_iter = extra.get("max_iter", 10_000)
        rel_tol = extra.get("rel_residual_tol")
        epsilon = 1e-300 if rel_tol is not None else 1e-6
        rec["epsilon"] = epsilon
        rec["max_iter"] = max_iter
        rec["rel_residual_tol"] = rel_tol if rel_tol is not None else 0.0
        for sched in ("parallel", "broadcast"):
            opts = gabp.SolveOptions(schedule=sched)
            st = gabp.initial_state(g, sched)
            precs, meanss, changes = [], [], []
            sing_at = -1
            for t in range(TRACE_SWEEPS):
                try:
                    st, c = gabp.sweep(g, st, opts)
                except gabp.solver.SingularSubgraphError:
                    sing_at = t + 1
                    break
                precs.append(st.prec.copy())
                meanss.append(st.mean.copy())
                changes.append(c)
            E = g.num_edges
            rec[f"{sched}_trace_prec"] = np.array(precs).reshape(len(precs), E)
            rec[f"{sched}_trace_mean"] = np.array(meanss).reshape(len(meanss), E)
            rec[f"{sched}_trace_change"] = np.array(changes)
            rec[f"{sched}_trace_singular_at"] = sing_at
            conv, div, iters, means, pr, chh, rhh = ref_solve(system, sched, epsilon, max_iter,
                                                             rel_tol)
            rec[f"{sched}_converged"] = conv
            rec[f"{sched}_diverged"] = div
            rec[f"{sched}_iterations"] = iters
            rec[f"{sched}_means"] = means
            rec[f"{sched}_precisions"] = pr
            rec[f"{sched}_change_hist"] = chh
            rec[f"{sched}_res_hist"] = rhh
            print(f"{case:15s} {sched:9s} conv={conv} div={div} iters={iters} E={E}")
        np.savez_compressed(os.path.join(HERE, f"{case}.npz"), **rec)


if __name__ == "__main__":
    main()
