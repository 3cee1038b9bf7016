"""Serial-schedule fixtures, made by running the REFERENCE package itself.

Run in the build container (the reference is importable only there):

    python tests/golden/make_golden_serial.py

For every case of make_golden.py it records the reference's in-place serial sweep
(solver.py:176-217) over the first sweeps, with the default ascending order and with a
seeded custom order (a permutation with one node repeated and one left out), and a full
serial ``solve`` (solver.py:307-346, plus the relative-residual stop where the case asks
for it), as tests/golden/serial/<case>.npz.  They pin the C oracle's serial sweep
(tests/test_oracle_golden.py) and the device sweep (tests/test_gpu_parity.py).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import make_golden as M  # noqa: E402  (cases, reference import, ref_solve)

gabp = M.gabp
TRACE_SWEEPS = 4
OUT = os.path.join(HERE, "serial")


def custom_order(n, seed):
    rng = np.random.default_rng(seed)
    if n == 1:
        return [0, 0]
    perm = [int(v) for v in rng.permutation(n)]
    return perm[1:] + [perm[len(perm) // 2]]  # one node left out, one node twice


def trace(g, order):
    opts = gabp.SolveOptions(schedule="serial", serial_order=order)
    st = gabp.initial_state(g, "serial")
    precs, means, changes = [], [], []
    sing_at = -1
    for t in range(TRACE_SWEEPS):
        try:
            st, c = gabp.sweep(g, st, opts)
        except gabp.solver.SingularSubgraphError:
            sing_at = t + 1
            break
        precs.append(st.prec.copy())
        means.append(st.mean.copy())
        changes.append(c)
    E = g.num_edges
    return (np.array(precs).reshape(len(precs), E), np.array(means).reshape(len(means), E),
            np.array(changes), sing_at)


def main():
    os.makedirs(OUT, exist_ok=True)
    for case, (s, extra) in M.cases().items():
        system = M.ref_system(s.pair_i, s.pair_j, s.pair_v, s.diag, s.rhs)
        g = gabp.build_graph(system)
        rec = {}
        order = custom_order(s.n, 1234)
        rec["order"] = np.array(order, dtype=np.int64)
        for tag, o in (("asc", None), ("custom", order)):
            p, m, c, sa = trace(g, o)
            rec[f"{tag}_trace_prec"] = p
            rec[f"{tag}_trace_mean"] = m
            rec[f"{tag}_trace_change"] = c
            rec[f"{tag}_trace_singular_at"] = sa
        max_iter = extra.get("max_iter", 10_000)
        rel_tol = extra.get("rel_residual_tol")
        epsilon = 1e-300 if rel_tol is not None else 1e-6
        conv, div, iters, means, pr, chh, rhh = M.ref_solve(system, "serial", epsilon, max_iter,
                                                           rel_tol)
        rec.update(serial_converged=conv, serial_diverged=div, serial_iterations=iters,
                   serial_means=means, serial_precisions=pr, serial_change_hist=chh,
                   serial_res_hist=rhh)
        print(f"{case:15s} serial conv={conv} div={div} iters={iters} E={g.num_edges}")
        np.savez_compressed(os.path.join(OUT, f"{case}.npz"), **rec)


if __name__ == "__main__":
    main()
