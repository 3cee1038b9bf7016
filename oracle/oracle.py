"""CPU oracle for the GaBP sweep path -- TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and ``bench.py`` (its cpu_baseline leg and
``--impl reference``) may import this module; the product package never does.

Thin numpy/ctypes wrapper over ``oracle/gabp_oracle.c``, the plain-C restatement of
the reference's synchronous sweep (reference file:line citations are in that file's
header).  Parity is pinned: ``tests/test_oracle_golden.py`` checks these functions
bitwise against fixtures produced by running the reference package itself
(``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libgabp_oracle.so")
_lib = None

SCHEDULE_IDS = {"parallel": 0, "broadcast": 2}

_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)


class _SweepOut(ctypes.Structure):
    _fields_ = [("max_change", ctypes.c_double), ("singular", ctypes.c_int64),
                ("singular_is_node", ctypes.c_int)]


class _Options(ctypes.Structure):
    _fields_ = [("epsilon", ctypes.c_double), ("max_iter", ctypes.c_int64),
                ("blowup", ctypes.c_double), ("schedule", ctypes.c_int),
                ("rel_residual_tol", ctypes.c_double)]


class _Report(ctypes.Structure):
    _fields_ = [("converged", ctypes.c_int), ("diverged", ctypes.c_int),
                ("iterations", ctypes.c_int64), ("n_hist", ctypes.c_int64)]


def build() -> str:
    """Compile the oracle library (gcc, OpenMP) in place; returns its path."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = ctypes.CDLL(_LIB_PATH)
        _lib.oracle_build_graph.restype = ctypes.c_int
        _lib.oracle_residual_sq.restype = ctypes.c_double
        _lib.oracle_solve.restype = ctypes.c_int
        _lib.oracle_num_threads.restype = ctypes.c_int
    return _lib


def _p64(a):
    return a.ctypes.data_as(_i64p)


def _pf(a):
    return a.ctypes.data_as(_f64p)


def set_threads(t: int) -> None:
    lib().oracle_set_threads(ctypes.c_int(int(t)))


def num_threads() -> int:
    return int(lib().oracle_num_threads())


@dataclass
class OracleGraph:
    n: int
    row_ptr: np.ndarray
    col: np.ndarray
    rev: np.ndarray
    coeff: np.ndarray
    diag: np.ndarray
    rhs: np.ndarray
    prior_num: np.ndarray

    @property
    def num_edges(self) -> int:
        return int(self.row_ptr[-1])

    @property
    def src(self) -> np.ndarray:
        return np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.row_ptr))


def build_graph(diag, rhs, pair_i, pair_j, pair_v) -> OracleGraph:
    """graph.py:63-120 restated: directed CSR, twin index, coefficients."""
    diag = np.ascontiguousarray(diag, dtype=np.float64)
    rhs = np.ascontiguousarray(rhs, dtype=np.float64)
    pi = np.ascontiguousarray(pair_i, dtype=np.int64)
    pj = np.ascontiguousarray(pair_j, dtype=np.int64)
    pv = np.ascontiguousarray(pair_v, dtype=np.float64)
    n = diag.size
    E = 2 * pi.size
    row_ptr = np.empty(n + 1, dtype=np.int64)
    col = np.empty(E, dtype=np.int64)
    rev = np.empty(E, dtype=np.int64)
    coeff = np.empty(E, dtype=np.float64)
    rc = lib().oracle_build_graph(ctypes.c_int64(n), ctypes.c_int64(pi.size), _p64(pi), _p64(pj),
                                  _pf(pv), _p64(row_ptr), _p64(col), _p64(rev), _pf(coeff))
    if rc != 0:
        raise ValueError(f"oracle_build_graph failed (rc={rc})")
    prior_num = np.empty(n, dtype=np.float64)
    lib().oracle_priors(ctypes.c_int64(n), _pf(diag), _pf(rhs), _pf(prior_num))
    return OracleGraph(n, row_ptr, col, rev, coeff, diag, rhs, prior_num)


def sweep(g: OracleGraph, prec, mean, schedule: str = "parallel"):
    """One synchronous sweep; returns (prec', mean', max_change, singular_index|-1)."""
    prec = np.ascontiguousarray(prec, dtype=np.float64)
    mean = np.ascontiguousarray(mean, dtype=np.float64)
    po = np.empty_like(prec)
    mo = np.empty_like(mean)
    out = _SweepOut()
    if schedule == "broadcast":
        node_p = np.empty(g.n)
        node_n = np.empty(g.n)
        lib().oracle_sweep_broadcast(ctypes.c_int64(g.n), _p64(g.row_ptr), _p64(g.col),
                                     _p64(g.rev), _pf(g.coeff), _pf(g.diag), _pf(g.prior_num),
                                     _pf(prec), _pf(mean), _pf(po), _pf(mo), _pf(node_p),
                                     _pf(node_n), ctypes.byref(out))
    else:
        lib().oracle_sweep_parallel(ctypes.c_int64(g.n), _p64(g.row_ptr), _p64(g.col),
                                    _p64(g.rev), _pf(g.coeff), _pf(g.diag), _pf(g.prior_num),
                                    _pf(prec), _pf(mean), _pf(po), _pf(mo), ctypes.byref(out))
    return po, mo, float(out.max_change), int(out.singular)


def sweep_serial(g: OracleGraph, prec, mean, order=None):
    """solver.py:176-217 on copies: (prec', mean', max_change, singular edge | -1)."""
    po = np.array(prec, dtype=np.float64, copy=True)
    mo = np.array(mean, dtype=np.float64, copy=True)
    out = _SweepOut()
    if order is None:
        optr, norder = None, 0
    else:
        o = np.ascontiguousarray(order, dtype=np.int64)
        optr, norder = _p64(o), o.size
    lib().oracle_sweep_serial(ctypes.c_int64(g.n), _p64(g.row_ptr), _p64(g.rev), _pf(g.coeff),
                              _pf(g.diag), _pf(g.prior_num), _pf(po), _pf(mo), optr,
                              ctypes.c_int64(norder), ctypes.byref(out))
    return po, mo, float(out.max_change), int(out.singular)


def solve_serial(g: OracleGraph, epsilon=1e-6, max_iter=10_000, blowup=1e10, order=None,
                 rel_residual_tol=None) -> "OracleReport":
    """solver.py:307-346 with the serial schedule (+ optional relative-residual stop)."""
    E = g.num_edges
    prec = np.zeros(E)
    mean = np.zeros(E)
    bnorm = float(np.linalg.norm(g.rhs))
    ch, rh = [], []
    converged = diverged = False
    it = 0
    for _ in range(max_iter):
        p2, m2, mc, sing = sweep_serial(g, prec, mean, order)
        if sing >= 0:
            diverged = True
            break
        prec, mean = p2, m2
        it += 1
        means, _ = marginals(g, prec, mean)
        finite_means = bool(np.all(np.isfinite(means)))
        res = float(np.sqrt(residual_sq(g, means)) / g.n) if finite_means else np.inf
        ch.append(mc)
        rh.append(res)
        with np.errstate(all="ignore"):
            biggest = max(float(np.max(np.abs(prec), initial=0.0)),
                          float(np.max(np.abs(mean), initial=0.0)))
        finite = bool(np.all(np.isfinite(prec)) and np.all(np.isfinite(mean)))
        if not finite or biggest > blowup or not finite_means:
            diverged = True
            break
        if mc < epsilon:
            converged = True
            break
        if rel_residual_tol and res * g.n < rel_residual_tol * bnorm:
            converged = True
            break
    if not converged and not diverged:
        diverged = True
    means, precs = marginals(g, prec, mean)
    return OracleReport(converged, diverged, it, means, precs, np.array(ch), np.array(rh))


def marginals(g: OracleGraph, prec, mean):
    prec = np.ascontiguousarray(prec, dtype=np.float64)
    mean = np.ascontiguousarray(mean, dtype=np.float64)
    means = np.empty(g.n)
    precs = np.empty(g.n)
    with np.errstate(all="ignore"):
        lib().oracle_marginals(ctypes.c_int64(g.n), _p64(g.row_ptr), _p64(g.rev), _pf(g.diag),
                               _pf(g.prior_num), _pf(prec), _pf(mean), _pf(means), _pf(precs))
    return means, precs


def residual_sq(g: OracleGraph, x) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64)
    return float(lib().oracle_residual_sq(ctypes.c_int64(g.n), _p64(g.row_ptr), _p64(g.col),
                                          _pf(g.coeff), _pf(g.diag), _pf(g.rhs), _pf(x)))


@dataclass
class OracleReport:
    converged: bool
    diverged: bool
    iterations: int
    means: np.ndarray
    precisions: np.ndarray
    max_change_history: np.ndarray
    residual_history: np.ndarray


def solve(g: OracleGraph, epsilon=1e-6, max_iter=10_000, blowup=1e10, schedule="parallel",
          rel_residual_tol=None) -> OracleReport:
    """solver.py:307-346 restated (+ optional relative-residual stop)."""
    opt = _Options(float(epsilon), int(max_iter), float(blowup), SCHEDULE_IDS[schedule],
                   float(rel_residual_tol or 0.0))
    means = np.empty(g.n)
    precs = np.empty(g.n)
    ch = np.empty(max_iter)
    rh = np.empty(max_iter)
    rep = _Report()
    rc = lib().oracle_solve(ctypes.c_int64(g.n), _p64(g.row_ptr), _p64(g.col), _p64(g.rev),
                            _pf(g.coeff), _pf(g.diag), _pf(g.rhs), ctypes.byref(opt), _pf(means),
                            _pf(precs), _pf(ch), _pf(rh), ctypes.byref(rep))
    if rc != 0:
        raise MemoryError(f"oracle_solve failed (rc={rc})")
    k = int(rep.n_hist)
    return OracleReport(bool(rep.converged), bool(rep.diverged), int(rep.iterations), means,
                        precs, ch[:k].copy(), rh[:k].copy())
