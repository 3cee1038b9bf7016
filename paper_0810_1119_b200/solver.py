"""Gaussian BP engine -- drop-in for the reference ``solver.py`` synchronous path.

Reference: /root/reference/pkg/src/gabp/solver.py.  Same names, signatures, argument
meaning and error behaviour for the synchronous schedules:

  SolveOptions      solver.py:38-54   (+ extensions, all defaulted: rel_residual_tol,
                                        sweeps_per_poll, device, record_means_history)
  MessageState      solver.py:57-74   device-resident messages, host copies on access
  SolveReport       solver.py:77-89   (+ device_ms, sweeps_launched, final_rel_residual)
  initial_state     solver.py:92-97
  sweep             solver.py:220-229 parallel | broadcast | serial
  broadcast_sweep   solver.py:232-272
  infer_marginals   solver.py:275-287
  solve             solver.py:307-346

Every sweep runs in the CUDA library (include/gabp_b200.h); there is no CPU path.
The "serial" schedule (solver.py:176-217: an in-place, node-ordered sweep) runs as
dependency levels of the order (gabp_sweep_serial: tasks on non-adjacent nodes in
parallel, bitwise the sequential loop); its solve loop is the reference's, driven from the
host one sweep at a time (solver.py:307-346), the other schedules solve on the device.
"""

from __future__ import annotations

import ctypes
import dataclasses
from collections.abc import Sequence
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .graph import GaussianGraph, build_graph
from .linalg import SymSystem

SCHEDULES = ("parallel", "serial", "broadcast")
GPU_SCHEDULES = ("parallel", "broadcast")  # device solve loop (gabp_solve)
_AUTO_MEANS_HISTORY_DOUBLES = 1 << 24
_SERIAL_COOP_MAX_LEVELS = 512  # capi.cu gabp_sweep_serial: cooperative sweep up to here


class SingularSubgraphError(ArithmeticError):
    """An exclusion precision hit exactly zero; the update is undefined (solver.py:34)."""


@dataclass
class SolveOptions:
    epsilon: float = 1e-6
    max_iter: int = 10_000
    blowup: float = 1e10
    schedule: str = "parallel"
    serial_order: list[int] | None = None
    # extensions (not in the reference)
    rel_residual_tol: float | None = None   # also stop when ||Ax-b||/||b|| < tol
    sweeps_per_poll: int = 0                # sweeps per CUDA-graph chunk; 0 = auto
    device: int | None = None
    record_means_history: bool | None = None  # None: auto (n * max_iter <= 2^24)
    gather_mode: str = "auto"   # auto | message | recompute | slice | rows (bitwise-identical)

    def __post_init__(self):
        if self.epsilon <= 0.0:
            raise ValueError("epsilon must be positive")
        if self.max_iter < 1:
            raise ValueError("max_iter must be >= 1")
        if not self.blowup > 1.0:
            raise ValueError("blowup must exceed 1")
        if self.schedule not in SCHEDULES:
            raise ValueError(f"schedule must be one of {SCHEDULES}")
        if self.gather_mode not in _lib.GATHER_IDS:
            raise ValueError(f"gather_mode must be one of {tuple(_lib.GATHER_IDS)}")
        if self.gather_mode in ("slice", "rows") and self.schedule == "serial":
            raise ValueError("the slice layout runs the synchronous schedules")


def _gpu_schedule(schedule: str) -> int:
    if schedule not in GPU_SCHEDULES:
        raise ValueError(
            f"schedule {schedule!r} is not a synchronous sweep; the B200 path implements "
            f"{GPU_SCHEDULES} (the serial schedule is sequential by definition)")
    return _lib.SCHED_IDS[schedule]


class MessageState:
    """Per-directed-edge (P, mu) messages held in HBM (solver.py:57-74)."""

    def __init__(self, graph: GaussianGraph, schedule: str = "parallel", _handle=None):
        self.graph = graph
        self.schedule = schedule
        if _handle is None:
            h = ctypes.c_void_p()
            _lib.check(_lib.load().gabp_state_create(graph.handle, ctypes.byref(h)))
            _handle = h
        self._h = _handle

    @property
    def handle(self):
        return self._h

    def _counters(self):
        it = ctypes.c_int64()
        ms = ctypes.c_int64()
        _lib.check(_lib.load().gabp_state_counters(self._h, ctypes.byref(it), ctypes.byref(ms)))
        return int(it.value), int(ms.value)

    @property
    def iteration(self) -> int:
        return self._counters()[0]

    @property
    def messages_sent(self) -> int:
        return self._counters()[1]

    def _read(self):
        E = self.graph.num_edges
        p = np.empty(E)
        m = np.empty(E)
        _lib.check(_lib.load().gabp_state_read(self._h, _lib.ptr(p), _lib.ptr(m)))
        return p, m

    @property
    def prec(self) -> np.ndarray:
        return self._read()[0]

    @prec.setter
    def prec(self, value) -> None:
        # the reference assigns the buffers directly (acceleration.py:123-126); here the
        # assignment writes through to the device state
        self.set_messages(value, self._read()[1])

    @property
    def mean(self) -> np.ndarray:
        return self._read()[1]

    @mean.setter
    def mean(self, value) -> None:
        self.set_messages(self._read()[0], value)

    def gather(self, edges) -> tuple[np.ndarray, np.ndarray]:
        """(prec, mean) of the given edge ids, read from the device (point reads of
        the buffers, as compute_message indexes them)."""
        idx = np.ascontiguousarray(np.asarray(edges, dtype=np.int64).reshape(-1))
        p = np.empty(idx.size)
        m = np.empty(idx.size)
        _lib.check(_lib.load().gabp_state_gather(self._h, _lib.ptr(idx), idx.size,
                                                  _lib.ptr(p), _lib.ptr(m)))
        return p, m

    def set_messages(self, prec, mean) -> None:
        prec = np.ascontiguousarray(prec, dtype=np.float64)
        mean = np.ascontiguousarray(mean, dtype=np.float64)
        if prec.shape != (self.graph.num_edges,) or mean.shape != prec.shape:
            raise ValueError("message arrays must have one entry per directed edge")
        _lib.check(_lib.load().gabp_state_write(self._h, _lib.ptr(prec), _lib.ptr(mean)))

    def copy(self) -> "MessageState":
        h = ctypes.c_void_p()
        _lib.check(_lib.load().gabp_state_clone(self._h, ctypes.byref(h)))
        return MessageState(self.graph, self.schedule, _handle=h)

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.load().gabp_state_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class SolveReport:
    converged: bool
    diverged: bool
    iterations: int
    means: np.ndarray
    precisions: np.ndarray | None
    max_change_history: list = field(default_factory=list)
    residual_history: list = field(default_factory=list)
    means_history: list = field(default_factory=list)
    messages_sent: int = 0
    precisions_exact: bool | None = None
    # extensions
    device_ms: float = 0.0
    sweeps_launched: int = 0
    final_rel_residual: float = float("nan")
    residual_probes: int = 0
    kernel_launches: int = 0
    split_sweeps: int = 0   # multi-rank: sweeps run as boundary part + interior part
    dist_layout: int = 0    # multi-rank kernel family: 1 slice, 2 tiles, 3 diagonal
    message_bins: int = 0   # parallel row kernel: bins of the binned message order (0: CSR)


def initial_state(graph: GaussianGraph, schedule: str = "parallel") -> MessageState:
    """solver.py:92-97: all messages exactly zero."""
    return MessageState(graph, schedule)


def _exclusion(graph: GaussianGraph, state: MessageState, i: int, j: int):
    """P_{i\\j} and the matching precision-weighted mean numerator (solver.py:100-111):
    the prior plus every incoming message but j's, in ascending neighbour order."""
    rp = graph.row_ptr
    lo, hi = int(rp[i]), int(rp[i + 1])
    nbr = graph.dst[lo:hi]
    prec, mean = state.gather(graph.rev[lo:hi])  # incoming m_ki, k ascending
    acc_p = float(graph.prior_prec[i])
    acc_num = float(graph.prior_prec[i]) * float(graph.prior_mean[i])
    for pos in range(nbr.size):
        if int(nbr[pos]) == j:
            continue
        acc_p += float(prec[pos])
        acc_num += float(prec[pos]) * float(mean[pos])
    return acc_p, acc_num


def _edge_coeff(graph: GaussianGraph, i: int, j: int) -> float:
    rp = graph.row_ptr
    lo, hi = int(rp[i]), int(rp[i + 1])
    pos = int(np.searchsorted(graph.dst[lo:hi], j))
    if not (0 <= i < graph.n) or pos >= hi - lo or int(graph.dst[lo + pos]) != j:
        raise KeyError(f"({i}, {j}) is not an edge")
    return float(graph.coeff[lo + pos])


def compute_message(graph: GaussianGraph, state: MessageState, i: int, j: int):
    """Sum-product message (P_ij, mu_ij) from the current buffers (solver.py:114-122)."""
    i, j = int(i), int(j)
    if not (0 <= i < graph.n):
        raise KeyError(f"({i}, {j}) is not an edge")
    a = _edge_coeff(graph, i, j)
    p_excl, num = _exclusion(graph, state, i, j)
    if p_excl == 0.0:
        raise SingularSubgraphError(f"P_excl({i} -> {j}) = 0")
    return -a * a / p_excl, num / a


def compute_message_max_product(graph: GaussianGraph, state: MessageState, i: int, j: int):
    """Max-product message via the closed-form argmax of the integrand (solver.py:125-143):
    equal to the sum-product message in exact arithmetic, rounded differently."""
    i, j = int(i), int(j)
    if not (0 <= i < graph.n):
        raise KeyError(f"({i}, {j}) is not an edge")
    a = _edge_coeff(graph, i, j)
    p_excl, num = _exclusion(graph, state, i, j)
    if p_excl == 0.0:
        raise SingularSubgraphError(f"P_excl({i} -> {j}) = 0")
    mu_excl = num / p_excl
    prec = -a * a / p_excl
    return prec, -a * mu_excl / prec


def _sweep(graph: GaussianGraph, state: MessageState, schedule: str):
    sched = _gpu_schedule(schedule)
    out = state.copy()
    out.schedule = schedule
    mc = ctypes.c_double()
    si = ctypes.c_int64()
    node = ctypes.c_int32()
    rc = _lib.load().gabp_sweep(graph.handle, out.handle, sched, ctypes.byref(mc),
                                ctypes.byref(si), ctypes.byref(node))
    if rc == _lib.GABP_ESINGULAR:
        out.close()
        k = int(si.value)
        if node.value:
            raise SingularSubgraphError(f"aggregate precision P~({k}) = 0")
        src = int(graph.src[k])
        dst = int(graph.dst[k])
        raise SingularSubgraphError(f"P_excl({src} -> {dst}) = 0")
    _lib.check(rc)
    return out, float(mc.value)


def _order_arg(order):
    if order is None:
        return None, 0, None
    arr = np.ascontiguousarray(np.asarray(order, dtype=np.int64).reshape(-1))
    return arr, int(arr.size), arr.ctypes.data_as(ctypes.c_void_p)


def _serial_inplace(graph: GaussianGraph, state: MessageState, order_arg, blowup: float):
    """One serial sweep in place on `state`: (max change, out of range, levels)."""
    _, norder, optr = order_arg
    mc = ctypes.c_double()
    oor = ctypes.c_int32()
    se = ctypes.c_int64()
    nl = ctypes.c_int32()
    rc = _lib.load().gabp_sweep_serial(graph.handle, state.handle, optr, norder, blowup,
                                       ctypes.byref(mc), ctypes.byref(oor), ctypes.byref(se),
                                       ctypes.byref(nl))
    if rc == _lib.GABP_ESINGULAR:
        k = int(se.value)
        raise SingularSubgraphError(f"P_excl({int(graph.src[k])} -> {int(graph.dst[k])}) = 0")
    _lib.check(rc)
    return float(mc.value), bool(oor.value), int(nl.value)


def _sweep_serial(graph: GaussianGraph, state: MessageState, order):
    """solver.py:176-217: in-place node-ordered round on a copy of the state."""
    out = state.copy()
    out.schedule = "serial"
    try:
        mc, _, _ = _serial_inplace(graph, out, _order_arg(order), float("inf"))
    except BaseException:
        out.close()
        raise
    return out, mc


def sweep(graph: GaussianGraph, state: MessageState, options: SolveOptions):
    """One message-passing round; returns (new state, max message change)."""
    if options.schedule == "serial":
        return _sweep_serial(graph, state, options.serial_order)
    return _sweep(graph, state, options.schedule)


def broadcast_sweep(graph: GaussianGraph, state: MessageState, options=None):
    """solver.py:232-272: aggregate-and-subtract round."""
    return _sweep(graph, state, "broadcast")


def infer_marginals(graph: GaussianGraph, state: MessageState):
    """solver.py:275-287: (means, precisions); non-finite means where prec_tot == 0."""
    means = np.empty(graph.n)
    precs = np.empty(graph.n)
    _lib.check(_lib.load().gabp_infer_marginals(graph.handle, state.handle, _lib.ptr(means),
                                                 _lib.ptr(precs)))
    return means, precs


def _options_struct(options: SolveOptions, n: int, hist: np.ndarray | None) -> _lib.Options:
    o = _lib.Options()
    o.epsilon = float(options.epsilon)
    o.max_iter = int(options.max_iter)
    o.blowup = float(options.blowup)
    o.schedule = _gpu_schedule(options.schedule)
    o.sweeps_per_poll = int(options.sweeps_per_poll)
    o.rel_residual_tol = float(options.rel_residual_tol or 0.0)
    o.gather_mode = _lib.GATHER_IDS[options.gather_mode]
    if hist is not None:
        o.means_history = hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        o.means_history_rows = hist.shape[0]
    return o


def _want_means_history(options: SolveOptions, n: int) -> bool:
    if options.record_means_history is None:
        return n * options.max_iter <= _AUTO_MEANS_HISTORY_DOUBLES
    return bool(options.record_means_history)


class MeansHistory(Sequence):
    """SolveReport.means_history (solver.py:319, 332: the tentative means of every sweep),
    materialised on first access.

    A solve whose n x max_iter would not fit the eager host buffer (record_means_history
    left at None) records none on the device; the first read of this sequence replays the
    solve -- bitwise deterministic, so the same messages and means sweep for sweep -- with
    max_iter = the number of sweeps the solve ran, recording every row."""

    def __init__(self, count: int, replay):
        self._count = int(count)
        self._replay = replay
        self._rows = None

    def _load(self):
        if self._rows is None:
            rows = self._replay()
            if len(rows) != self._count:
                raise RuntimeError(f"means-history replay ran {len(rows)} sweeps, "
                                   f"the solve ran {self._count}")
            self._rows = rows
            self._replay = None
        return self._rows

    def __len__(self) -> int:
        return self._count

    def __getitem__(self, t):
        return self._load()[t]

    def __eq__(self, other):
        return list(self) == list(other) if isinstance(other, (list, Sequence)) else NotImplemented

    def __repr__(self) -> str:
        state = "loaded" if self._rows is not None else "not loaded"
        return f"MeansHistory({self._count} sweeps, {state})"


def _replay_options(options: SolveOptions, k: int) -> SolveOptions:
    return dataclasses.replace(options, max_iter=max(int(k), 1), record_means_history=True)


def _solve_serial(graph: GaussianGraph, options: SolveOptions) -> SolveReport:
    """solver.py:307-346 with the serial schedule: one device sweep (dependency levels)
    per iteration, then the reference's tests on the tentative means (device marginals and
    residual), the message change and the blow-up / finiteness flags of the sweep."""
    import time
    n = graph.n
    lib = _lib.load()
    order_arg = _order_arg(options.serial_order)
    state = initial_state(graph, "serial")
    want_hist = _want_means_history(options, n)
    bnorm = float(graph.info.rhs_norm)
    max_hist, res_hist, means_hist = [], [], []
    converged = diverged = False
    res = float("nan")
    launches = 0
    t0 = time.perf_counter()
    try:
        for _ in range(options.max_iter):
            try:
                max_change, out_of_range, levels = _serial_inplace(graph, state, order_arg,
                                                                   float(options.blowup))
            except SingularSubgraphError:
                diverged = True
                break
            # one cooperative launch for short orders, one launch per level otherwise
            # (capi.cu: gabp_sweep_serial)
            launches += 1 if levels <= _SERIAL_COOP_MAX_LEVELS else levels
            means, _ = infer_marginals(graph, state)
            means_finite = bool(np.all(np.isfinite(means)))
            if means_finite:
                r = ctypes.c_double()
                _lib.check(lib.gabp_residual_norm_per_eq(graph.handle, _lib.ptr(means),
                                                         ctypes.byref(r)))
                res = float(r.value)
            else:
                res = float("inf")
            max_hist.append(max_change)
            res_hist.append(res)
            if want_hist:
                means_hist.append(means)
            if out_of_range or not means_finite:
                diverged = True
                break
            if max_change < options.epsilon:
                converged = True
                break
            if (options.rel_residual_tol and bnorm > 0.0
                    and res * n / bnorm < options.rel_residual_tol):
                converged = True
                break
        if not converged and not diverged:
            diverged = True  # cap exhausted
        means, precs = infer_marginals(graph, state)
        if not want_hist and options.record_means_history is None:
            k = len(max_hist)
            means_hist = MeansHistory(k, lambda: list(
                _solve_serial(graph, _replay_options(options, k)).means_history)[:k])
        return SolveReport(
            converged=converged, diverged=diverged, iterations=state.iteration,
            means=means, precisions=precs, max_change_history=max_hist,
            residual_history=res_hist, means_history=means_hist,
            messages_sent=state.messages_sent, precisions_exact=graph.is_tree(),
            device_ms=(time.perf_counter() - t0) * 1e3, sweeps_launched=state.iteration,
            final_rel_residual=(res * n / bnorm) if bnorm > 0.0 and res_hist else float("nan"),
            kernel_launches=launches)
    finally:
        state.close()


def solve_graph(graph: GaussianGraph, options: SolveOptions | None = None) -> SolveReport:
    """solve() on an already built graph (reuses its device workspace)."""
    options = options or SolveOptions()
    if options.schedule == "serial":
        return _solve_serial(graph, options)
    n = graph.n
    hist = np.empty((options.max_iter, n)) if _want_means_history(options, n) else None
    o = _options_struct(options, n, hist)
    means = np.empty(n)
    precs = np.empty(n)
    ch = np.empty(options.max_iter)
    rh = np.empty(options.max_iter)
    rep = _lib.Report()
    _lib.check(_lib.load().gabp_solve(graph.handle, ctypes.byref(o), _lib.ptr(means),
                                      _lib.ptr(precs), _lib.ptr(ch), _lib.ptr(rh),
                                      ctypes.byref(rep)))
    k = int(rep.n_hist)
    if hist is not None:
        means_hist = [hist[t].copy() for t in range(k)]
    elif options.record_means_history is None:
        means_hist = MeansHistory(k, lambda: list(
            solve_graph(graph, _replay_options(options, k)).means_history)[:k])
    else:
        means_hist = []
    return SolveReport(
        converged=bool(rep.converged),
        diverged=bool(rep.diverged),
        iterations=int(rep.iterations),
        means=means,
        precisions=precs,
        max_change_history=ch[:k].tolist(),
        residual_history=rh[:k].tolist(),
        means_history=means_hist,
        messages_sent=int(rep.messages_sent),
        precisions_exact=graph.is_tree(),
        device_ms=float(rep.device_ms),
        sweeps_launched=int(rep.sweeps_launched),
        final_rel_residual=float(rep.final_rel_residual),
        residual_probes=int(rep.residual_probes),
        kernel_launches=int(rep.kernel_launches),
        message_bins=int(rep.message_bins),
    )


def solve(system: SymSystem, options: SolveOptions | None = None) -> SolveReport:
    """solver.py:307-346: run GaBP to convergence, divergence or the sweep cap.

    The sweep that first leaves every message within epsilon of its previous value is
    counted; per-sweep message change and residual_norm_per_eq of the tentative means
    are recorded.  Divergence (blowup, non-finite values, a singular exclusion sum, the
    sweep cap) is reported, never raised."""
    options = options or SolveOptions()
    if options.schedule != "serial":
        _gpu_schedule(options.schedule)
    graph = build_graph(system, options.device)
    try:
        rep = solve_graph(graph, options)
    finally:
        graph.close()
    if isinstance(rep.means_history, MeansHistory):
        k = len(rep.means_history)

        def replay():
            g = build_graph(system, options.device)
            try:
                return list(solve_graph(g, _replay_options(options, k)).means_history)[:k]
            finally:
                g.close()

        rep.means_history = MeansHistory(k, replay)
    return rep
