"""Binned message order of the four-rows-per-warp parallel kernel (rowpar.cu: rowquad_kernel,
build.cu: build_bins): the solve keeps its messages at the rank of (bin of the destination,
source, destination) instead of the CSR edge order.  The order is internal to a solve, so every
result must stay bitwise the C oracle's (solver.py:146-173) and the CSR-order kernel's.  Small
graphs take the binned order here through a tiny window (GABP_BIN_WINDOW_MB); the full-size
default is covered by test_random_1m_default_is_binned."""

import os

import numpy as np
import pytest

import paper_0810_1119_b200 as G
from oracle import oracle
from paper_0810_1119_b200 import _lib
from tests.test_fuzz_gpu import _system

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    _lib.load()
    assert _lib.device_count() > 0, "no CUDA device: " + _lib.last_error()
    oracle.build()


def _bits(a):
    return np.asarray(a, dtype=np.float64).view(np.uint64)


@pytest.fixture
def tiny_window(monkeypatch):
    monkeypatch.setenv("GABP_BIN_WINDOW_MB", "0.002")  # 2 KB of messages per bin
    monkeypatch.delenv("GABP_ROW_NO_BIN", raising=False)


def _solve_rows(s, **kw):
    return G.solve(s, G.SolveOptions(schedule="parallel", gather_mode="rows", **kw))


CASES = [
    # n, mean degree, hub rows (70..250 edges: the long-row path), dominance, isolated rows
    (300, 6.0, 0, 1.3, False),
    (900, 13.0, 2, 1.3, True),
    (2500, 30.0, 2, 1.05, False),
    (7000, 55.0, 0, 1.3, False),
    (20000, 13.0, 2, 0.8, True),   # not diagonally dominant: diverges
    (60000, 5.0, 2, 1.3, True),
]


@pytest.mark.parametrize("n,deg,hubs,dom,iso", CASES)
def test_binned_order_matches_oracle_and_csr_order(tiny_window, monkeypatch, n, deg, hubs, dom,
                                                   iso):
    s = _system(np.random.default_rng(n + 17), n, deg, hubs, dom, iso)
    og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
    kw = dict(epsilon=1e-300, rel_residual_tol=1e-10, max_iter=60)
    o = oracle.solve(og, schedule="parallel", **kw)
    r = _solve_rows(s, **kw)
    assert r.message_bins >= 2, "the solve did not run in binned order"
    assert r.iterations == o.iterations and r.converged == o.converged
    assert r.diverged == o.diverged
    np.testing.assert_array_equal(_bits(r.means), _bits(o.means))
    np.testing.assert_array_equal(_bits(r.precisions), _bits(o.precisions))
    np.testing.assert_array_equal(np.asarray(r.max_change_history), o.max_change_history)
    if o.iterations and np.all(np.isfinite(o.residual_history)):
        # (summation order: rows in CSR order here, dict order in the reference; a residual
        # far below the first one is the rounding error of that sum)
        np.testing.assert_allclose(r.residual_history, o.residual_history, rtol=1e-9,
                                   atol=1e-12 * o.residual_history[0])
    np.testing.assert_array_equal(_bits(r.means_history[-1]), _bits(r.means))
    # the same solve in CSR order (a fresh graph: the order is chosen once per graph)
    monkeypatch.setenv("GABP_ROW_NO_BIN", "1")
    c = _solve_rows(s, **kw)
    assert c.message_bins == 0
    assert c.iterations == r.iterations
    np.testing.assert_array_equal(_bits(c.means), _bits(r.means))
    np.testing.assert_array_equal(np.asarray(c.max_change_history),
                                  np.asarray(r.max_change_history))


@pytest.mark.parametrize("sweep_cap", [1, 2, 3, 5, 60])
def test_binned_order_degree_ladder(tiny_window, sweep_cap):
    """Every degree class the four-rows-per-warp kernel distinguishes (0, 1..64 in the quads,
    one or two own blocks, an odd last block; 65..255 through the long-row path) in binned
    order, stopped after each of the first launches and at convergence."""
    from tests.test_gpu_parity import _degree_ladder_system

    s = _degree_ladder_system()
    og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
    o = oracle.solve(og, epsilon=1e-12, max_iter=sweep_cap, schedule="parallel")
    r = _solve_rows(s, epsilon=1e-12, max_iter=sweep_cap)
    assert r.message_bins >= 2
    assert r.iterations == o.iterations and r.converged == o.converged
    np.testing.assert_array_equal(_bits(r.means), _bits(o.means))
    np.testing.assert_array_equal(_bits(r.precisions), _bits(o.precisions))
    np.testing.assert_array_equal(np.asarray(r.max_change_history),
                                  np.asarray(o.max_change_history))


@pytest.mark.parametrize("binned", [False, True])
@pytest.mark.parametrize("slots", [2, 4, 6, 8])
def test_every_slot_count_on_the_degree_ladder(monkeypatch, slots, binned):
    """rowquad_kernel is instantiated for 2, 4, 6 and 8 slots per lane (rows of up to 16 .. 64
    edges in the quads; a graph normally runs the smallest one that covers its rows).  Forced
    here (GABP_QUAD_SLOTS), so every longer row of the ladder takes the long-row path: both
    message orders, bitwise the oracle."""
    from tests.test_gpu_parity import _degree_ladder_system

    monkeypatch.setenv("GABP_QUAD_SLOTS", str(slots))
    if binned:
        monkeypatch.setenv("GABP_BIN_WINDOW_MB", "0.002")
        monkeypatch.delenv("GABP_ROW_NO_BIN", raising=False)
    else:
        monkeypatch.setenv("GABP_ROW_NO_BIN", "1")
    s = _degree_ladder_system()
    og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
    for cap in (2, 60):
        o = oracle.solve(og, epsilon=1e-12, max_iter=cap, schedule="parallel")
        r = _solve_rows(s, epsilon=1e-12, max_iter=cap)
        assert (r.message_bins >= 2) == binned
        assert r.iterations == o.iterations and r.converged == o.converged
        np.testing.assert_array_equal(_bits(r.means), _bits(o.means))
        np.testing.assert_array_equal(_bits(r.precisions), _bits(o.precisions))
        np.testing.assert_array_equal(np.asarray(r.max_change_history),
                                      np.asarray(o.max_change_history))


def test_binned_graph_is_reused_and_reproducible(tiny_window):
    """One graph, several solves (different caps, then a new right-hand side): the index arrays
    are built once, every solve is bitwise the oracle, repeated solves agree bit for bit."""
    s = _system(np.random.default_rng(5), 4000, 24.0, 1, 1.2, False)
    og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
    g = G.build_graph(s, 0)
    try:
        prev = None
        for cap in (3, 40, 40):
            opts = G.SolveOptions(schedule="parallel", gather_mode="rows", epsilon=1e-300,
                                  rel_residual_tol=1e-11, max_iter=cap)
            r = G.solve_graph(g, opts)
            o = oracle.solve(og, schedule="parallel", epsilon=1e-300, rel_residual_tol=1e-11,
                             max_iter=cap)
            assert r.message_bins >= 2
            assert r.iterations == o.iterations
            np.testing.assert_array_equal(_bits(r.means), _bits(o.means))
            if prev is not None and prev.iterations == r.iterations:
                np.testing.assert_array_equal(_bits(prev.means), _bits(r.means))
                assert list(prev.residual_history) == list(r.residual_history)
            prev = r
    finally:
        g.close()


def test_broadcast_and_single_sweeps_stay_in_csr_order(tiny_window):
    """Only the parallel row kernel's solve loop uses the binned order: the single-sweep API
    (messages visible to the caller) and the broadcast schedule are untouched by it."""
    s = _system(np.random.default_rng(9), 1500, 14.0, 0, 1.3, False)
    og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
    r = _solve_rows(s, epsilon=1e-300, rel_residual_tol=1e-10, max_iter=30)
    assert r.message_bins >= 2
    b = G.solve(s, G.SolveOptions(schedule="broadcast", epsilon=1e-300, rel_residual_tol=1e-10,
                                  max_iter=30))
    assert b.message_bins == 0
    ob = oracle.solve(og, schedule="broadcast", epsilon=1e-300, rel_residual_tol=1e-10,
                      max_iter=30)
    np.testing.assert_array_equal(_bits(b.means), _bits(ob.means))
    g = G.build_graph(s, 0)
    try:
        G.solve_graph(g, G.SolveOptions(schedule="parallel", gather_mode="rows",
                                        epsilon=1e-300, max_iter=5))
        st = G.initial_state(g)
        po = np.zeros(g.num_edges)
        mo = np.zeros(g.num_edges)
        for _ in range(3):
            st, _ = G.sweep(g, st, G.SolveOptions(schedule="parallel"))
            po, mo, _, _ = oracle.sweep(og, po, mo, "parallel")
        np.testing.assert_array_equal(_bits(st.prec), _bits(po))
        np.testing.assert_array_equal(_bits(st.mean), _bits(mo))
    finally:
        g.close()


def test_random_1m_default_is_binned():
    """BASELINE config 1 with default settings: 0.54 GB of messages per generation exceed L2,
    so the parallel solve runs binned -- bitwise the CSR-order solve, run twice (run-to-run
    reproducible residual history)."""
    os.environ.pop("GABP_BIN_WINDOW_MB", None)
    os.environ.pop("GABP_ROW_NO_BIN", None)
    s = G.gen_random_sparse(1 << 20, 16, 0).system
    kw = dict(schedule="parallel", epsilon=1e-300, rel_residual_tol=1e-8, max_iter=50,
              record_means_history=False)
    r1 = G.solve(s, G.SolveOptions(**kw))
    assert r1.message_bins >= 2 and r1.converged
    r2 = G.solve(s, G.SolveOptions(**kw))
    os.environ["GABP_ROW_NO_BIN"] = "1"
    try:
        c = G.solve(s, G.SolveOptions(**kw))
    finally:
        os.environ.pop("GABP_ROW_NO_BIN", None)
    assert c.message_bins == 0
    assert r1.iterations == r2.iterations == c.iterations
    np.testing.assert_array_equal(_bits(r1.means), _bits(c.means))
    np.testing.assert_array_equal(_bits(r1.means), _bits(r2.means))
    assert list(r1.residual_history) == list(r2.residual_history)
    np.testing.assert_array_equal(np.asarray(r1.max_change_history),
                                  np.asarray(c.max_change_history))
