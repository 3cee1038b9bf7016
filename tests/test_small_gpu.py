"""Small graphs: the whole broadcast solve in one launch of one thread-block cluster
(csrc/small.cu: row blocks over <= 8 CTAs, distributed shared memory) --
BASELINE config 0, the reference's own case (Poisson 32x32 to ||Ax-b||/||b|| < 1e-8,
1731 sweeps), bitwise against the C oracle and against the sweep-per-launch slice loop.
The golden fixtures run through it in tests/test_gpu_parity.py (gather mode auto)."""

import numpy as np
import pytest

import paper_0810_1119_b200 as G
from oracle import oracle
from paper_0810_1119_b200 import _lib

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    _lib.load()
    assert _lib.device_count() > 0, "no CUDA device: " + _lib.last_error()
    oracle.build()


def _bits(a):
    return np.asarray(a, dtype=np.float64).view(np.uint64)


@pytest.mark.parametrize("kw", [dict(epsilon=1e-300, rel_residual_tol=1e-8),
                                dict(epsilon=1e-9),
                                dict(epsilon=1e-300, max_iter=7)])
def test_config0_one_cta_matches_oracle_and_slice_loop(kw):
    s = G.gen_poisson2d(32, 0).system
    og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
    o = oracle.solve(og, schedule="broadcast", **kw)
    r = G.solve(s, G.SolveOptions(schedule="broadcast", record_means_history=True, **kw))
    assert r.kernel_launches == 1  # the persistent CTA ran the whole loop
    assert (r.iterations, r.converged, r.diverged) == (o.iterations, o.converged, o.diverged)
    np.testing.assert_array_equal(_bits(r.means), _bits(o.means))
    np.testing.assert_array_equal(_bits(r.precisions), _bits(o.precisions))
    np.testing.assert_array_equal(np.asarray(r.max_change_history), o.max_change_history)
    np.testing.assert_allclose(r.residual_history, o.residual_history, rtol=1e-9, atol=0)
    sl = G.solve(s, G.SolveOptions(schedule="broadcast", record_means_history=True,
                                   gather_mode="slice", **kw))
    assert sl.iterations == r.iterations
    assert len(r.means_history) == len(sl.means_history) == r.iterations
    for t in range(0, r.iterations, max(1, r.iterations // 7)):
        np.testing.assert_array_equal(_bits(r.means_history[t]), _bits(sl.means_history[t]))
    np.testing.assert_array_equal(_bits(r.means_history[-1]), _bits(r.means))


def test_config0_rel_residual_reached_and_fast():
    s = G.gen_poisson2d(32, 0).system
    opts = G.SolveOptions(schedule="broadcast", epsilon=1e-300, rel_residual_tol=1e-8,
                          record_means_history=False)
    g = G.build_graph(s)
    try:
        G.solve_graph(g, opts)
        r = G.solve_graph(g, opts)
    finally:
        g.close()
    rel = np.linalg.norm(s.matvec(r.means) - s.rhs) / np.linalg.norm(s.rhs)
    assert r.converged and rel < 1e-8
    assert r.iterations == 1731
    # (not a benchmark: a loose bound that the launch-per-sweep loop, ~16-20 us per sweep,
    # cannot meet)
    assert r.device_ms / r.iterations < 10e-3, r.device_ms


@pytest.mark.parametrize("n,k", [(700, 3), (1500, 1), (64, 20), (3000, 2), (6000, 1)])
def test_random_small_graphs_match_oracle(n, k):
    s = G.gen_random_sparse(n, k, 11).system
    og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
    kw = dict(epsilon=1e-300, rel_residual_tol=1e-11, max_iter=500)
    o = oracle.solve(og, schedule="broadcast", **kw)
    r = G.solve(s, G.SolveOptions(schedule="broadcast", **kw))
    assert r.kernel_launches == 1
    assert r.iterations == o.iterations
    np.testing.assert_array_equal(_bits(r.means), _bits(o.means))
    np.testing.assert_array_equal(np.asarray(r.max_change_history), o.max_change_history)


def test_cluster_divergence_matches_oracle():
    """A dense CDMA system of 96 users (9120 directed edges over 8 CTAs): GaBP blows up on
    it; the divergent trajectory, its stop sweep and flags are the oracle's."""
    s = G.gen_cdma_detection(192, 96, 0.5, 3)[0].system
    og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
    kw = dict(epsilon=1e-12, max_iter=400)
    o = oracle.solve(og, schedule="broadcast", **kw)
    r = G.solve(s, G.SolveOptions(schedule="broadcast", **kw))
    assert r.kernel_launches == 1
    assert (r.iterations, r.converged, r.diverged) == (o.iterations, o.converged, o.diverged)
    np.testing.assert_array_equal(_bits(r.means), _bits(o.means))
    np.testing.assert_array_equal(_bits(np.asarray(r.max_change_history)),
                                  _bits(o.max_change_history))


def test_hub_row_larger_than_a_cta_takes_the_launch_per_sweep_path():
    """A star with a hub of 2500 edges: no CTA of the cluster can hold the hub's row, so the
    solve runs one launch per sweep -- same results as the oracle."""
    n = 2501
    pi = np.zeros(n - 1, dtype=np.int64)
    pj = np.arange(1, n, dtype=np.int64)
    rng = np.random.default_rng(5)
    pv = rng.uniform(-1.0, 1.0, n - 1)
    diag = np.full(n, 2.0)
    diag[0] = 1.1 * np.abs(pv).sum()
    s = G.SymSystem.from_pairs(diag, pi, pj, pv, rng.standard_normal(n))
    og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
    kw = dict(epsilon=1e-10, max_iter=200)
    o = oracle.solve(og, schedule="broadcast", **kw)
    r = G.solve(s, G.SolveOptions(schedule="broadcast", **kw))
    assert r.kernel_launches > 1
    assert r.iterations == o.iterations
    np.testing.assert_array_equal(_bits(r.means), _bits(o.means))


@pytest.mark.parametrize("kw", [dict(epsilon=1e-300, rel_residual_tol=1e-8),
                                dict(epsilon=1e-9), dict(epsilon=1e-300, max_iter=7)])
def test_config0_parallel_schedule_in_the_cluster(kw):
    """The reference's default schedule (solver.py:146-173) through the cluster kernel:
    exclusion sums over the row's local slots, bitwise the oracle."""
    s = G.gen_poisson2d(32, 0).system
    og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
    o = oracle.solve(og, schedule="parallel", **kw)
    r = G.solve(s, G.SolveOptions(schedule="parallel", record_means_history=True, **kw))
    assert r.kernel_launches == 1
    assert (r.iterations, r.converged, r.diverged) == (o.iterations, o.converged, o.diverged)
    np.testing.assert_array_equal(_bits(r.means), _bits(o.means))
    np.testing.assert_array_equal(_bits(r.precisions), _bits(o.precisions))
    np.testing.assert_array_equal(np.asarray(r.max_change_history), o.max_change_history)
    np.testing.assert_allclose(r.residual_history, o.residual_history, rtol=1e-9, atol=0)
    assert len(r.means_history) == r.iterations
    np.testing.assert_array_equal(_bits(r.means_history[-1]), _bits(r.means))


@pytest.mark.parametrize("n,k", [(700, 3), (64, 20), (3000, 2)])
def test_random_small_graphs_parallel_match_oracle(n, k):
    s = G.gen_random_sparse(n, k, 12).system
    og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
    kw = dict(epsilon=1e-300, rel_residual_tol=1e-11, max_iter=500)
    o = oracle.solve(og, schedule="parallel", **kw)
    r = G.solve(s, G.SolveOptions(schedule="parallel", **kw))
    assert r.kernel_launches == 1
    assert r.iterations == o.iterations
    np.testing.assert_array_equal(_bits(r.means), _bits(o.means))
    np.testing.assert_array_equal(np.asarray(r.max_change_history), o.max_change_history)


def test_cluster_parallel_divergence_matches_oracle():
    s = G.gen_cdma_detection(192, 96, 0.5, 3)[0].system
    og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
    kw = dict(epsilon=1e-12, max_iter=400)
    o = oracle.solve(og, schedule="parallel", **kw)
    r = G.solve(s, G.SolveOptions(schedule="parallel", **kw))
    assert r.kernel_launches == 1
    assert (r.iterations, r.converged, r.diverged) == (o.iterations, o.converged, o.diverged)
    np.testing.assert_array_equal(_bits(r.means), _bits(o.means))
    np.testing.assert_array_equal(_bits(np.asarray(r.max_change_history)),
                                  _bits(o.max_change_history))
