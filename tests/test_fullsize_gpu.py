"""BASELINE configs 2 (Poisson 4096^2) and 4 (Poisson 512^3) at full size, through the real
solve loop and the real row-block partitions.

* 4096^2: 200 sweeps of solve() from zero messages, bitwise against the C oracle -- the
  diagonal-layout kernel (auto), the slice layout, and the parallel schedule.  Solving to
  1e-8 is out of reach for any GaBP here: sweeps to 1e-8 grow ~N^2 (455, 1731, 6185, 22781
  sweeps at 16^2, 32^2, 64^2, 128^2 with the oracle), so long bitwise prefixes are the bar.
* 4096^2 in 2, 4 and 8 row strips (in-process partitions on one GPU: the multi-rank kernels,
  halo lists and decision, device-copy transport), 120 sweeps, bitwise the one-partition
  solve, with the split boundary/interior sweep engaged on every strip.
* 512^3: 40 sweeps at full size (804 M directed edges); marginals on two sub-boxes of 100^3
  bitwise the oracle's on the restricted system (after T sweeps a marginal depends only on
  rows within T+1 hops).
* 400^3 (the largest cube that fits twice) in 2, 4 and 8 slabs, 100 sweeps, bitwise the
  one-partition solve.
The grids are generated on the device (grid.py: b ~ N(0,1) from a seeded Philox stream).
"""

import numpy as np
import pytest

import paper_0810_1119_b200 as G
from oracle import oracle
from paper_0810_1119_b200 import _lib, dist as D, grid as GR, problems as P

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    _lib.load()
    assert _lib.device_count() > 0, "no CUDA device: " + _lib.last_error()
    oracle.build()
    import os
    oracle.set_threads(os.cpu_count() or 1)


@pytest.fixture(autouse=True)
def _fresh_memory():
    yield
    _lib.release_cached(0)  # (the 400^3 partitions need the memory earlier tests cached)


def _bits(a):
    return np.asarray(a, dtype=np.float64).view(np.uint64)


def _same(a, b, res=True):
    assert (a.iterations, a.converged, a.diverged) == (b.iterations, b.converged, b.diverged)
    np.testing.assert_array_equal(_bits(a.means), _bits(b.means))
    np.testing.assert_array_equal(_bits(a.precisions), _bits(b.precisions))
    np.testing.assert_array_equal(np.asarray(a.max_change_history),
                                  np.asarray(b.max_change_history))
    if res:
        np.testing.assert_allclose(a.residual_history, b.residual_history, rtol=1e-9, atol=0)


@pytest.fixture(scope="module")
def grid4096():
    spec = GR.GridSpec(2, 4096, 0)
    g = GR.GridGraph(spec, 0, keep_arrays=True)
    host = g.host_arrays()
    yield spec, g, host
    g.close()


@pytest.mark.parametrize("sched", ["broadcast", "parallel"])
def test_config2_4096_200_sweeps_vs_oracle(grid4096, sched):
    spec, g, (diag, rhs, pi, pj, pv) = grid4096
    T = 200
    og = oracle.build_graph(diag, rhs, pi, pj, pv)
    o = oracle.solve(og, epsilon=1e-300, max_iter=T, schedule=sched)
    assert o.iterations == T
    modes = ("auto", "slice") if sched == "broadcast" else ("auto",)
    for mode in modes:
        r = G.solve_graph(g, G.SolveOptions(schedule=sched, epsilon=1e-300, max_iter=T,
                                            gather_mode=mode, record_means_history=False))
        assert (r.iterations, r.diverged) == (T, True), mode  # the sweep cap
        np.testing.assert_array_equal(_bits(r.means), _bits(o.means))
        np.testing.assert_array_equal(_bits(r.precisions), _bits(o.precisions))
        np.testing.assert_array_equal(np.asarray(r.max_change_history), o.max_change_history)
        np.testing.assert_allclose(r.residual_history, o.residual_history, rtol=1e-9, atol=0)
    if sched == "broadcast":
        assert g.info.dia_diagonals == 4  # (auto ran the diagonal layout)


@pytest.mark.parametrize("layout", ["diagonal", "slice"])
@pytest.mark.parametrize("nparts", [2, 4, 8])
def test_config2_4096_strips_bitwise_one_partition(grid4096, nparts, layout, monkeypatch):
    """diagonal: the ranks' stencil layout (message + node-state halo per cut edge);
    slice: the slice layout with the split sweep (boundary rows first, the exchange under
    the interior rows)."""
    spec, g, _ = grid4096
    if layout == "slice":
        monkeypatch.setenv("GABP_NO_DIST_DIA", "1")
    opts = G.SolveOptions(schedule="broadcast", epsilon=1e-300, max_iter=120,
                          record_means_history=False)
    one = G.solve_graph(g, opts)
    part = D.solve_grid_partitioned_local(spec, nparts, opts)
    if layout == "slice":
        assert part.dist_layout == 1 and part.split_sweeps > 0
    else:
        assert part.dist_layout == 3
    _same(part, one)


def test_config4_512_full_size_locality_vs_oracle():
    spec = GR.GridSpec(3, 512, 0)
    T, L, p = 40, 100, 512
    g = GR.GridGraph(spec, 0)
    try:
        r = G.solve_graph(g, G.SolveOptions(schedule="broadcast", epsilon=1e-300, max_iter=T,
                                            record_means_history=False))
    finally:
        g.close()
    assert r.iterations == T
    rhs = GR.rhs_device(spec, 0).cpu().numpy()
    margin = T + 2  # from a cut face
    for lo in ((0, 0, 0), (200, 300, 100)):
        z, y, x = np.meshgrid(*(np.arange(c, c + L) for c in lo), indexing="ij")
        glob = (z * p * p + y * p + x).ravel()
        pi, pj = P._grid3d_pairs(L)  # the box's own grid, lexicographic = ascending
        og = oracle.build_graph(np.full(L ** 3, 6.0), rhs[glob], pi, pj,
                                np.full(pi.size, -1.0))
        o = oracle.solve(og, epsilon=1e-300, max_iter=T, schedule="broadcast")
        assert o.iterations == T
        k = np.arange(L)
        ok = [(k >= (0 if c == 0 else margin)) & (k < L - margin) for c in lo]
        inner = (ok[0][:, None, None] & ok[1][None, :, None] & ok[2][None, None, :]).ravel()
        assert inner.sum() >= 4096  # (interior box: (100 - 2 x 42)^3)
        np.testing.assert_array_equal(_bits(r.means[glob[inner]]), _bits(o.means[inner]))
        np.testing.assert_array_equal(_bits(r.precisions[glob[inner]]),
                                      _bits(o.precisions[inner]))


@pytest.fixture(scope="module")
def cube400():
    spec = GR.GridSpec(3, 400, 1)
    g = GR.GridGraph(spec, 0)
    opts = G.SolveOptions(schedule="broadcast", epsilon=1e-300, max_iter=100,
                          record_means_history=False)
    one = G.solve_graph(g, opts)
    g.close()
    return spec, opts, one


@pytest.mark.parametrize("layout", ["diagonal", "slice"])
@pytest.mark.parametrize("nparts", [2, 4, 8])
def test_config4_400_cube_slabs_bitwise_one_partition(cube400, nparts, layout, monkeypatch):
    spec, opts, one = cube400
    if layout == "slice":
        monkeypatch.setenv("GABP_NO_DIST_DIA", "1")
    part = D.solve_grid_partitioned_local(spec, nparts, opts)
    if layout == "slice":
        assert part.dist_layout == 1 and part.split_sweeps > 0
    else:
        assert part.dist_layout == 3
    _same(part, one)
