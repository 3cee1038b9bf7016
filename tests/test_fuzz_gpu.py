"""Randomised systems of many shapes through the drop-in solve(), both synchronous
schedules, automatic kernel choice (cluster solve, diagonal layout, slice groups, four rows
per warp, dense) -- every result bitwise the C oracle's."""

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


def _system(rng, n, mean_deg, hubs, dominance, isolated):
    m = int(n * mean_deg / 2)
    pi = rng.integers(0, n, m)
    pj = rng.integers(0, n, m)
    for h in range(hubs):  # a few rows of 70..250 edges (the long-row paths)
        k = int(rng.integers(70, min(250, n - 1) + 1)) if n > 80 else 0
        pi = np.concatenate([pi, np.full(k, h)])
        pj = np.concatenate([pj, rng.choice(np.arange(hubs, n), k, replace=False)])
    if isolated:
        lone = rng.choice(n, max(1, n // 10), replace=False)
        keep = ~(np.isin(pi, lone) | np.isin(pj, lone))
        pi, pj = pi[keep], pj[keep]
    keep = pi != pj
    lo, hi = np.minimum(pi[keep], pj[keep]), np.maximum(pi[keep], pj[keep])
    key = np.unique(lo.astype(np.int64) * n + hi)
    pi, pj = key // n, key % n
    pv = rng.uniform(-1.0, 1.0, pi.size)
    pv[pv == 0.0] = 0.25
    absrow = np.bincount(pi, np.abs(pv), n) + np.bincount(pj, np.abs(pv), n)
    diag = dominance * absrow + (absrow == 0) * rng.uniform(0.5, 2.0, n)
    return G.SymSystem.from_pairs(diag, pi, pj, pv, rng.standard_normal(n))


CASES = []
_rng = np.random.default_rng(2024)
for _n in (1, 2, 7, 33, 150, 900, 2500, 7000, 20000, 60000):
    for _deg in (1.5, 5.0, 13.0, 30.0, 55.0):
        if _deg >= _n:
            continue
        for _rep in range(3):
            CASES.append((_n, _deg, int(_n > 300 and _rng.random() < 0.5) * 2,
                          float(_rng.choice([1.05, 1.3, 0.8])), bool(_rng.random() < 0.3),
                          int(_rng.integers(1 << 30))))


@pytest.mark.parametrize("n,deg,hubs,dom,iso,seed", CASES)
@pytest.mark.parametrize("sched", ["broadcast", "parallel"])
def test_random_system_matches_oracle(n, deg, hubs, dom, iso, seed, sched):
    s = _system(np.random.default_rng(seed), n, deg, hubs, dom, iso)
    kw = dict(epsilon=1e-9, max_iter=60)
    og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
    o = oracle.solve(og, schedule=sched, **kw)
    r = G.solve(s, G.SolveOptions(schedule=sched, **kw))
    assert (r.iterations, r.converged, r.diverged) == (o.iterations, o.converged, o.diverged)
    np.testing.assert_array_equal(_bits(np.asarray(r.max_change_history)),
                                  _bits(o.max_change_history))
    fin = np.isfinite(o.means)
    np.testing.assert_array_equal(np.isfinite(r.means), fin)
    np.testing.assert_array_equal(_bits(r.means[fin]), _bits(o.means[fin]))
    if o.iterations and np.all(np.isfinite(o.residual_history)):
        # (1e-9 relative, plus the cancellation floor: a residual at rounding level depends
        # on the summation order)
        np.testing.assert_allclose(r.residual_history, o.residual_history, rtol=1e-9,
                                   atol=1e-12 * o.residual_history[0])
