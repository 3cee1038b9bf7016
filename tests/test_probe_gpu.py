"""Residual probe: a launch that expects the previous sweep to
end the solve runs residual-only and decides it one launch early; when that expectation is
wrong the next launch runs the full sweep.  GABP_PROBE_FORCE=1 requests a probe after
every launch, so every mispredicted path runs; results must stay bitwise the oracle's
(iterations, means, precisions, change history) on both schedules and every slice kernel
variant.  The child processes read the environment once, at library load."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_0810_1119_b200 as G
from oracle import oracle
from tests import golden_cases as gc

oracle.build()
systems = [gc.system(gc.load(c)) for c in gc.names()]
systems += [G.gen_random_sparse(1 << 14, 16, 5).system, G.gen_poisson2d(64, 2).system]
probes = 0
for s in systems:
    og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
    g = G.build_graph(s)
    for sched in ("broadcast", "parallel"):
        for kw in (dict(epsilon=1e-300, max_iter=60, rel_residual_tol=1e-8),
                   dict(epsilon=1e-7, max_iter=400), dict(epsilon=1e-300, max_iter=7)):
            o = oracle.solve(og, schedule=sched, **kw)
            r = G.solve_graph(g, G.SolveOptions(schedule=sched, **kw))
            probes += r.residual_probes
            assert (r.iterations, r.converged, r.diverged) == (o.iterations, o.converged,
                                                               o.diverged), (sched, kw)
            np.testing.assert_array_equal(r.means, o.means)
            np.testing.assert_array_equal(r.precisions, o.precisions)
            np.testing.assert_array_equal(np.asarray(r.max_change_history),
                                          o.max_change_history)
print("probes", probes)
"""


def _run(env_extra):
    env = dict(os.environ)
    env.update(env_extra)
    p = subprocess.run([sys.executable, "-c", CHILD, REPO], env=env, cwd=REPO,
                       capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-4000:]
    return int(p.stdout.split("probes")[-1])


@pytest.mark.parametrize("variant", ["2", "0", "1"])
def test_forced_probes_bitwise(variant):
    probes = _run({"GABP_PROBE_FORCE": "1", "GABP_SLICE_VARIANT": variant})
    assert probes > 0


def test_probes_fire_on_certain_decisions():
    # no forcing: the epsilon and sweep-cap decisions are certain one launch early
    assert _run({}) > 0
