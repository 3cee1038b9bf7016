"""CPU-only checks: the C-ABI library loads and exports every declared symbol, host-side
API mirrors the reference (options validation, storage conversions, generators)."""

import os
import re

import numpy as np
import pytest

import paper_0810_1119_b200 as G
from paper_0810_1119_b200 import _lib

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for fn in os.listdir(os.path.join(REPO, "include")):
        if fn.endswith(".h"):
            text = open(os.path.join(REPO, "include", fn)).read()
            names |= set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(gabp_\w+)\s*\(", text, re.M))
    return names


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    declared = _declared()
    assert len(declared) >= 20
    for name in sorted(declared):
        assert hasattr(lib, name), name
    assert set(_lib.EXPORTED) == declared


def test_library_reports_no_device_without_gpu():
    # the CPU container has no driver: the library must say so, not fall back
    if _lib.device_count() == 0:
        assert _lib.last_error()


def test_solve_options_validation():
    with pytest.raises(ValueError):
        G.SolveOptions(epsilon=0.0)
    with pytest.raises(ValueError):
        G.SolveOptions(max_iter=0)
    with pytest.raises(ValueError):
        G.SolveOptions(blowup=1.0)
    with pytest.raises(ValueError):
        G.SolveOptions(schedule="bogus")


def test_serial_schedule_options():
    """The serial schedule runs on the device (gabp_sweep_serial, dependency levels); it
    has no slice / row-kernel gather modes and no device solve-loop options struct."""
    G.SolveOptions(schedule="serial", serial_order=[2, 0, 1])
    for mode in ("slice", "rows"):
        with pytest.raises(ValueError):
            G.SolveOptions(schedule="serial", gather_mode=mode)
    with pytest.raises(ValueError, match="synchronous"):
        G.solver._gpu_schedule("serial")


def test_symsystem_forms_agree():
    a = np.array([[4.0, -1.0, 0.5], [-1.0, 3.0, 0.0], [0.5, 0.0, 2.0]])
    s = G.SymSystem.from_dense(a, np.ones(3))
    assert s.offdiag == {(0, 1): -1.0, (0, 2): 0.5}
    np.testing.assert_array_equal(s.to_dense()[0], a)
    t = G.SymSystem(diag=[4.0, 3.0, 2.0], offdiag={(0, 1): -1.0, (0, 2): 0.5}, rhs=np.ones(3))
    np.testing.assert_array_equal(t.matvec(np.arange(3.0)), a @ np.arange(3.0))
    with pytest.raises(ValueError, match="explicit zero"):
        G.SymSystem(diag=np.ones(2), offdiag={(0, 1): 0.0}, rhs=np.ones(2))
    with pytest.raises(ValueError, match="bad off-diagonal"):
        G.SymSystem(diag=np.ones(2), offdiag={(1, 0): 1.0}, rhs=np.ones(2))
    with pytest.raises(ValueError, match="not symmetric"):
        G.SymSystem.from_dense(np.array([[1.0, 2.0], [3.0, 1.0]]), np.ones(2))


def test_residual_norm_per_eq_toy3():
    s = G.load_instance("toy3").system
    assert G.residual_norm_per_eq(s, np.array([1.0, 2.0, -1.0])) == 0.0
    assert G.residual_norm_per_eq(s, np.zeros(3)) == pytest.approx(np.sqrt(40.0) / 3)


def test_poisson_matrix_exact():
    a, b = G.gen_poisson(3).system.to_dense()
    assert a[4].tolist() == [0, -1, 0, -1, 4, -1, 0, -1, 0]
    assert np.all(b == 1.0 / 16.0)


def test_generators_deterministic_and_dominant():
    s1 = G.gen_random_sparse(5000, 16, 7).system
    s2 = G.gen_random_sparse(5000, 16, 7).system
    np.testing.assert_array_equal(s1.pair_v, s2.pair_v)
    assert G.dominance_class(s1) == "strict"
    assert np.all(s1.pair_i < s1.pair_j)
    keys = s1.pair_i * s1.n + s1.pair_j
    assert np.unique(keys).size == keys.size
    p3 = G.gen_poisson3d(5, 0).system
    assert p3.pair_v.size == 3 * 5 * 5 * 4 and np.all(p3.diag == 6.0)
    inst, s = G.gen_cdma_detection(64, 16, 0.5, 1)
    a, _ = inst.system.to_dense()
    np.testing.assert_array_equal(a, a.T)
    np.testing.assert_allclose(np.diag(a), 1.5)


# ---- host planning of the one-launch cluster solve (csrc/small.cu: small_plan) -----------

def _small_plan(row_ptr):
    import ctypes
    lib = _lib.load()
    rp = np.ascontiguousarray(row_ptr, dtype=np.uint32)
    bounds = np.zeros(9, dtype=np.int64)
    ce, cr = ctypes.c_int64(), ctypes.c_int64()
    C = lib.gabp_small_plan(rp.size - 1, rp.ctypes.data, bounds.ctypes.data,
                            ctypes.byref(ce), ctypes.byref(cr))
    return C, bounds[:C + 1], ce.value, cr.value


def _grid_row_ptr(p):
    deg = np.full((p, p), 4)
    deg[0, :] -= 1
    deg[-1, :] -= 1
    deg[:, 0] -= 1
    deg[:, -1] -= 1
    return np.concatenate([[0], np.cumsum(deg.ravel())])


def test_small_plan_config0_eight_balanced_blocks():
    rp = _grid_row_ptr(32)  # config 0: 1024 rows, 3968 edge slots
    C, b, ce, cr = _small_plan(rp)
    assert C == 8 and b[0] == 0 and b[-1] == 1024
    assert np.all(np.diff(b) > 0)
    edges = rp[b[1:]] - rp[b[:-1]]
    rows = np.diff(b)
    assert edges.max() <= ce and rows.max() <= cr
    assert edges.max() - edges.min() <= 16 and rows.max() - rows.min() <= 8


def test_small_plan_covers_every_row_once_and_respects_capacity():
    rng = np.random.default_rng(7)
    for n, lam in ((3, 1.0), (50, 3.0), (700, 6.0), (3000, 4.0), (6000, 2.0), (64, 40.0)):
        deg = rng.poisson(lam, n)
        rp = np.concatenate([[0], np.cumsum(deg)])
        C, b, ce, cr = _small_plan(rp)
        assert C in (1, 2, 4, 8), (n, lam)
        assert b[0] == 0 and b[-1] == n and np.all(np.diff(b) >= 0)
        assert (rp[b[1:]] - rp[b[:-1]]).max() <= ce
        assert np.diff(b).max() <= cr


def test_small_plan_rejects_what_no_cluster_holds():
    # a hub row wider than any CTA's edge capacity; a graph with too many rows
    rp = np.concatenate([[0], np.cumsum([2500] + [1] * 2500)])
    assert _small_plan(rp)[0] == 0
    assert _small_plan(np.arange(0, 4 * 20001, 4))[0] == 0
    # one CTA's worth of work stays on one CTA
    assert _small_plan(np.arange(0, 3 * 41, 3))[0] == 1
