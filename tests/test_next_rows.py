"""Rows beside the sweep (DESIGN.md row f): Matrix Market / vector I/O, the augmented
least-squares embedding, and the Steffensen / Aitken wrappers -- against fixtures made by
running the reference itself (tests/golden/make_golden_next.py)."""

import glob
import json
import os

import numpy as np
import pytest

import paper_0810_1119_b200 as G
from paper_0810_1119_b200 import acceleration as A
from paper_0810_1119_b200 import linalg as L
from paper_0810_1119_b200 import pseudoinverse as PI

NEXT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "next")
MM = json.load(open(os.path.join(NEXT, "mm_cases.json")))


def _npz(path):
    with np.load(path) as z:
        return {k: z[k] for k in z.files}


def _bits(a):
    return np.asarray(a, dtype=np.float64).view(np.uint64)


# ---- Matrix Market / vector text I/O (CPU) -----------------------------------------------

@pytest.mark.parametrize("k", range(len(MM["cases"])))
def test_matrix_market_parse_write_vs_reference(k):
    case = MM["cases"][k]
    r = L.parse_matrix_market(case["text"])
    assert (r.m, r.n) == (case["m"], case["n"])
    got = [[i, j, repr(v)] for (i, j), v in r.entries.items()]
    assert got == case["entries"]  # same entries, values and dict order
    assert L.write_matrix_market(r) == case["write"]
    if "system" in case:
        s = L.system_from_matrix_market(case["text"], np.arange(r.m, dtype=float))
        assert [repr(v) for v in s.diag] == case["system"]["diag"]
        assert [[i, j, repr(v)] for (i, j), v in s.offdiag.items()] == case["system"]["pairs"]
        assert L.write_matrix_market(s) == case["system"]["write"]
    if "system_error" in case:
        with pytest.raises(L.MatrixMarketError, match=None) as ei:
            L.system_from_matrix_market(case["text"], np.arange(r.m, dtype=float))
        assert str(ei.value) == case["system_error"]


@pytest.mark.parametrize("k", range(len(MM["errors"])))
def test_matrix_market_errors_vs_reference(k):
    case = MM["errors"][k]
    if case["error"] is None:
        L.parse_matrix_market(case["text"])
        return
    with pytest.raises(ValueError) as ei:
        L.parse_matrix_market(case["text"])
    assert type(ei.value).__name__ == case["type"]
    assert str(ei.value) == case["error"]


@pytest.mark.parametrize("k", range(len(MM["system_errors"])))
def test_system_from_matrix_market_errors_vs_reference(k):
    case = MM["system_errors"][k]
    with pytest.raises(ValueError) as ei:
        L.system_from_matrix_market(case["text"], np.zeros(2))
    assert str(ei.value) == case["error"]


def test_vector_io_vs_reference():
    v = MM["vector"]
    vals = [float(x) for x in v["values"]]
    assert L.write_vector(vals) == v["text"]
    assert [repr(x) for x in L.parse_vector("\n" + v["text"] + "\n\n")] == v["parsed"]
    with pytest.raises(L.MatrixMarketError):
        L.parse_vector("\n \n")


def test_matrix_market_large_roundtrip():
    """A 200k-entry symmetric file takes the vectorised path and round-trips exactly."""
    s = G.gen_random_sparse(20000, 5, 3).system
    text = L.write_matrix_market(s)
    s2 = L.system_from_matrix_market(text, s.rhs)
    np.testing.assert_array_equal(_bits(s2.diag), _bits(s.diag))
    a = np.lexsort((s.pair_j, s.pair_i))
    b = np.lexsort((s2.pair_j, s2.pair_i))
    np.testing.assert_array_equal(s2.pair_i[b], s.pair_i[a])
    np.testing.assert_array_equal(s2.pair_j[b], s.pair_j[a])
    np.testing.assert_array_equal(_bits(s2.pair_v[b]), _bits(s.pair_v[a]))


# ---- augmented least squares: the embedding (CPU) ------------------------------------------

LSQ = sorted(glob.glob(os.path.join(NEXT, "lsq_*.npz")))


@pytest.mark.parametrize("path", LSQ, ids=os.path.basename)
def test_build_augmented_vs_reference(path):
    rec = _npz(path)
    s = L.RectMatrix.from_dense(rec["dense"])
    aug = PI.build_augmented(s, rec["y"], float(rec["psi"]))
    a = aug.assembled
    np.testing.assert_array_equal(_bits(a.diag), _bits(rec["aug_diag"]))
    np.testing.assert_array_equal(_bits(a.rhs), _bits(rec["aug_rhs"]))
    np.testing.assert_array_equal(a.pair_i, rec["aug_pair_i"])
    np.testing.assert_array_equal(a.pair_j, rec["aug_pair_j"])
    np.testing.assert_array_equal(_bits(a.pair_v), _bits(rec["aug_pair_v"]))
    np.testing.assert_array_equal(PI.normal_equations_oracle(s, rec["y"], float(rec["psi"])),
                                  rec["oracle"])


def test_build_augmented_rejects():
    s = L.RectMatrix.from_dense(np.ones((3, 2)))
    with pytest.raises(ValueError):
        PI.build_augmented(s, np.zeros(3), 0.0)
    with pytest.raises(ValueError):
        PI.build_augmented(s, np.zeros(2), 1e-3)


# ---- acceleration: host utilities and configuration (CPU) ----------------------------------

def test_aitken_extrapolate_exact_cases():
    assert A.aitken_extrapolate(np.array([5.0]), np.array([3.5]), np.array([2.75]))[0] == 2.0
    np.testing.assert_array_equal(
        A.aitken_extrapolate(np.array([3.0, -1.0]), np.array([3.0, -1.0]),
                             np.array([3.0, -1.0])), [3.0, -1.0])
    with pytest.raises(ValueError):
        A.aitken_extrapolate(np.zeros(2), np.zeros(3), np.zeros(3))


def test_accel_config_and_dispatch_errors():
    with pytest.raises(ValueError):
        A.AccelConfig(mode="nesterov")
    with pytest.raises(ValueError):
        A.AccelConfig(denom_guard=0.0)
    with pytest.raises(ValueError):
        A.AccelConfig(target="messages")
    s = G.load_instance("cdma3").system
    with pytest.raises(ValueError):
        A.accelerated_solve("cg", s, G.SolveOptions())
    with pytest.raises(ValueError):  # classical base solvers are not on the GPU path
        A.steffensen_solve("jacobi", s)


# ---- acceleration on the device (GPU) -------------------------------------------------------

ACCEL = sorted(glob.glob(os.path.join(NEXT, "accel_*.npz")))


def _same_report(r, rec, prefix, exact_means=True):
    assert int(r.converged) == int(rec[f"{prefix}_converged"])
    assert int(r.diverged) == int(rec[f"{prefix}_diverged"])
    assert r.iterations == int(rec[f"{prefix}_iterations"])
    np.testing.assert_array_equal(_bits(r.max_change_history), _bits(rec[f"{prefix}_change"]))
    np.testing.assert_array_equal(_bits(r.means), _bits(rec[f"{prefix}_means"]))
    np.testing.assert_array_equal(_bits(r.precisions), _bits(rec[f"{prefix}_precisions"]))
    mh = rec[f"{prefix}_means_history"]
    assert len(r.means_history) == mh.shape[0]
    for got, want in zip(r.means_history, mh):
        np.testing.assert_array_equal(_bits(got), _bits(want))
    want = rec[f"{prefix}_residual"]
    fin = np.isfinite(want)
    np.testing.assert_array_equal(np.isfinite(r.residual_history), fin)
    np.testing.assert_allclose(np.asarray(r.residual_history)[fin], want[fin], rtol=1e-9,
                               atol=1e-15)


@pytest.mark.gpu
@pytest.mark.parametrize("sched", ["parallel", "broadcast"])
@pytest.mark.parametrize("path", ACCEL, ids=os.path.basename)
def test_steffensen_and_aitken_bitwise_vs_reference(path, sched):
    rec = _npz(path)
    s = L.SymSystem.from_pairs(rec["diag"], rec["pair_i"], rec["pair_j"], rec["pair_v"],
                               rec["rhs"])
    opts = G.SolveOptions(schedule=sched)
    _same_report(A.steffensen_solve("gabp", s, opts), rec, f"{sched}_steff")
    _same_report(A.aitken_solve("gabp", s, opts), rec, f"{sched}_aitken")
    _same_report(A.steffensen_solve("gabp", s, opts, A.AccelConfig(stability=0.0)), rec,
                 f"{sched}_steff_s0")


ACCEL_SERIAL = sorted(glob.glob(os.path.join(os.path.dirname(NEXT), "serial", "accel_*.npz")))


@pytest.mark.gpu
@pytest.mark.parametrize("path", ACCEL_SERIAL, ids=os.path.basename)
def test_steffensen_and_aitken_serial_bitwise_vs_reference(path):
    """Acceleration around the serial schedule (device dependency levels)."""
    rec = _npz(path)
    s = L.SymSystem.from_pairs(rec["diag"], rec["pair_i"], rec["pair_j"], rec["pair_v"],
                               rec["rhs"])
    opts = G.SolveOptions(schedule="serial")
    _same_report(A.steffensen_solve("gabp", s, opts), rec, "serial_steff")
    _same_report(A.aitken_solve("gabp", s, opts), rec, "serial_aitken")


@pytest.mark.gpu
def test_accelerated_solve_dispatch_gpu():
    s = G.load_instance("cdma3").system
    none = A.accelerated_solve("gabp", s, G.SolveOptions())
    assert none.iterations == G.solve(s, G.SolveOptions()).iterations
    st = A.accelerated_solve("gabp", s, G.SolveOptions(), A.AccelConfig(mode="steffensen"))
    assert st.converged and st.iterations < none.iterations
    with pytest.raises(ValueError):  # restarts replace mean messages only (GaBP)
        A.steffensen_solve("gabp", s, G.SolveOptions(),
                           A.AccelConfig(target="solution_vector"))


@pytest.mark.gpu
def test_steffensen_large_graph_device_restart():
    """Config-1-shaped graph (65k rows): Steffensen runs with its states in HBM and reaches
    the plain solve's answer."""
    s = G.gen_random_sparse(1 << 16, 16, 5).system
    opts = G.SolveOptions(schedule="broadcast", epsilon=1e-10, max_iter=400)
    st = A.steffensen_solve("gabp", s, opts)
    plain = G.solve(s, opts)
    assert st.converged and plain.converged
    np.testing.assert_allclose(st.means, plain.means, atol=1e-8)


# ---- augmented least squares: the solve (GPU) ----------------------------------------------

LSQ_DEFAULT = sorted(glob.glob(os.path.join(os.path.dirname(NEXT), "serial", "lsq_*.npz")))


@pytest.mark.gpu
@pytest.mark.parametrize("path", LSQ_DEFAULT, ids=os.path.basename)
def test_solve_least_squares_default_options_vs_reference(path):
    """The reference's default options (serial schedule, epsilon 1e-10): same x bit for
    bit, or the same divergence with the same spectral diagnostic."""
    rec = _npz(path)
    s = L.RectMatrix.from_dense(rec["dense"])
    if int(rec["diverged"]):
        with pytest.raises(PI.LeastSquaresDivergence) as ei:
            PI.solve_least_squares(s, rec["y"], float(rec["psi"]))
        assert ei.value.rho == pytest.approx(float(rec["rho"]), rel=1e-9)
        return
    x = PI.solve_least_squares(s, rec["y"], float(rec["psi"]))
    np.testing.assert_array_equal(_bits(x), _bits(rec["x"]))


def test_lsq_default_fixtures_present():
    assert len(LSQ_DEFAULT) == 7


@pytest.mark.gpu
@pytest.mark.parametrize("path", LSQ, ids=os.path.basename)
def test_solve_least_squares_vs_reference(path):
    rec = _npz(path)
    s = L.RectMatrix.from_dense(rec["dense"])
    opts = G.SolveOptions(schedule="parallel", epsilon=1e-10, max_iter=6000)
    if int(rec["diverged"]):
        with pytest.raises(PI.LeastSquaresDivergence) as ei:
            PI.solve_least_squares(s, rec["y"], float(rec["psi"]), opts)
        assert ei.value.rho == pytest.approx(float(rec["rho"]), rel=1e-9)
        assert "rho" in str(ei.value)
        return
    x = PI.solve_least_squares(s, rec["y"], float(rec["psi"]), opts)
    np.testing.assert_array_equal(_bits(x), _bits(rec["x"]))
    assert np.max(np.abs(x - rec["oracle"])) <= 1e-5 * (1.0 + np.max(np.abs(x)))
