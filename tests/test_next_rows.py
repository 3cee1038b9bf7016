"""Rows beside the sweep (DESIGN.md row f): Matrix Market / vector I/O -- against fixtures
made by running the reference itself (tests/golden/make_golden_next.py)."""

import json
import os

import numpy as np
import pytest

import paper_0810_1119_b200 as G
from paper_0810_1119_b200 import linalg as L

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
