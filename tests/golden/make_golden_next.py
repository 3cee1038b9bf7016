"""Generate the fixtures of the Matrix Market / vector I/O row by running the REFERENCE
package itself.

Run in the build container (the reference is importable only there):

    python tests/golden/make_golden_next.py

Outputs tests/golden/next/mm_cases.json.  The GPU box never
reads /root/reference; tests/test_next_rows.py reads only these files.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "next")
sys.path.insert(0, "/root/reference/pkg/src")

import gabp  # noqa: E402  (the reference)


def mm_fixtures():
    rng = np.random.default_rng(11)
    texts = []
    # coordinate general / symmetric with comments, blank lines, zeros, unordered entries
    texts.append("%%MatrixMarket matrix coordinate real general\n% a comment\n\n3 4 5\n"
                 "1 1 1.5\n3 4 -2e-3\n2 2 0\n1 4 7\n3 1 0.1\n")
    texts.append("%%MatrixMarket matrix coordinate real symmetric\n4 4 6\n1 1 4\n2 1 -1\n"
                 "3 2 -1.25\n4 4 4\n4 3 1e300\n3 3 4.0000000000000001\n")
    texts.append("%%MatrixMarket Matrix Coordinate Real Symmetric\n2 2 2\n  1 1 2  \n2 1 -0.5\n")
    texts.append("%%MatrixMarket matrix array real general\n2 3\n1\n0\n-2.5\n4\n0.5\n6\n")
    texts.append("%%MatrixMarket matrix array real symmetric\n3 3\n2\n-1\n0\n2\n-1\n2\n")
    # a random symmetric coordinate file, shuffled
    n = 40
    dense = np.zeros((n, n))
    iu = np.triu_indices(n, 1)
    mask = rng.random(iu[0].size) < 0.1
    vals = rng.standard_normal(mask.sum())
    dense[iu[0][mask], iu[1][mask]] = vals
    dense = dense + dense.T + np.diag(rng.uniform(1, 2, n))
    lo = [(i, j, dense[i, j]) for i in range(n) for j in range(i + 1) if dense[i, j] != 0.0]
    order = rng.permutation(len(lo))
    body = "".join(f"{lo[k][0] + 1} {lo[k][1] + 1} {float(lo[k][2])!r}\n" for k in order)
    texts.append(f"%%MatrixMarket matrix coordinate real symmetric\n{n} {n} {len(lo)}\n" + body)
    errors = [
        "", "%%MatrixMarket matrix coordinate real\n1 1 1\n1 1 1\n",
        "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1\n",
        "%%MatrixMarket matrix dense real general\n1 1\n1\n",
        "%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1\n",
        "%%MatrixMarket matrix coordinate real general\n% only a comment\n",
        "%%MatrixMarket matrix coordinate real general\n2 2\n1 1 1\n",
        "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n",
        "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n2 2\n",
        "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n3 1 1\n",
        "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n2 1 5\n1 1 2\n",
        "%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n2 1 1\n1 2 3\n",
        "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n1 1 2\n3 3 1\n",
        "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n3 3 1\n1 1 2\n",
        "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n",
        "%%MatrixMarket matrix array real symmetric\n2 3\n1\n2\n3\n",
        "%%MatrixMarket matrix array real general\n2\n1\n",
    ]
    sys_errors = [
        "%%MatrixMarket matrix coordinate real general\n2 3 1\n1 1 1\n",
        "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n1 2 2\n2 1 3\n",
        "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n1 2 2\n",
    ]
    cases = []
    for t in texts:
        r = gabp.parse_matrix_market(t)
        ent = [[i, j, repr(v)] for (i, j), v in r.entries.items()]
        case = {"text": t, "m": r.m, "n": r.n, "entries": ent,
                "write": gabp.write_matrix_market(r)}
        if r.m == r.n:
            try:
                s = gabp.system_from_matrix_market(t, np.arange(r.m, dtype=float))
                case["system"] = {"diag": [repr(v) for v in s.diag],
                                  "pairs": [[i, j, repr(v)] for (i, j), v in s.offdiag.items()],
                                  "write": gabp.write_matrix_market(s)}
            except gabp.MatrixMarketError as exc:
                case["system_error"] = str(exc)
        cases.append(case)
    errs = []
    for t in errors:
        try:
            gabp.parse_matrix_market(t)
            errs.append({"text": t, "error": None})
        except Exception as exc:  # noqa: BLE001
            errs.append({"text": t, "type": type(exc).__name__, "error": str(exc)})
    serrs = []
    for t in sys_errors:
        try:
            gabp.system_from_matrix_market(t, np.zeros(2))
            serrs.append({"text": t, "error": None})
        except Exception as exc:  # noqa: BLE001
            serrs.append({"text": t, "type": type(exc).__name__, "error": str(exc)})
    vec = [float(v) for v in rng.standard_normal(7)]
    vtext = gabp.write_vector(vec)
    out = {"cases": cases, "errors": errs, "system_errors": serrs,
           "vector": {"values": [repr(v) for v in vec], "text": vtext,
                      "parsed": [repr(v) for v in gabp.parse_vector("\n" + vtext + "\n\n")]}}
    with open(os.path.join(OUT, "mm_cases.json"), "w") as fh:
        json.dump(out, fh, indent=0)


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    mm_fixtures()
    print("wrote", sorted(os.listdir(OUT)))
