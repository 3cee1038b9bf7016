"""Symmetric system storage (mirror of the reference ``linalg.py`` SymSystem).

Reference: /root/reference/pkg/src/gabp/linalg.py:33-103 (SymSystem) and :285-288
(residual_norm_per_eq).

Same constructor, fields and invariants as the reference -- ``SymSystem(diag, offdiag,
rhs)`` with ``offdiag`` a dict of unordered pairs ``(i, j), i < j`` -- plus an array
form (``SymSystem.from_pairs``) for the 10^7..10^9-edge workloads, where a Python dict
is not an option.  Internally the off-diagonals are always three parallel arrays
(``pair_i < pair_j``, ``pair_v != 0``) in the dict's iteration order; that is exactly
what the device graph builder (``gabp_graph_create``) consumes.
"""

from __future__ import annotations

import numpy as np


class MatrixMarketError(ValueError):
    """Malformed Matrix Market input (linalg.py:17-18)."""


class SingularMatrixError(ValueError):
    """Pivot collapsed to working precision (linalg.py:21-22)."""


class ZeroDiagonalError(ValueError):
    """An operation that scales by the diagonal met a zero entry (linalg.py:25-26)."""


class SymSystem:
    """Square symmetric system A x = b with sparse off-diagonal storage."""

    __slots__ = ("diag", "rhs", "pair_i", "pair_j", "pair_v", "_offdiag")

    def __init__(self, diag, offdiag=None, rhs=None, *, _pairs=None, _validate=True):
        diag = np.array(diag, dtype=np.float64, copy=True)
        rhs = np.array(rhs, dtype=np.float64, copy=True)
        if diag.ndim != 1 or diag.size < 1:
            raise ValueError("diag must be a non-empty vector")
        if rhs.shape != diag.shape:
            raise ValueError("rhs length must equal matrix dimension")
        n = diag.size
        if _pairs is not None:
            pi, pj, pv = _pairs
            self._offdiag = None
        else:
            offdiag = {} if offdiag is None else offdiag
            m = len(offdiag)
            pi = np.empty(m, dtype=np.int64)
            pj = np.empty(m, dtype=np.int64)
            pv = np.empty(m, dtype=np.float64)
            for k, ((i, j), v) in enumerate(offdiag.items()):
                if not (0 <= i < j < n):
                    raise ValueError(f"bad off-diagonal key ({i}, {j}) for n={n}")
                if v == 0.0:
                    raise ValueError(f"explicit zero stored at ({i}, {j})")
                pi[k], pj[k], pv[k] = i, j, v
            self._offdiag = dict(offdiag)
            _validate = False
        pi = np.ascontiguousarray(pi, dtype=np.int64)
        pj = np.ascontiguousarray(pj, dtype=np.int64)
        pv = np.ascontiguousarray(pv, dtype=np.float64)
        if _validate and pi.size:
            bad = ~((pi >= 0) & (pi < pj) & (pj < n))
            if bad.any():
                k = int(np.flatnonzero(bad)[0])
                raise ValueError(f"bad off-diagonal key ({pi[k]}, {pj[k]}) for n={n}")
            zero = pv == 0.0
            if zero.any():
                k = int(np.flatnonzero(zero)[0])
                raise ValueError(f"explicit zero stored at ({pi[k]}, {pj[k]})")
        for a in (diag, rhs, pi, pj, pv):
            a.setflags(write=False)
        self.diag, self.rhs = diag, rhs
        self.pair_i, self.pair_j, self.pair_v = pi, pj, pv

    # -- constructors -----------------------------------------------------------------
    @classmethod
    def from_pairs(cls, diag, pair_i, pair_j, pair_v, rhs, validate=True) -> "SymSystem":
        """Array form: upper-triangle pairs (i < j), nonzero values, no duplicates.
        Duplicates are detected by the device graph builder (GABP_EDUP)."""
        return cls(diag, None, rhs, _pairs=(pair_i, pair_j, pair_v), _validate=validate)

    @classmethod
    def from_dense(cls, a, b) -> "SymSystem":
        """linalg.py:68-83: asymmetry rejected, exact zeros are not stored."""
        a = np.asarray(a, dtype=float)
        b = np.asarray(b, dtype=float)
        if a.ndim != 2 or a.shape[0] != a.shape[1]:
            raise ValueError("matrix must be square")
        n = a.shape[0]
        iu, ju = np.triu_indices(n, 1)
        up, lo = a[iu, ju], a[ju, iu]
        asym = up != lo
        if asym.any():
            k = int(np.flatnonzero(asym)[0])
            raise ValueError(f"matrix not symmetric at ({iu[k]}, {ju[k]})")
        nz = up != 0.0
        return cls.from_pairs(a.diagonal().copy(), iu[nz], ju[nz], up[nz], b, validate=False)

    # -- reference surface ----------------------------------------------------------------
    @property
    def n(self) -> int:
        return self.diag.size

    @property
    def nnz_offdiag(self) -> int:
        return int(self.pair_v.size)

    @property
    def offdiag(self) -> dict:
        """The reference's unordered-pair map (built lazily; small systems only)."""
        if self._offdiag is None:
            if self.pair_v.size > 5_000_000:
                raise MemoryError("offdiag dict of a >5M-pair system; use pair_i/pair_j/pair_v")
            self._offdiag = {(int(i), int(j)): float(v)
                             for i, j, v in zip(self.pair_i, self.pair_j, self.pair_v)}
        return self._offdiag

    def to_dense(self) -> tuple[np.ndarray, np.ndarray]:
        a = np.diag(self.diag)
        a[self.pair_i, self.pair_j] = self.pair_v
        a[self.pair_j, self.pair_i] = self.pair_v
        return a, self.rhs.copy()

    def with_rhs(self, b) -> "SymSystem":
        return SymSystem.from_pairs(self.diag, self.pair_i, self.pair_j, self.pair_v, b,
                                    validate=False)

    def matvec(self, x) -> np.ndarray:
        """y = A x (linalg.py:95-103), host-side utility."""
        x = np.asarray(x, dtype=float)
        if x.shape != (self.n,):
            raise ValueError(f"vector length {x.size} != dimension {self.n}")
        y = self.diag * x
        y += np.bincount(self.pair_i, weights=self.pair_v * x[self.pair_j], minlength=self.n)
        y += np.bincount(self.pair_j, weights=self.pair_v * x[self.pair_i], minlength=self.n)
        return y

    def __repr__(self) -> str:
        return f"SymSystem(n={self.n}, offdiag_nnz={self.nnz_offdiag})"


def residual_norm_per_eq(system: SymSystem, x) -> float:
    """||A x - b||_2 / n (linalg.py:285-288), host-side utility.  The solve loop
    computes the same quantity on the device every sweep."""
    r = system.matvec(x) - system.rhs
    return float(np.sqrt(np.sum(r * r)) / system.n)


def dominance_class(system: SymSystem) -> str:
    """linalg.py:332-343: 'strict', 'weak' or 'none'."""
    off = np.bincount(system.pair_i, weights=np.abs(system.pair_v), minlength=system.n) + \
        np.bincount(system.pair_j, weights=np.abs(system.pair_v), minlength=system.n)
    ad = np.abs(system.diag)
    if np.all(ad > off):
        return "strict"
    if np.all(ad >= off):
        return "weak"
    return "none"
