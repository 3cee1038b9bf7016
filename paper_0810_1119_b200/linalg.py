"""Symmetric system storage and its file formats (mirror of the reference ``linalg.py``).

Reference: /root/reference/pkg/src/gabp/linalg.py:33-103 (SymSystem), :106-141
(RectMatrix), :153-282 (Matrix Market and vector text I/O), :285-288
(residual_norm_per_eq), :291-329 (the rho(|I - D^-1 A|) diagnostic).

Same constructor, fields and invariants as the reference -- ``SymSystem(diag, offdiag,
rhs)`` with ``offdiag`` a dict of unordered pairs ``(i, j), i < j`` -- plus an array
form (``SymSystem.from_pairs``) for the 10^7..10^9-edge workloads, where a Python dict
is not an option.  Internally the off-diagonals are always three parallel arrays
(``pair_i < pair_j``, ``pair_v != 0``) in the dict's iteration order; that is exactly
what the device graph builder (``gabp_graph_create``) consumes.
"""

from __future__ import annotations

import math

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


def spectral_radius_gabp_test(system: SymSystem) -> float:
    """linalg.py:313-329: rho(|I - D^-1 A|) by power iteration on the Perron-shifted
    absolute iteration matrix from the all-ones start (linalg.py:291-310).  A diagnostic
    carried by LeastSquaresDivergence; host-side, dense, small systems."""
    if np.any(system.diag == 0.0):
        row = int(np.flatnonzero(system.diag == 0.0)[0])
        raise ZeroDiagonalError(f"zero diagonal entry at row {row}")
    n = system.n
    m = np.zeros((n, n))
    m[system.pair_i, system.pair_j] = np.abs(system.pair_v / system.diag[system.pair_i])
    m[system.pair_j, system.pair_i] = np.abs(system.pair_v / system.diag[system.pair_j])
    x = np.ones(n) / math.sqrt(n)
    lam = 0.0
    for _ in range(10_000):
        y = m @ x + x
        norm = float(np.linalg.norm(y))
        if norm == 0.0:
            lam = 0.0
            break
        lam = float(x @ y)
        if float(np.linalg.norm(y - lam * x)) <= 1e-6 * max(1.0, abs(lam)):
            break
        x = y / norm
    return max(lam - 1.0, 0.0)


# ---------------------------------------------------------------------------------------
# General sparse matrices and the Matrix Market text format (linalg.py:106-282)
# ---------------------------------------------------------------------------------------

class RectMatrix:
    """m x n sparse matrix (linalg.py:106-141): ``RectMatrix(m, n, entries)`` with a dict of
    (i, j) -> value, or ``RectMatrix.from_arrays`` with parallel index / value arrays (the
    dict is then built on first use)."""

    __slots__ = ("m", "n", "rows", "cols", "vals", "_entries")

    def __init__(self, m: int, n: int, entries=None, *, _arrays=None):
        if m < 1 or n < 1:
            raise ValueError("matrix dimensions must be >= 1")
        self.m, self.n = int(m), int(n)
        if _arrays is not None:
            r, c, v = (np.ascontiguousarray(a) for a in _arrays)
            self._entries = None
        else:
            entries = {} if entries is None else dict(entries)
            r = np.fromiter((k[0] for k in entries), dtype=np.int64, count=len(entries))
            c = np.fromiter((k[1] for k in entries), dtype=np.int64, count=len(entries))
            v = np.fromiter(entries.values(), dtype=np.float64, count=len(entries))
            self._entries = entries
        bad = ~((r >= 0) & (r < self.m) & (c >= 0) & (c < self.n))
        if bad.any():
            k = int(np.flatnonzero(bad)[0])
            raise ValueError(f"entry ({r[k]}, {c[k]}) outside {self.m}x{self.n}")
        self.rows = r.astype(np.int64, copy=False)
        self.cols = c.astype(np.int64, copy=False)
        self.vals = v.astype(np.float64, copy=False)

    @classmethod
    def from_arrays(cls, m, n, rows, cols, vals) -> "RectMatrix":
        return cls(m, n, _arrays=(rows, cols, vals))

    @classmethod
    def from_dense(cls, a) -> "RectMatrix":
        a = np.asarray(a, dtype=float)
        r, c = np.nonzero(a)  # row-major order, the reference's loop order
        return cls.from_arrays(a.shape[0], a.shape[1], r, c, a[r, c])

    @property
    def entries(self) -> dict:
        if self._entries is None:
            self._entries = {(int(i), int(j)): float(v)
                             for i, j, v in zip(self.rows, self.cols, self.vals)}
        return self._entries

    def to_dense(self) -> np.ndarray:
        a = np.zeros((self.m, self.n))
        a[self.rows, self.cols] = self.vals
        return a

    @property
    def nnz(self) -> int:
        return int(self.vals.size)

    def __eq__(self, other) -> bool:
        if not isinstance(other, RectMatrix):
            return NotImplemented
        return self.m == other.m and self.n == other.n and self.entries == other.entries

    def __repr__(self) -> str:
        return f"RectMatrix(m={self.m}, n={self.n}, nnz={self.nnz})"


def _first_duplicate(keys: np.ndarray):
    """Index (into keys, in insertion order) of the first insertion whose key is already
    present, or None -- the event a sequential dict insertion would fail at."""
    if keys.size < 2:
        return None
    order = np.argsort(keys, kind="stable")
    ks = keys[order]
    rep = np.flatnonzero(ks[1:] == ks[:-1]) + 1  # later occurrences, insertion-sorted per key
    if rep.size == 0:
        return None
    return int(order[rep].min())


def parse_matrix_market(text: str) -> RectMatrix:
    """linalg.py:156-227: a real coordinate or array Matrix Market string.  Symmetric
    coordinate files expand to both orientations; file order never matters; a repeated
    position is an error (the first one in file order is reported); zeros are dropped.
    The entry lines are converted with numpy in one pass; files numpy refuses go through
    the per-line loop, which raises the reference's exact errors."""
    lines = text.splitlines()
    if not lines or not lines[0].startswith("%%MatrixMarket"):
        raise MatrixMarketError("missing %%MatrixMarket header")
    header = lines[0].split()
    if len(header) != 5 or header[1].lower() != "matrix":
        raise MatrixMarketError(f"malformed header: {lines[0]!r}")
    layout, dtype, sym = (w.lower() for w in header[2:5])
    if layout not in ("coordinate", "array"):
        raise MatrixMarketError(f"unsupported layout {layout!r}")
    if dtype != "real":
        raise MatrixMarketError(f"unsupported field type {dtype!r}")
    if sym not in ("general", "symmetric"):
        raise MatrixMarketError(f"unsupported symmetry {sym!r}")
    body = [ln for ln in lines[1:] if ln.strip() and not ln.lstrip().startswith("%")]
    if not body:
        raise MatrixMarketError("missing size line")
    size = body[0].split()
    if layout == "coordinate":
        return _parse_coordinate(body, size, sym)
    return _parse_array(body, size, sym)


def _parse_coordinate(body, size, sym) -> RectMatrix:
    if len(size) != 3:
        raise MatrixMarketError(f"bad coordinate size line: {body[0]!r}")
    m, n, nnz = (int(w) for w in size)
    if len(body) - 1 != nnz:
        raise MatrixMarketError(f"expected {nnz} entries, found {len(body) - 1}")
    rows = cols = vals = None
    try:
        tok = np.array([ln.split() for ln in body[1:]], dtype=object)
        if nnz and (tok.ndim != 2 or tok.shape[1] != 3):
            raise ValueError
        if nnz:
            rows = np.array(tok[:, 0], dtype=np.int64) - 1
            cols = np.array(tok[:, 1], dtype=np.int64) - 1
            vals = np.array([float(t) for t in tok[:, 2]], dtype=np.float64)
        else:
            rows = cols = np.zeros(0, np.int64)
            vals = np.zeros(0)
        if np.any((rows < 0) | (rows >= m) | (cols < 0) | (cols >= n)):
            raise ValueError
    except (ValueError, TypeError, OverflowError):
        rows = None
    if rows is None:  # the reference's per-line loop: its exact error for the bad line
        return _parse_coordinate_loop(body, m, n, sym)
    # insertion events in file order: (i, j), then (j, i) for off-diagonal symmetric entries
    if sym == "general":
        ev_r, ev_c = rows, cols
    else:
        mirror = rows != cols
        k = np.arange(rows.size) * 2
        ev_idx = np.concatenate([k, k[mirror] + 1])
        order = np.argsort(ev_idx, kind="stable")
        ev_r = np.concatenate([rows, cols[mirror]])[order]
        ev_c = np.concatenate([cols, rows[mirror]])[order]
    dup = _first_duplicate(ev_r * n + ev_c)
    if dup is not None:
        raise MatrixMarketError(
            f"duplicate entry for position ({ev_r[dup] + 1}, {ev_c[dup] + 1})")
    ev_v = vals if sym == "general" else np.concatenate([vals, vals[rows != cols]])[order]
    keep = ev_v != 0.0
    return RectMatrix.from_arrays(m, n, ev_r[keep], ev_c[keep], ev_v[keep])


def _parse_coordinate_loop(body, m, n, sym) -> RectMatrix:
    entries: dict = {}
    for ln in body[1:]:
        parts = ln.split()
        if len(parts) != 3:
            raise MatrixMarketError(f"bad entry line: {ln!r}")
        i, j, v = int(parts[0]) - 1, int(parts[1]) - 1, float(parts[2])
        if not (0 <= i < m and 0 <= j < n):
            raise MatrixMarketError(f"entry ({i + 1}, {j + 1}) outside {m}x{n}")
        keys = [(i, j)] if (sym == "general" or i == j) else [(i, j), (j, i)]
        for key in keys:
            if key in entries:
                raise MatrixMarketError(
                    f"duplicate entry for position ({key[0] + 1}, {key[1] + 1})")
            entries[key] = v
    return RectMatrix(m, n, {k: v for k, v in entries.items() if v != 0.0})


def _parse_array(body, size, sym) -> RectMatrix:
    if len(size) != 2:
        raise MatrixMarketError(f"bad array size line: {body[0]!r}")
    m, n = (int(w) for w in size)
    if sym == "symmetric" and m != n:
        raise MatrixMarketError("symmetric array file must be square")
    values = np.array([float(ln) for ln in body[1:]], dtype=np.float64)
    expected = m * n if sym == "general" else m * (m + 1) // 2
    if values.size != expected:
        raise MatrixMarketError(f"expected {expected} array values, found {values.size}")
    # column-major; a symmetric file stores the lower triangle (linalg.py:213-226)
    if sym == "general":
        jj, ii = np.divmod(np.arange(m * n), m)
        nz = values != 0.0
        return RectMatrix.from_arrays(m, n, ii[nz], jj[nz], values[nz])
    jj = np.repeat(np.arange(n), n - np.arange(n))
    ii = np.concatenate([np.arange(j, m) for j in range(n)]) if n else np.zeros(0, np.int64)
    nz = values != 0.0
    ii, jj, vv = ii[nz], jj[nz], values[nz]
    off = ii != jj
    # insertion order: (i, j) then (j, i) for every stored off-diagonal value
    k = np.arange(ii.size) * 2
    order = np.argsort(np.concatenate([k, k[off] + 1]), kind="stable")
    r = np.concatenate([ii, jj[off]])[order]
    c = np.concatenate([jj, ii[off]])[order]
    v = np.concatenate([vv, vv[off]])[order]
    return RectMatrix.from_arrays(m, n, r, c, v)


def system_from_matrix_market(text: str, rhs) -> SymSystem:
    """linalg.py:230-250: a square, exactly symmetric Matrix Market matrix as a SymSystem
    (pairs in the order the reference's dict would hold them)."""
    rect = parse_matrix_market(text)
    if rect.m != rect.n:
        raise MatrixMarketError(f"matrix is {rect.m}x{rect.n}, not square")
    n = rect.m
    r, c, v = rect.rows, rect.cols, rect.vals
    diag = np.zeros(n)
    on = r == c
    diag[r[on]] = v[on]
    offm = ~on
    ro, co, vo = r[offm], c[offm], v[offm]
    # mirrored value of every off-diagonal entry (absent -> asymmetric)
    key = ro * n + co
    mkey = co * n + ro
    srt = np.argsort(key)
    pos = np.searchsorted(key[srt], mkey)
    pos_ok = pos < key.size
    found = np.zeros(ro.size, dtype=bool)
    found[pos_ok] = key[srt][pos[pos_ok]] == mkey[pos_ok]
    mv = np.zeros(ro.size)
    mv[found] = vo[srt][pos[found]]
    bad = ~found | (mv != vo)
    if bad.any():
        # the reference walks the entries in dict order: the first offending one
        k = int(np.flatnonzero(bad)[0])
        raise MatrixMarketError(f"asymmetric entries at ({ro[k] + 1}, {co[k] + 1})")
    # dict order of the reference's `off`: first occurrence of each unordered pair
    lo, hi = np.minimum(ro, co), np.maximum(ro, co)
    _, first = np.unique(lo * n + hi, return_index=True)
    first.sort()
    return SymSystem.from_pairs(diag, lo[first], hi[first], vo[first], rhs)


def write_matrix_market(mat) -> str:
    """linalg.py:253-266: coordinate text, lossless for binary64 (repr of every value)."""
    if isinstance(mat, SymSystem):
        d = np.flatnonzero(mat.diag != 0.0)
        ent = list(zip(d.tolist(), d.tolist(), mat.diag[d].tolist()))
        ent += list(zip(mat.pair_j.tolist(), mat.pair_i.tolist(), mat.pair_v.tolist()))
        ent.sort()
        out = ["%%MatrixMarket matrix coordinate real symmetric", f"{mat.n} {mat.n} {len(ent)}"]
    else:
        ent = sorted(zip(mat.rows.tolist(), mat.cols.tolist(), mat.vals.tolist()))
        out = ["%%MatrixMarket matrix coordinate real general", f"{mat.m} {mat.n} {len(ent)}"]
    out += [f"{i + 1} {j + 1} {v!r}" for i, j, v in ent]
    return "\n".join(out) + "\n"


def parse_vector(text: str) -> np.ndarray:
    """linalg.py:269-274: one decimal per line."""
    values = [float(ln) for ln in text.splitlines() if ln.strip()]
    if not values:
        raise MatrixMarketError("empty vector file")
    return np.array(values)


def write_vector(x) -> str:
    """linalg.py:277-278."""
    return "\n".join(f"{float(v)!r}" for v in np.asarray(x, dtype=float)) + "\n"
