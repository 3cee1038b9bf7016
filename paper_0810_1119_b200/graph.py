"""Device-resident Gaussian graphical model (mirror of the reference ``graph.py``).

Reference: /root/reference/pkg/src/gabp/graph.py:53-163.  ``build_graph(system)`` hands
the SymSystem pair arrays to ``gabp_graph_create`` (include/gabp_b200.h), which builds
the CSR, the twin-edge index and the sweep tiles on the GPU.  The per-edge arrays the
reference exposes (``src``, ``dst``, ``rev``, ``coeff``, ``neighbors``, ``edge_index``)
are available as host copies on demand, numbered exactly like the reference's edge ids.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .linalg import SymSystem, ZeroDiagonalError


class DegenerateProductError(ValueError):
    """Gaussian product with exactly cancelling precisions (graph.py:19-20)."""


@dataclass(frozen=True)
class ScalarGaussian:
    """graph.py:23-36."""

    mean: float
    prec: float

    def __post_init__(self):
        if not (np.isfinite(self.mean) and np.isfinite(self.prec)):
            raise ValueError("mean and precision must be finite")


def gaussian_product(a: ScalarGaussian, b: ScalarGaussian) -> ScalarGaussian:
    """graph.py:39-50 (scalar lemma used by the message derivation)."""
    prec = a.prec + b.prec
    if prec == 0.0:
        raise DegenerateProductError("precisions cancel exactly")
    return ScalarGaussian(mean=(a.prec * a.mean + b.prec * b.mean) / prec, prec=prec)


DENSE_MIN_FILL = 0.5       # off-diagonal fill above which the dense kernels are used
DENSE_MIN_N = 256          # ... for systems from this size
DENSE_MAX_N = 1 << 14      # ... up to this size (3 x n^2 x 16 B of messages)


class GaussianGraph:
    """Handle to a graph built on the GPU (graph.py:53-120).

    Systems whose off-diagonal fill exceeds DENSE_MIN_FILL (linear detection, BASELINE
    config 3) also get the dense representation: the broadcast solve then runs the dense
    column-walk / edge-tile kernels (csrc/dense.cu), bitwise identical to the sparse path."""

    def __init__(self, system: SymSystem, device: int | None = None, dense: bool | None = None):
        lib = _lib.load()
        zero = np.flatnonzero(system.diag == 0.0)
        if zero.size:
            raise ZeroDiagonalError(
                f"zero diagonal entry at row {int(zero[0])}: node priors need b_i / A_ii")
        self.system = system
        self.n = system.n
        self.device = _lib.default_device() if device is None else int(device)
        if dense is None:
            fill = 2.0 * system.pair_v.size / max(system.n * (system.n - 1), 1)
            dense = DENSE_MIN_N <= system.n <= DENSE_MAX_N and fill > DENSE_MIN_FILL
        h = ctypes.c_void_p()
        if dense:
            a, _ = system.to_dense()
            a = np.ascontiguousarray(a)
            rc = lib.gabp_graph_create_dense(system.n, _lib.ptr(a), _lib.ptr(system.rhs),
                                             self.device, ctypes.byref(h))
        else:
            rc = lib.gabp_graph_create(system.n, system.pair_v.size, _lib.ptr(system.diag),
                                       _lib.ptr(system.rhs), _lib.ptr(system.pair_i),
                                       _lib.ptr(system.pair_j), _lib.ptr(system.pair_v),
                                       self.device, ctypes.byref(h))
        if rc == _lib.GABP_EZERODIAG:
            raise ZeroDiagonalError(_lib.last_error())
        if rc in (_lib.GABP_EINVAL, _lib.GABP_EDUP):
            raise ValueError(_lib.last_error())
        _lib.check(rc)
        self._h = h
        info = _lib.GraphInfo()
        _lib.check(lib.gabp_graph_info(h, ctypes.byref(info)))
        self.info = info
        self._export = None
        self.prior_prec = system.diag
        with np.errstate(divide="ignore", invalid="ignore"):
            self.prior_mean = system.rhs / system.diag

    @property
    def handle(self):
        return self._h

    @property
    def num_edges(self) -> int:
        return int(self.info.num_edges)

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.load().gabp_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- host copies of the reference's per-edge arrays -------------------------------
    def _arrays(self):
        if self._export is None:
            E = self.num_edges
            rp = np.empty(self.n + 1, dtype=np.int64)
            col = np.empty(E, dtype=np.int64)
            rev = np.empty(E, dtype=np.int64)
            coeff = np.empty(E, dtype=np.float64)
            _lib.check(_lib.load().gabp_graph_export(self._h, _lib.ptr(rp), _lib.ptr(col),
                                                      _lib.ptr(rev), _lib.ptr(coeff)))
            self._export = (rp, col, rev, coeff)
        return self._export

    @property
    def row_ptr(self) -> np.ndarray:
        return self._arrays()[0]

    @property
    def dst(self) -> np.ndarray:
        return self._arrays()[1]

    @property
    def rev(self) -> np.ndarray:
        return self._arrays()[2]

    @property
    def coeff(self) -> np.ndarray:
        return self._arrays()[3]

    @property
    def src(self) -> np.ndarray:
        return np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.row_ptr))

    @property
    def neighbors(self) -> list:
        rp, col = self.row_ptr, self.dst
        return [col[rp[i]:rp[i + 1]].tolist() for i in range(self.n)]

    @property
    def edge_index(self) -> dict:
        return {(int(i), int(j)): e for e, (i, j) in enumerate(zip(self.src, self.dst))}

    def is_tree(self) -> bool:
        """Connected and acyclic (graph.py:126-139)."""
        if self.system.nnz_offdiag != self.n - 1:
            return False
        if self.n == 1:
            return True
        rp, col = self.row_ptr, self.dst
        seen = np.zeros(self.n, dtype=bool)
        seen[0] = True
        frontier = np.array([0], dtype=np.int64)
        while frontier.size:
            nb = np.concatenate([col[rp[i]:rp[i + 1]] for i in frontier])
            nb = np.unique(nb[~seen[nb]])
            seen[nb] = True
            frontier = nb
        return bool(seen.all())


def build_graph(system: SymSystem, device: int | None = None,
                dense: bool | None = None) -> GaussianGraph:
    """graph.py:161-163: build the graphical model on the GPU."""
    return GaussianGraph(system, device, dense)
