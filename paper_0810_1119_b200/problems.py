"""Benchmark systems: the reference's desk-scale instances and the five north-star configs.

The small named instances restate ``problems.py`` of the reference
(/root/reference/pkg/src/gabp/problems.py:33-149); the large generators produce the
seeded synthetic workloads of BASELINE.json ``configs`` directly in array (pair-list)
form, because a dict with 10^8 keys -- the reference's ``SymSystem.offdiag`` storage --
does not fit a Python process.

All generators are deterministic in their seed.  Off-diagonal values that come out as
exactly 0.0 are dropped, matching the reference invariant that stored off-diagonals are
exactly the nonzeros (linalg.py:46-60).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .linalg import SymSystem


@dataclass(frozen=True)
class ProblemInstance:
    """problems.py:23-30."""

    id: str
    system: SymSystem
    reference_solution: np.ndarray | None = None
    reference_iterations: dict = field(default_factory=dict)
    classical_diverges: bool = False


# ---------------------------------------------------------------------------
# reference desk-scale instances (problems.py:33-149)
# ---------------------------------------------------------------------------

def gen_toy3() -> ProblemInstance:
    system = SymSystem(diag=np.array([1.0, 1.0, 1.0]),
                       offdiag={(0, 1): -2.0, (0, 2): 3.0},
                       rhs=np.array([-6.0, 0.0, 2.0]))
    return ProblemInstance("toy3", system, reference_solution=np.array([1.0, 2.0, -1.0]))


def gen_cdma(n: int) -> ProblemInstance:
    if n == 3:
        r = np.array([[7, -1, 3], [-1, 7, -5], [3, -5, 7]], dtype=float) / 7.0
    elif n == 4:
        r = np.array([[7, -1, 3, 3], [-1, 7, 3, -1], [3, 3, 7, -1], [3, -1, -1, 7]],
                     dtype=float) / 7.0
    else:
        raise ValueError("only the 3- and 4-user correlation matrices are defined")
    return ProblemInstance(f"cdma{n}", SymSystem.from_dense(r, np.ones(n)))


def gen_nonpsd3() -> ProblemInstance:
    a = np.array([[1, 2, 3], [2, 2, 1], [3, 1, 1]], dtype=float)
    return ProblemInstance("nonpsd3", SymSystem.from_dense(a, np.ones(3)),
                           classical_diverges=True)


def gen_poisson(p: int, f: float = -1.0) -> ProblemInstance:
    """5-point Dirichlet Laplacian, b = -f h^2 (problems.py:100-134)."""
    if p < 1:
        raise ValueError("p must be >= 1")
    h = 1.0 / (p + 1)
    n = p * p
    pi, pj = _grid2d_pairs(p)
    system = SymSystem.from_pairs(np.full(n, 4.0), pi, pj, np.full(pi.size, -1.0),
                                  np.full(n, -f * h * h))
    return ProblemInstance(f"poisson:{p}", system)


def load_instance(name: str) -> ProblemInstance:
    """problems.py:137-149."""
    if name == "toy3":
        return gen_toy3()
    if name == "cdma3":
        return gen_cdma(3)
    if name == "cdma4":
        return gen_cdma(4)
    if name == "nonpsd3":
        return gen_nonpsd3()
    if name.startswith("poisson:"):
        return gen_poisson(int(name.split(":", 1)[1]))
    raise ValueError(f"unknown problem {name!r}")


# ---------------------------------------------------------------------------
# north-star configs (BASELINE.json "configs")
# ---------------------------------------------------------------------------

def _grid2d_pairs(p: int):
    idx = np.arange(p * p, dtype=np.int64).reshape(p, p)  # [row y][col x], natural order
    right_i = idx[:, :-1].ravel()
    up_i = idx[:-1, :].ravel()
    pi = np.concatenate([right_i, up_i])
    pj = np.concatenate([right_i + 1, up_i + p])
    return pi, pj


def _grid3d_pairs(p: int):
    idx = np.arange(p ** 3, dtype=np.int64).reshape(p, p, p)  # [z][y][x]
    a = idx[:, :, :-1].ravel()
    b = idx[:, :-1, :].ravel()
    c = idx[:-1, :, :].ravel()
    pi = np.concatenate([a, b, c])
    pj = np.concatenate([a + 1, b + p, c + p * p])
    return pi, pj


def gen_poisson2d(p: int, seed: int = 0) -> ProblemInstance:
    """Configs 0 and 2: 5-point Laplacian (diag 4, neighbours -1), b ~ N(0,1)."""
    rng = np.random.default_rng(seed)
    n = p * p
    pi, pj = _grid2d_pairs(p)
    rhs = rng.standard_normal(n)
    system = SymSystem.from_pairs(np.full(n, 4.0), pi, pj, np.full(pi.size, -1.0), rhs)
    return ProblemInstance(f"poisson2d:{p}:{seed}", system)


def gen_poisson3d(p: int, seed: int = 0) -> ProblemInstance:
    """Config 4: 7-point Laplacian (diag 6, neighbours -1) on p^3, b ~ N(0,1)."""
    rng = np.random.default_rng(seed)
    n = p ** 3
    pi, pj = _grid3d_pairs(p)
    rhs = rng.standard_normal(n)
    system = SymSystem.from_pairs(np.full(n, 6.0), pi, pj, np.full(pi.size, -1.0), rhs)
    return ProblemInstance(f"poisson3d:{p}:{seed}", system)


def gen_random_sparse(n: int, k: int = 16, seed: int = 0, dominance: float = 1.1
                      ) -> ProblemInstance:
    """Config 1: each row draws k uniformly random columns != i, pairs are symmetrised
    (first draw wins on a collision), off-diagonals U(-1,1), A_ii = dominance * sum|A_ij|,
    b ~ N(0,1)."""
    if n < 2:
        raise ValueError("n must be >= 2")
    rng = np.random.default_rng(seed)
    rows = np.repeat(np.arange(n, dtype=np.int64), k)
    cols = rng.integers(0, n - 1, size=n * k, dtype=np.int64)
    cols += cols >= rows  # uniform over columns != row
    vals = rng.uniform(-1.0, 1.0, size=n * k)
    lo = np.minimum(rows, cols)
    hi = np.maximum(rows, cols)
    key = lo * n + hi
    _, first = np.unique(key, return_index=True)
    first.sort()
    pi, pj, pv = lo[first], hi[first], vals[first]
    nz = pv != 0.0
    pi, pj, pv = pi[nz], pj[nz], pv[nz]
    absum = np.bincount(pi, weights=np.abs(pv), minlength=n) + \
        np.bincount(pj, weights=np.abs(pv), minlength=n)
    diag = dominance * absum
    diag[diag == 0.0] = 1.0  # isolated node keeps a usable prior
    rhs = rng.standard_normal(n)
    return ProblemInstance(f"random:{n}:{k}:{seed}", SymSystem.from_pairs(diag, pi, pj, pv, rhs))


def gen_cdma_detection(N: int = 8192, K: int = 4096, sigma2: float = 0.5, seed: int = 0):
    """Config 3: S in R^{N x K} with i.i.d. +-1/sqrt(N) entries, A = S^T S + sigma2 I,
    b = S^T (S s + w), s i.i.d. +-1, w ~ N(0, sigma2).

    Returns (ProblemInstance, s).  S^T S is formed exactly as (integer Gram) / N, so the
    zero pattern of A is exact; the dense (K x K) matrix is also available through
    ``system.to_dense()``."""
    rng = np.random.default_rng(seed)
    sb = np.where(rng.random((N, K)) < 0.5, -1.0, 1.0)  # +-1, exact
    s = np.where(rng.random(K) < 0.5, -1.0, 1.0)
    w = rng.standard_normal(N) * np.sqrt(sigma2)
    gram = sb.T @ sb  # integers, exact in fp64 (|G| <= N < 2^53)
    a = gram / N
    a[np.diag_indices(K)] += sigma2
    y = (sb @ s) / np.sqrt(N) + w
    b = (sb.T @ y) / np.sqrt(N)
    iu, ju = np.triu_indices(K, 1)
    v = a[iu, ju]
    nz = v != 0.0
    system = SymSystem.from_pairs(np.ascontiguousarray(np.diag(a)), iu[nz], ju[nz], v[nz], b)
    return ProblemInstance(f"cdma:{N}:{K}:{seed}", system), s


def gen_random(kind: str, n: int, seed: int) -> ProblemInstance:
    """problems.py:159-206 restated: 'tree', 'strict_dominant' or 'spd' instances drawn
    from the same numpy Generator call sequence as the reference."""
    if n < 1:
        raise ValueError("n must be >= 1")
    rng = np.random.default_rng(seed)
    if kind == "tree":
        off: dict = {}
        for child in range(1, n):
            parent = int(rng.integers(0, child))
            w = float(rng.uniform(0.2, 1.5)) * (1.0 if rng.random() < 0.5 else -1.0)
            off[(parent, child)] = w
        rowsum = np.zeros(n)
        for (i, j), v in off.items():
            rowsum[i] += abs(v)
            rowsum[j] += abs(v)
        signs = np.where(rng.random(n) < 0.5, 1.0, -1.0)
        diag = signs * (rowsum + rng.uniform(0.5, 1.5, size=n))
        system = SymSystem(diag=diag, offdiag=off, rhs=rng.standard_normal(n))
    elif kind == "strict_dominant":
        off = {}
        for i in range(n):
            for j in range(i + 1, n):
                if rng.random() < 0.5:
                    w = float(rng.uniform(-1.0, 1.0))
                    if w != 0.0:
                        off[(i, j)] = w
        rowsum = np.zeros(n)
        for (i, j), v in off.items():
            rowsum[i] += abs(v)
            rowsum[j] += abs(v)
        system = SymSystem(diag=rowsum + 1.0, offdiag=off, rhs=rng.standard_normal(n))
    elif kind == "spd":
        m = rng.standard_normal((n, n))
        a = m.T @ m + np.eye(n)
        a = (a + a.T) / 2.0
        system = SymSystem.from_dense(a, rng.standard_normal(n))
    else:
        raise ValueError(f"unknown kind {kind!r}")
    return ProblemInstance(f"{kind}-{n}-{seed}", system)


def decorrelator_detect(system: SymSystem, y, solve_fn) -> np.ndarray:
    """problems.py:152-156: sign(R^-1 y) with sign(0) -> +1."""
    solution = np.asarray(solve_fn(system.with_rhs(y)), dtype=float)
    return np.where(solution >= 0.0, 1.0, -1.0)


CONFIGS = {
    0: ("poisson2d-32", lambda seed=0: gen_poisson2d(32, seed)),
    1: ("random-1M-k16", lambda seed=0: gen_random_sparse(1 << 20, 16, seed)),
    2: ("poisson2d-4096", lambda seed=0: gen_poisson2d(4096, seed)),
    3: ("cdma-8192x4096", lambda seed=0: gen_cdma_detection(8192, 4096, 0.5, seed)[0]),
    4: ("poisson3d-512", lambda seed=0: gen_poisson3d(512, seed)),
}
