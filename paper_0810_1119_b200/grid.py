"""Poisson grid systems generated on the device, whole or as one rank's slab.

The large north-star configs (BASELINE.json configs 2 and 4: the 5-point Laplacian on a
4096^2 grid, the 7-point Laplacian on a 512^3 grid) have 33.5 M and 402 M off-diagonal
pairs.  Building them on the host (problems.gen_poisson2d/3d + SymSystem) costs seconds
to minutes of numpy and 10 GB of host memory per rank; here the pair arrays of a node
window are formed on the GPU with torch and handed to the library in HBM
(``gabp_graph_create_device_ex``), so a rank of a slab partition materialises only its
own rows and their halo -- never the global system.

Grid numbering is the reference's natural order (x fastest; problems.py:100-134 for the
2-D case): node (z, y, x) = z p^2 + y p + x, neighbours at +-1, +-p (and +-p^2), A_ii = 4
(2-D) or 6 (3-D), off-diagonals -1.  b ~ N(0, 1) is drawn on the device from a seeded
torch generator (Philox: the same values for a seed on every device and at every world
size), so the system is identical whichever number of ranks builds it.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib


@dataclass(frozen=True)
class GridSpec:
    dims: int          # 2 or 3
    p: int             # points per side
    seed: int = 0

    def __post_init__(self):
        if self.dims not in (2, 3) or self.p < 2:
            raise ValueError("a 2-D or 3-D grid of at least 2 points per side")

    @property
    def n(self) -> int:
        return self.p ** self.dims

    @property
    def plane(self) -> int:
        """Largest neighbour offset: a grid row (2-D) or plane (3-D) -- the slab halo."""
        return self.p ** (self.dims - 1)

    @property
    def diag_value(self) -> float:
        return 2.0 * self.dims

    @property
    def npairs(self) -> int:
        return self.dims * (self.p - 1) * self.p ** (self.dims - 1)

    @property
    def name(self) -> str:
        return f"poisson{self.dims}d-{self.p}"


def _dev(device: int) -> str:
    """torch device string; device < 0 selects the CPU (host-side tests of the layout)."""
    return "cpu" if device is not None and device < 0 else f"cuda:{device}"


def rhs_device(spec: GridSpec, device: int):
    import torch
    g = torch.Generator(device=_dev(device))
    g.manual_seed(int(spec.seed))
    return torch.randn(spec.n, generator=g, dtype=torch.float64, device=_dev(device))


def _pairs(spec: GridSpec, a: int, b: int, lo: int, hi: int, device: int):
    """Global pairs (i < j) of the window [a, b) with an endpoint in [lo, hi)."""
    import torch
    dev = _dev(device)
    p = spec.p
    i = torch.arange(a, b, dtype=torch.int64, device=dev)
    outs_i, outs_j = [], []
    offs = [1, p] + ([p * p] if spec.dims == 3 else [])
    for k, off in enumerate(offs):
        # neighbour along axis k exists when that coordinate is below p - 1
        coord = (i // (p ** k)) % p
        j = i + off
        m = (coord < p - 1) & (j < b) & (((i >= lo) & (i < hi)) | ((j >= lo) & (j < hi)))
        outs_i.append(i[m])
        outs_j.append(j[m])
        del coord, j, m
    return torch.cat(outs_i), torch.cat(outs_j)


@dataclass
class GridPart:
    """One rank's slab: owned global rows [lo, hi) (whole grid rows / planes when the
    bounds fall on them; any bounds with hi - lo >= the plane size work), halo = the plane
    below and above, local id = global id - a for the window [a, b)."""
    spec: GridSpec
    rank: int
    world: int
    lo: int
    hi: int
    a: int
    b: int
    diag: object = None     # torch tensors on the device (local ids)
    rhs: object = None
    pair_i: object = None
    pair_j: object = None
    pair_v: object = None
    peers: list = field(default_factory=list)
    send_idx: dict = field(default_factory=dict)
    recv_idx: dict = field(default_factory=dict)

    @property
    def n_global(self) -> int:
        return self.spec.n

    @property
    def n_local(self) -> int:
        return self.b - self.a

    @property
    def row_lo(self) -> int:
        return self.lo - self.a

    @property
    def row_hi(self) -> int:
        return self.hi - self.a

    @property
    def npairs(self) -> int:
        return int(self.pair_v.numel())

    def halo_bytes_per_sweep(self) -> int:
        return 24 * int(sum(v.size for v in self.send_idx.values()) +
                        sum(v.size for v in self.recv_idx.values()))


def slab_bounds(spec: GridSpec, world: int) -> np.ndarray:
    """Row blocks of whole grid rows / planes, as equal as the plane count allows."""
    planes = spec.p
    if world < 1 or world > planes:
        raise ValueError(f"need 1 <= world <= {planes}")
    return np.array([(planes * r) // world * spec.plane for r in range(world + 1)],
                    dtype=np.int64)


def grid_part(spec: GridSpec, world: int, rank: int, device: int, rhs=None) -> GridPart:
    """Rank `rank`'s slab of the grid on `device` (world 1: the whole graph)."""
    import torch
    bounds = slab_bounds(spec, world)
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    h = spec.plane
    a = max(0, lo - h) if rank > 0 else lo
    b = min(spec.n, hi + h) if rank < world - 1 else hi
    if rhs is None:
        rhs = rhs_device(spec, device)
    dev = _dev(device)
    gi, gj = _pairs(spec, a, b, lo, hi, device)
    part = GridPart(spec, rank, world, lo, hi, a, b)
    part.pair_i = gi - a
    part.pair_j = gj - a
    part.pair_v = torch.full((gi.numel(),), -1.0, dtype=torch.float64, device=dev)
    diag = torch.ones(b - a, dtype=torch.float64, device=dev)  # halo rows: unused prior
    diag[lo - a:hi - a] = spec.diag_value
    r = torch.zeros(b - a, dtype=torch.float64, device=dev)
    r[lo - a:hi - a] = rhs[lo:hi]
    part.diag, part.rhs = diag, r
    if rank > 0:
        part.recv_idx[rank - 1] = np.arange(0, lo - a, dtype=np.int64)
        part.send_idx[rank - 1] = np.arange(lo - a, lo - a + h, dtype=np.int64)
    if rank < world - 1:
        part.recv_idx[rank + 1] = np.arange(hi - a, b - a, dtype=np.int64)
        part.send_idx[rank + 1] = np.arange(hi - a - h, hi - a, dtype=np.int64)
    part.peers = sorted(set(part.recv_idx) | set(part.send_idx))
    return part


def part_graph(part: GridPart, device: int):
    """Build the part's graph in the library from its device arrays; returns the handle."""
    import torch
    torch.cuda.synchronize(device)  # the arrays were made on torch's stream
    h = ctypes.c_void_p()
    _lib.check(_lib.load().gabp_graph_create_device_ex(
        part.n_local, part.npairs, part.diag.data_ptr(), part.rhs.data_ptr(),
        part.pair_i.data_ptr(), part.pair_j.data_ptr(), part.pair_v.data_ptr(),
        part.row_lo, part.row_hi, device, ctypes.byref(h)))
    return h


class GridGraph:
    """The whole grid built on one device (duck-types GaussianGraph for solve_graph)."""

    def __init__(self, spec: GridSpec, device: int = 0, keep_arrays: bool = False):
        self.spec = spec
        self.n = spec.n
        self.device = device
        part = grid_part(spec, 1, 0, device)
        self._h = part_graph(part, device)
        self.part = part if keep_arrays else None
        info = _lib.GraphInfo()
        _lib.check(_lib.load().gabp_graph_info(self._h, ctypes.byref(info)))
        self.info = info
        del part

    @property
    def handle(self):
        return self._h

    @property
    def num_edges(self) -> int:
        return int(self.info.num_edges)

    def is_tree(self) -> bool:
        return False

    def host_arrays(self):
        """(diag, rhs, pair_i, pair_j, pair_v) on the host (oracle comparisons)."""
        p = self.part or grid_part(self.spec, 1, 0, self.device)
        return tuple(t.cpu().numpy() for t in (p.diag, p.rhs, p.pair_i, p.pair_j, p.pair_v))

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.load().gabp_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
