"""Row-block partitioning of a SymSystem for multi-GPU synchronous GaBP.

BASELINE.json north_star: "nodes are partitioned in contiguous row blocks.  Cut-edge
messages are exchanged each sweep as a halo".  Design:

* rank r owns rows [lo_r, hi_r) and every directed edge leaving them;
* its local graph also holds the *halo*: remote neighbours of owned rows.  Local node ids
  are the ranks of the involved global ids in ascending order (halo-below, owned,
  halo-above), so every row's neighbours keep the reference's ascending order and the
  per-row sums stay bitwise identical to the single-GPU solve;
* with the broadcast schedule's aggregate-recompute gather (sweep.cu) an owned row needs,
  of a remote neighbour j, only j's node aggregate {P_j, P_j mu~_j} and marginal x_j of the
  previous launch -- never a message -- so the per-sweep halo is node-level: 24 bytes per
  boundary node and peer (for a row-strip Poisson partition, one grid row per side);
* per-sweep statistics (max change, residual partial, divergence flags) are all-reduced
  before the decision, so every rank decides identically.

This module is host-side only (numpy): the partition and the halo index lists.  The CUDA
library consumes them through ``gabp_graph_create_ex`` / ``gabp_dist_attach``.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .linalg import SymSystem


def partition_rows(n: int, world: int) -> np.ndarray:
    """Contiguous, equal-size row blocks: bounds[r] .. bounds[r+1]."""
    if world < 1 or n < world:
        raise ValueError("need 1 <= world <= n")
    return np.array([(n * r) // world for r in range(world + 1)], dtype=np.int64)


@dataclass
class LocalPart:
    rank: int
    world: int
    n_global: int
    lo: int                      # owned global rows [lo, hi)
    hi: int
    glob: np.ndarray             # local id -> global id (ascending)
    row_lo: int                  # owned rows in local ids: [row_lo, row_hi)
    row_hi: int
    diag: np.ndarray             # local node arrays (halo entries: diag 1, rhs 0)
    rhs: np.ndarray
    pair_i: np.ndarray           # local-id pairs (i < j): owned-owned and owned-halo
    pair_j: np.ndarray
    pair_v: np.ndarray
    peers: list = field(default_factory=list)          # peer ranks
    send_idx: dict = field(default_factory=dict)       # peer -> local ids of owned nodes
    recv_idx: dict = field(default_factory=dict)       # peer -> local ids of halo nodes

    @property
    def n_local(self) -> int:
        return int(self.glob.size)


def local_part(system: SymSystem, bounds: np.ndarray, rank: int) -> LocalPart:
    """The local graph of `rank` and its halo exchange lists."""
    world = bounds.size - 1
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    pi, pj, pv = system.pair_i, system.pair_j, system.pair_v
    own_i = (pi >= lo) & (pi < hi)
    own_j = (pj >= lo) & (pj < hi)
    keep = own_i | own_j
    ki, kj, kv = pi[keep], pj[keep], pv[keep]
    glob = np.unique(np.concatenate([np.arange(lo, hi, dtype=np.int64), ki, kj]))
    li = np.searchsorted(glob, ki)
    lj = np.searchsorted(glob, kj)  # glob ascending -> li < lj whenever ki < kj
    row_lo = int(np.searchsorted(glob, lo))
    row_hi = row_lo + (hi - lo)
    diag = np.ones(glob.size)
    rhs = np.zeros(glob.size)
    owned = (glob >= lo) & (glob < hi)
    diag[owned] = system.diag[glob[owned]]
    rhs[owned] = system.rhs[glob[owned]]
    halo = glob[~owned]
    owner = np.searchsorted(bounds, halo, side="right") - 1
    part = LocalPart(rank, world, system.n, lo, hi, glob, row_lo, row_hi, diag, rhs,
                     li, lj, kv)
    # receive: halo nodes grouped by owner, ascending global id
    halo_local = np.flatnonzero(~owned)
    for peer in np.unique(owner):
        part.recv_idx[int(peer)] = halo_local[owner == peer]
    # send: owned nodes that are halo of a peer (i.e. have a neighbour owned by the peer)
    ext_i = own_i & ~own_j    # owned i, remote j
    ext_j = own_j & ~own_i    # remote i, owned j
    rem = np.concatenate([pj[ext_i], pi[ext_j]])
    mine = np.concatenate([pi[ext_i], pj[ext_j]])
    rem_owner = np.searchsorted(bounds, rem, side="right") - 1
    for peer in np.unique(rem_owner):
        nodes = np.unique(mine[rem_owner == peer])
        part.send_idx[int(peer)] = np.searchsorted(glob, nodes)
    part.peers = sorted(set(part.recv_idx) | set(part.send_idx))
    return part


def halo_bytes_per_sweep(part: LocalPart) -> int:
    """{P, P mu~} (16 B) + x (8 B) per exchanged node and direction."""
    return 24 * int(sum(v.size for v in part.send_idx.values()) +
                    sum(v.size for v in part.recv_idx.values()))


# ---------------------------------------------------------------------------------------
# solves
# ---------------------------------------------------------------------------------------

def _part_graph(part: LocalPart, device: int):
    lib = _lib.load()
    h = ctypes.c_void_p()
    _lib.check(lib.gabp_graph_create_ex(part.n_local, part.pair_v.size, _lib.ptr(part.diag),
                                        _lib.ptr(part.rhs), _lib.ptr(part.pair_i),
                                        _lib.ptr(part.pair_j), _lib.ptr(part.pair_v),
                                        part.row_lo, part.row_hi, device, ctypes.byref(h)))
    return h


def _attach(h, part: LocalPart, nccl_id, bnorm: float):
    peers = np.array(part.peers, dtype=np.int32)
    empty = np.zeros(0, dtype=np.int64)
    sc = np.array([part.send_idx.get(p, empty).size for p in part.peers], dtype=np.int64)
    rc = np.array([part.recv_idx.get(p, empty).size for p in part.peers], dtype=np.int64)
    si = np.concatenate([part.send_idx.get(p, empty) for p in part.peers] + [empty])
    ri = np.concatenate([part.recv_idx.get(p, empty) for p in part.peers] + [empty])
    si = np.ascontiguousarray(si, dtype=np.int64)
    ri = np.ascontiguousarray(ri, dtype=np.int64)
    _lib.check(_lib.load().gabp_dist_attach(
        h, nccl_id, part.rank, part.world, part.n_global, float(bnorm), len(part.peers),
        _lib.ptr(peers) if peers.size else None, _lib.ptr(sc) if sc.size else None,
        _lib.ptr(si) if si.size else None, _lib.ptr(rc) if rc.size else None,
        _lib.ptr(ri) if ri.size else None))


def _report(parts, outs, rep, ch, rh, ms):
    from .solver import SolveReport
    n = sum(p.hi - p.lo for p in parts)
    means = np.empty(n)
    precs = np.empty(n)
    for p, (m, pr) in zip(parts, outs):
        means[p.lo:p.hi] = m
        precs[p.lo:p.hi] = pr
    k = int(rep.n_hist)
    return SolveReport(converged=bool(rep.converged), diverged=bool(rep.diverged),
                       iterations=int(rep.iterations), means=means, precisions=precs,
                       max_change_history=ch[:k].tolist(), residual_history=rh[:k].tolist(),
                       messages_sent=int(rep.messages_sent), device_ms=float(ms),
                       sweeps_launched=int(rep.sweeps_launched),
                       final_rel_residual=float(rep.final_rel_residual),
                       split_sweeps=int(rep.split_sweeps),
                       dist_layout=int(rep.dist_layout))


def solve_partitioned_local(system: SymSystem, nparts: int, options=None, device: int = 0):
    """The multi-rank broadcast solve with `nparts` row blocks on ONE device (halo moved by
    device copies, statistics reduced on the host): the partitioned kernels and halo lists
    exactly as the NCCL path runs them, testable without several GPUs."""
    from .solver import SolveOptions, _options_struct
    options = options or SolveOptions(schedule="broadcast")
    bounds = partition_rows(system.n, nparts)
    parts = [local_part(system, bounds, r) for r in range(nparts)]
    bnorm = float(np.sqrt(np.sum(system.rhs * system.rhs)))
    handles = [_part_graph(p, device) for p in parts]
    lib = _lib.load()
    try:
        for h, p in zip(handles, parts):
            _attach(h, p, None, bnorm)
        o = _options_struct(options, system.n, None)
        arr = (ctypes.c_void_p * nparts)(*[h.value for h in handles])
        ms = ctypes.c_double()
        _lib.check(lib.gabp_dist_solve_local(nparts, arr, ctypes.byref(o), ctypes.byref(ms)))
        outs = []
        ch = np.empty(options.max_iter)
        rh = np.empty(options.max_iter)
        rep = _lib.Report()
        for h, p in zip(handles, parts):
            m = np.empty(p.hi - p.lo)
            pr = np.empty(p.hi - p.lo)
            _lib.check(lib.gabp_dist_results(h, ctypes.byref(o), _lib.ptr(m), _lib.ptr(pr),
                                             _lib.ptr(ch), _lib.ptr(rh), ctypes.byref(rep)))
            outs.append((m, pr))
        return _report(parts, outs, rep, ch, rh, ms.value)
    finally:
        for h in handles:
            lib.gabp_graph_destroy(h)


def solve_grid_partitioned_local(spec, nparts: int, options=None, device: int = 0):
    """solve_partitioned_local for a Poisson grid generated on the device (grid.py): the
    nparts slabs are built from device arrays, never from a host system."""
    from . import grid as GR
    from .solver import SolveOptions, _options_struct
    options = options or SolveOptions(schedule="broadcast")
    rhs = GR.rhs_device(spec, device)
    bnorm = float(rhs.norm())
    parts, handles = [], []
    lib = _lib.load()
    try:
        for r in range(nparts):
            part = GR.grid_part(spec, nparts, r, device, rhs)
            handles.append(GR.part_graph(part, device))
            part.diag = part.rhs = part.pair_i = part.pair_j = part.pair_v = None
            parts.append(part)
        del rhs
        for h, p in zip(handles, parts):
            _attach(h, p, None, bnorm)
        o = _options_struct(options, spec.n, None)
        arr = (ctypes.c_void_p * nparts)(*[h.value for h in handles])
        ms = ctypes.c_double()
        _lib.check(lib.gabp_dist_solve_local(nparts, arr, ctypes.byref(o), ctypes.byref(ms)))
        outs = []
        ch = np.empty(options.max_iter)
        rh = np.empty(options.max_iter)
        rep = _lib.Report()
        for h, p in zip(handles, parts):
            m = np.empty(p.hi - p.lo)
            pr = np.empty(p.hi - p.lo)
            _lib.check(lib.gabp_dist_results(h, ctypes.byref(o), _lib.ptr(m), _lib.ptr(pr),
                                             _lib.ptr(ch), _lib.ptr(rh), ctypes.byref(rep)))
            outs.append((m, pr))
        return _report(parts, outs, rep, ch, rh, ms.value)
    finally:
        for h in handles:
            lib.gabp_graph_destroy(h)


def _nccl_id(rank: int, world: int, group):
    import torch.distributed as dist
    if world <= 1:
        return None
    raw = (ctypes.c_char * 128)()
    if rank == 0:
        _lib.check(_lib.load().gabp_nccl_unique_id(raw))
    obj = [bytes(raw) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return (ctypes.c_char * 128).from_buffer_copy(obj[0])


class DistributedGraph:
    """One rank's row block of a system, built once on this rank's GPU and attached to the
    multi-rank loop (NCCL halo exchange inside the CUDA library); solve() may be called
    repeatedly.  Every rank constructs it with the same system (or, from_grid, the same
    grid spec: then each rank generates only its own slab on its device)."""

    def __init__(self, system: SymSystem | None, group=None, device: int | None = None,
                 _grid=None):
        import torch.distributed as dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = _lib.default_device() if device is None else int(device)
        nid = _nccl_id(self.rank, self.world, group)
        if _grid is not None:
            from . import grid as GR
            self.n = _grid.n
            rhs = GR.rhs_device(_grid, self.device)
            bnorm = float(rhs.norm())
            self.part = GR.grid_part(_grid, self.world, self.rank, self.device, rhs)
            del rhs
            self._h = GR.part_graph(self.part, self.device)
            p = self.part
            p.diag = p.rhs = p.pair_i = p.pair_j = p.pair_v = None
        else:
            self.n = system.n
            bounds = partition_rows(system.n, self.world)
            self.part = local_part(system, bounds, self.rank)
            bnorm = float(np.sqrt(np.sum(system.rhs * system.rhs)))
            self._h = _part_graph(self.part, self.device)
        _attach(self._h, self.part, nid, bnorm)

    @classmethod
    def from_grid(cls, spec, group=None, device: int | None = None) -> "DistributedGraph":
        return cls(None, group, device, _grid=spec)

    def halo_bytes_per_sweep(self) -> int:
        if hasattr(self.part, "halo_bytes_per_sweep"):
            return self.part.halo_bytes_per_sweep()
        return halo_bytes_per_sweep(self.part)

    def graph_info(self):
        info = _lib.GraphInfo()
        _lib.check(_lib.load().gabp_graph_info(self._h, ctypes.byref(info)))
        return info

    @property
    def handle(self):
        return self._h

    @property
    def slice_path(self) -> bool:
        """The rank's block runs the slice-layout kernels (else the row tiles)."""
        info = _lib.GraphInfo()
        _lib.check(_lib.load().gabp_graph_info(self._h, ctypes.byref(info)))
        return int(info.num_slices) > 0

    def solve_local_report(self, options):
        """Solve; returns (this rank's owned means, precs, Report, change, residual)."""
        from .solver import _options_struct
        lib = _lib.load()
        o = _options_struct(options, self.n, None)
        if self.world == 1:  # one rank: the local driver (no NCCL needed)
            arr = (ctypes.c_void_p * 1)(self._h.value)
            ms = ctypes.c_double()
            _lib.check(lib.gabp_dist_solve_local(1, arr, ctypes.byref(o), ctypes.byref(ms)))
        p = self.part
        m = np.empty(p.hi - p.lo)
        pr = np.empty(p.hi - p.lo)
        ch = np.empty(options.max_iter)
        rh = np.empty(options.max_iter)
        rep = _lib.Report()
        if self.world > 1:
            _lib.check(lib.gabp_solve(self._h, ctypes.byref(o), _lib.ptr(m), _lib.ptr(pr),
                                      _lib.ptr(ch), _lib.ptr(rh), ctypes.byref(rep)))
        else:
            _lib.check(lib.gabp_dist_results(self._h, ctypes.byref(o), _lib.ptr(m),
                                             _lib.ptr(pr), _lib.ptr(ch), _lib.ptr(rh),
                                             ctypes.byref(rep)))
            rep.device_ms = ms.value
        return m, pr, rep, ch, rh

    def solve(self, options=None):
        """Full report on every rank (means gathered from all ranks)."""
        import torch.distributed as dist
        from .solver import SolveOptions
        options = options or SolveOptions(schedule="broadcast")
        m, pr, rep, ch, rh = self.solve_local_report(options)
        gathered = [None] * self.world
        dist.all_gather_object(gathered, (self.part.lo, self.part.hi, m, pr), group=self.group)
        parts = [type("P", (), {"lo": g[0], "hi": g[1]}) for g in gathered]
        return _report(parts, [(g[2], g[3]) for g in gathered], rep, ch, rh, rep.device_ms)

    def close(self):
        if getattr(self, "_h", None):
            _lib.load().gabp_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def solve_distributed(system: SymSystem, options=None, group=None):
    """Multi-GPU broadcast solve over torch.distributed ranks (one GPU per rank, NCCL
    halo exchange inside the CUDA library).  Every rank passes the same system and gets
    the full report (means gathered from all ranks)."""
    dg = DistributedGraph(system, group,
                          None if options is None else getattr(options, "device", None))
    try:
        return dg.solve(options)
    finally:
        dg.close()
