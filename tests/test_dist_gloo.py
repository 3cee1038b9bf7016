"""Multi-rank host logic on CPU (gloo, world_size 2 and 3).

Each rank runs the distributed broadcast sweep exactly as the CUDA path does it -- owned
rows only, incoming messages rebuilt from node aggregates (the recompute gather), halo
aggregates exchanged per sweep over torch.distributed -- in numpy, then the messages and
marginals gathered on rank 0 must equal the single-process oracle BITWISE at every sweep.
This pins the partition, the order-preserving local numbering and the halo lists that the
GPU path (gabp_graph_create_ex / gabp_dist_attach) consumes.
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_0810_1119_b200 as G
from oracle import oracle
from paper_0810_1119_b200 import dist as D

SWEEPS = 12


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _system(kind):
    if kind == "poisson":
        return G.gen_poisson2d(24, 3).system
    return G.gen_random_sparse(600, 6, 11).system


def _local_run(part, exchange):
    """Distributed broadcast sweeps of one rank (numpy, reference operation order)."""
    g = oracle.build_graph(part.diag, part.rhs, part.pair_i, part.pair_j, part.pair_v)
    src = g.src
    own_e = (src >= part.row_lo) & (src < part.row_hi)
    eids = np.flatnonzero(own_e)
    rows = np.arange(part.row_lo, part.row_hi)
    col = g.col[eids]
    c = g.coeff[eids]
    prior_num = part.diag * (part.rhs / part.diag)
    E = eids.size
    m1 = np.zeros((E, 2))          # S_{s-1} on owned edges
    m2 = np.zeros((E, 2))          # S_{s-2}
    agg2 = np.zeros((part.n_local, 2))  # Agg(S_{s-2}) on local + halo nodes
    hist = []
    for s in range(1, SWEEPS + 1):
        if s == 1:
            pin = np.zeros(E)
            muin = np.zeros(E)
        else:   # rebuild m_ji^{(s-1)} exactly as node j built it (broadcast_sweep)
            pe = agg2[col, 0] - m2[:, 0]
            num = agg2[col, 1] - m2[:, 0] * m2[:, 1]
            pin = -c * c / pe
            muin = num / c
        sp = part.diag[rows].copy()
        sn = prior_num[rows].copy()
        local_row = src[eids] - part.row_lo
        np.add.at(sp, local_row, pin)              # ascending neighbour order
        np.add.at(sn, local_row, pin * muin)
        mu_t = sn / sp
        nn = sp * mu_t
        pe = sp[local_row] - pin
        num = nn[local_row] - pin * muin
        new = np.stack([-c * c / pe, num / c], axis=1)
        agg_now = np.zeros((part.n_local, 2))      # Agg(S_{s-1})
        agg_now[rows, 0] = sp
        agg_now[rows, 1] = nn
        exchange(agg_now)                          # fill the halo entries
        hist.append((new.copy(), (sn / sp).copy()))
        m2, m1, agg2 = m1, new, agg_now
    return eids, g, hist


def _worker(rank, world, port, kind, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    system = _system(kind)
    bounds = D.partition_rows(system.n, world)
    part = D.local_part(system, bounds, rank)

    def exchange(agg):
        reqs, bufs = [], {}
        for peer in part.peers:
            if peer in part.send_idx:
                t = torch.from_numpy(np.ascontiguousarray(agg[part.send_idx[peer]]))
                reqs.append(dist.isend(t, peer))
            if peer in part.recv_idx:
                bufs[peer] = torch.empty((part.recv_idx[peer].size, 2), dtype=torch.float64)
                reqs.append(dist.irecv(bufs[peer], peer))
        for r in reqs:
            r.wait()
        for peer, t in bufs.items():
            agg[part.recv_idx[peer]] = t.numpy()

    eids, g, hist = _local_run(part, exchange)
    # map owned local edges to global edge ids: same position inside the row
    gsrc = part.glob[g.src[eids]]
    pos = eids - g.row_ptr[g.src[eids]]
    q.put((rank, gsrc, pos, [h[0] for h in hist], [h[1] for h in hist], part.lo, part.hi,
           D.halo_bytes_per_sweep(part)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("kind,world", [("poisson", 2), ("random", 2), ("poisson", 3)])
def test_distributed_sweeps_bitwise_equal_single_process(kind, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    system = _system(kind)
    og = oracle.build_graph(system.diag, system.rhs, system.pair_i, system.pair_j,
                            system.pair_v)
    E = og.num_edges
    p = np.zeros(E)
    m = np.zeros(E)
    for s in range(SWEEPS):
        p_new, m_new, _, _ = oracle.sweep(og, p, m, "broadcast")
        means, _ = oracle.marginals(og, p, m)   # marginals of the state read (S_{s-1})
        got_p = np.full(E, np.nan)
        got_m = np.full(E, np.nan)
        got_x = np.full(system.n, np.nan)
        for (rank, gsrc, pos, msgs, xs, lo, hi, _) in res:
            ge = og.row_ptr[gsrc] + pos
            got_p[ge] = msgs[s][:, 0]
            got_m[ge] = msgs[s][:, 1]
            got_x[lo:hi] = xs[s]
        np.testing.assert_array_equal(got_p, p_new)
        np.testing.assert_array_equal(got_m, m_new)
        np.testing.assert_array_equal(got_x, means)
        p, m = p_new, m_new
    # the halo is node-level and small
    assert all(r[7] > 0 for r in res)


def test_partition_properties():
    s = G.gen_poisson2d(64, 0).system
    bounds = D.partition_rows(s.n, 4)
    assert bounds[0] == 0 and bounds[-1] == s.n and np.all(np.diff(bounds) == s.n // 4)
    for r in range(4):
        part = D.local_part(s, bounds, r)
        assert np.all(np.diff(part.glob) > 0)              # order-preserving local ids
        assert np.all(part.pair_i < part.pair_j)
        assert part.glob[part.row_lo] == part.lo and part.glob[part.row_hi - 1] == part.hi - 1
        # strips of a 64x64 grid: one grid row of halo per interior side
        expect = 64 * ((r > 0) + (r < 3))
        assert sum(v.size for v in part.recv_idx.values()) == expect
        assert sum(v.size for v in part.send_idx.values()) == expect
