"""Drop-in surface of the reference solver module beyond solve(): point message functions,
assignable message buffers, the means history at any size, the serial schedule on rows of
any degree, run-to-run reproducibility and the agreed multi-rank launch protocol.

References: solver.py:100-143 (compute_message*), :57-74 + acceleration.py:123-126
(MessageState buffers assigned), :307-346 (means_history recorded every sweep),
:176-217 (serial sweep, any degree), linalg.py:285-288 (the residual of every sweep).
"""

import numpy as np
import pytest

import paper_0810_1119_b200 as G
from oracle import oracle
from paper_0810_1119_b200 import _lib
from paper_0810_1119_b200 import dist as D

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    _lib.load()
    assert _lib.device_count() > 0, "no CUDA device: " + _lib.last_error()
    oracle.build()


def _bits(a):
    return np.asarray(a, dtype=np.float64).view(np.uint64)


# ---- compute_message / compute_message_max_product ------------------------------------

def _msg_ref(graph, prec, mean, i, j, max_product=False):
    """solver.py:100-143 verbatim in arithmetic: python floats over the host buffers."""
    rp, dst, rev, coeff = graph.row_ptr, graph.dst, graph.rev, graph.coeff
    lo, hi = int(rp[i]), int(rp[i + 1])
    acc_p = float(graph.prior_prec[i])
    acc_num = float(graph.prior_prec[i]) * float(graph.prior_mean[i])
    a = None
    for e in range(lo, hi):
        if int(dst[e]) == j:
            a = float(coeff[e])
            continue
        acc_p += float(prec[rev[e]])
        acc_num += float(prec[rev[e]]) * float(mean[rev[e]])
    if max_product:
        mu = acc_num / acc_p
        p = -a * a / acc_p
        return p, -a * mu / p
    return -a * a / acc_p, acc_num / a


@pytest.mark.parametrize("kind", ["poisson", "random"])
def test_compute_message_equals_parallel_sweep(kind):
    s = G.gen_poisson2d(12, 3).system if kind == "poisson" else \
        G.gen_random_sparse(500, 6, 4).system
    g = G.build_graph(s)
    try:
        st = G.initial_state(g)
        for _ in range(3):
            st, _ = G.sweep(g, st, G.SolveOptions(schedule="parallel"))
        nxt, _ = G.sweep(g, st, G.SolveOptions(schedule="parallel"))
        p0, m0 = st.prec, st.mean
        p1, m1 = nxt.prec, nxt.mean
        rng = np.random.default_rng(0)
        src, dst = g.src, g.dst
        for e in rng.choice(g.num_edges, 40, replace=False):
            i, j = int(src[e]), int(dst[e])
            got = G.compute_message(g, st, i, j)
            # the parallel sweep's message of edge e, bit for bit (same sums, same order)
            assert _bits(got[0]) == _bits(p1[e]) and _bits(got[1]) == _bits(m1[e])
            assert _bits(got) .tolist() == _bits(_msg_ref(g, p0, m0, i, j)).tolist()
            mp = G.compute_message_max_product(g, st, i, j)
            assert _bits(mp).tolist() == _bits(_msg_ref(g, p0, m0, i, j, True)).tolist()
            np.testing.assert_allclose(mp, got, rtol=1e-12)
        with pytest.raises(KeyError):
            G.compute_message(g, st, 0, 0)
        with pytest.raises(KeyError):
            G.compute_message_max_product(g, st, g.n + 5, 0)
    finally:
        g.close()


def test_message_state_buffers_assignable():
    s = G.gen_poisson2d(8, 1).system
    g = G.build_graph(s)
    try:
        st = G.initial_state(g)
        rng = np.random.default_rng(2)
        p = rng.uniform(0.1, 1.0, g.num_edges)
        m = rng.standard_normal(g.num_edges)
        st.prec = p
        st.mean = m
        np.testing.assert_array_equal(st.prec, p)
        np.testing.assert_array_equal(st.mean, m)
        # a sweep from the assigned buffers is the oracle's sweep from the same buffers
        og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
        nxt, mc = G.sweep(g, st, G.SolveOptions(schedule="broadcast"))
        po, mo, mco, _ = oracle.sweep(og, p, m, "broadcast")
        np.testing.assert_array_equal(nxt.prec, po)
        np.testing.assert_array_equal(nxt.mean, mo)
        assert mc == mco
        with pytest.raises(ValueError):
            st.prec = np.zeros(3)
    finally:
        g.close()


# ---- means_history at any size (lazy replay) ------------------------------------------

@pytest.mark.parametrize("sched", ["broadcast", "parallel", "serial"])
def test_means_history_always_recorded(sched):
    s = G.gen_random_sparse(3000, 6, 9).system
    # n x max_iter = 3e7 > 2^24: recorded lazily (replayed on first access)
    opts = G.SolveOptions(schedule=sched, epsilon=1e-300, rel_residual_tol=1e-9,
                          max_iter=10_000)
    lazy = G.solve(s, opts)
    assert isinstance(lazy.means_history, G.MeansHistory)
    assert len(lazy.means_history) == lazy.iterations > 0
    eager = G.solve(s, G.SolveOptions(schedule=sched, epsilon=1e-300, rel_residual_tol=1e-9,
                                      max_iter=10_000, record_means_history=True))
    assert isinstance(eager.means_history, list)
    assert len(eager.means_history) == eager.iterations == lazy.iterations
    for t in (0, lazy.iterations // 2, lazy.iterations - 1):
        np.testing.assert_array_equal(_bits(lazy.means_history[t]),
                                      _bits(eager.means_history[t]))
    np.testing.assert_array_equal(_bits(lazy.means_history[-1]), _bits(lazy.means))
    off = G.solve(s, G.SolveOptions(schedule=sched, epsilon=1e-300, rel_residual_tol=1e-9,
                                    max_iter=10_000, record_means_history=False))
    assert off.means_history == []


# ---- serial schedule on rows of more than 256 edges -----------------------------------

def _hub_system(deg=400, seed=3):
    """A hub of degree `deg` plus a sparse random part: serial tasks past the 256-term
    shared-memory strip (the reference's loop has no such bound)."""
    rng = np.random.default_rng(seed)
    n = deg + 300
    pairs = {(0, j): rng.uniform(-1, 1) for j in range(1, deg + 1)}
    for _ in range(900):
        i, j = sorted(int(v) for v in rng.choice(np.arange(1, n), 2, replace=False))
        pairs[(i, j)] = rng.uniform(-1, 1)
    pi = np.array([p[0] for p in pairs], dtype=np.int64)
    pj = np.array([p[1] for p in pairs], dtype=np.int64)
    pv = np.array(list(pairs.values()))
    absrow = np.zeros(n)
    np.add.at(absrow, pi, np.abs(pv))
    np.add.at(absrow, pj, np.abs(pv))
    diag = 1.3 * absrow + (absrow == 0)
    return G.SymSystem.from_pairs(diag, pi, pj, pv, rng.standard_normal(n))


@pytest.mark.parametrize("order", ["ascending", "custom"])
def test_serial_high_degree_matches_oracle(order):
    s = _hub_system()
    og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
    o = None
    if order == "custom":
        o = list(np.random.default_rng(5).permutation(s.n)) + [0, 7]
    r = G.solve(s, G.SolveOptions(schedule="serial", epsilon=1e-300, max_iter=12,
                                  serial_order=o))
    w = oracle.solve_serial(og, epsilon=1e-300, max_iter=12, order=o)
    assert r.iterations == w.iterations == 12
    np.testing.assert_array_equal(r.means, w.means)
    np.testing.assert_array_equal(np.asarray(r.max_change_history), w.max_change_history)


def test_state_blown_reads_the_whole_state():
    s = G.gen_poisson2d(6, 0).system
    g = G.build_graph(s)
    try:
        st = G.initial_state(g)
        lib = _lib.load()
        import ctypes
        flag = ctypes.c_int32()
        _lib.check(lib.gabp_state_blown(st.handle, 1e10, ctypes.byref(flag)))
        assert flag.value == 0
        p = np.zeros(g.num_edges)
        p[g.num_edges // 2] = 2e10
        st.prec = p
        _lib.check(lib.gabp_state_blown(st.handle, 1e10, ctypes.byref(flag)))
        assert flag.value == 1
        p[g.num_edges // 2] = np.nan
        st.prec = p
        _lib.check(lib.gabp_state_blown(st.handle, 1e300, ctypes.byref(flag)))
        assert flag.value == 1
    finally:
        g.close()


# ---- run-to-run reproducibility -------------------------------------------------------

@pytest.mark.parametrize("sched,mode", [("broadcast", "auto"), ("parallel", "slice"),
                                        ("parallel", "auto")])
def test_solve_bitwise_reproducible_random_1m(sched, mode):
    """Two solves of config 1 (random 1M, k=16): the same residual history bit for bit and
    the same stop sweep -- the group kernels claim work dynamically, their residual
    partials are summed per group in group order (csrc/slice.cu grp_resid_commit)."""
    s = G.gen_random_sparse(1 << 20, 16, 0).system
    g = G.build_graph(s)
    try:
        opts = G.SolveOptions(schedule=sched, epsilon=1e-300, rel_residual_tol=1e-8,
                              gather_mode=mode, record_means_history=False)
        runs = [G.solve_graph(g, opts) for _ in range(3)]
    finally:
        g.close()
    a = runs[0]
    assert a.converged
    for b in runs[1:]:
        assert b.iterations == a.iterations
        np.testing.assert_array_equal(_bits(b.residual_history), _bits(a.residual_history))
        np.testing.assert_array_equal(_bits(b.max_change_history), _bits(a.max_change_history))
        np.testing.assert_array_equal(_bits(b.means), _bits(a.means))


def test_parallel_quad_kernel_equals_one_row_per_warp_and_oracle_1m(monkeypatch):
    """Config 1 at full size, parallel schedule: the four-rows-per-warp kernel (AUTO), the
    slice-group kernel and the oracle agree bit for bit over 6 sweeps (messages through the
    marginals and the change history; every row of 8..64 edges and both walk paths)."""
    from oracle import oracle
    oracle.build()
    s = G.gen_random_sparse(1 << 20, 16, 0).system
    kw = dict(schedule="parallel", epsilon=1e-300, max_iter=6, record_means_history=False)
    a = G.solve(s, G.SolveOptions(**kw))
    b = G.solve(s, G.SolveOptions(gather_mode="slice", **kw))
    og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
    o = oracle.solve(og, schedule="parallel", epsilon=1e-300, max_iter=6)
    assert a.iterations == b.iterations == o.iterations == 6
    np.testing.assert_array_equal(_bits(a.means), _bits(o.means))
    np.testing.assert_array_equal(_bits(b.means), _bits(o.means))
    np.testing.assert_array_equal(_bits(a.precisions), _bits(o.precisions))
    np.testing.assert_array_equal(_bits(np.asarray(a.max_change_history)),
                                  _bits(o.max_change_history))
    np.testing.assert_allclose(a.residual_history, o.residual_history, rtol=1e-9, atol=0)


def test_cluster_solve_reproducible_20_runs():
    """The one-launch cluster solve (remote shared-memory stores, cluster barriers): 20 runs
    of config 0 on both schedules give the same bits."""
    s = G.gen_poisson2d(32, 0).system
    g = G.build_graph(s)
    try:
        for sched in ("broadcast", "parallel"):
            opts = G.SolveOptions(schedule=sched, epsilon=1e-300, rel_residual_tol=1e-8,
                                  record_means_history=False)
            runs = [G.solve_graph(g, opts) for _ in range(20)]
            a = runs[0]
            assert a.kernel_launches == 1 and a.converged
            for b in runs[1:]:
                assert b.iterations == a.iterations
                np.testing.assert_array_equal(_bits(b.means), _bits(a.means))
                np.testing.assert_array_equal(_bits(b.residual_history),
                                              _bits(a.residual_history))
                np.testing.assert_array_equal(_bits(b.max_change_history),
                                              _bits(a.max_change_history))
    finally:
        g.close()


def test_probe_and_poll_modes_reproducible():
    s = G.gen_random_sparse(1 << 17, 16, 7).system
    outs = []
    for poll in (0, 1, 4):
        outs.append(G.solve(s, G.SolveOptions(schedule="broadcast", epsilon=1e-300,
                                              rel_residual_tol=1e-9, sweeps_per_poll=poll)))
    for b in outs[1:]:
        assert b.iterations == outs[0].iterations
        np.testing.assert_array_equal(_bits(b.residual_history),
                                      _bits(outs[0].residual_history))


# ---- multi-rank launch protocol agreed by all ranks -----------------------------------

@pytest.mark.parametrize("kind,nparts,split", [("poisson3d_32", 8, False),
                                               ("poisson2d_256", 4, True),
                                               ("poisson3d_32", 2, True)])
def test_partitions_agree_on_the_split(kind, nparts, split, monkeypatch):
    """Poisson 32^3 in 8 row blocks: the end blocks could split their sweep (one boundary
    plane), the middle ones cannot (two planes, 5 of 9 groups) -- every rank must then run
    whole sweeps, or the NCCL call sequences differ.  The solve stays bitwise
    the single-partition one either way."""
    s = G.gen_poisson3d(32, 1).system if kind.startswith("poisson3d") else \
        G.gen_poisson2d(256, 1).system
    opts = G.SolveOptions(schedule="broadcast", epsilon=1e-300, rel_residual_tol=1e-6,
                          max_iter=3000)
    one = G.solve(s, opts)
    # the grids would agree on the diagonal layout; this is the slice protocol's test
    monkeypatch.setenv("GABP_NO_DIST_DIA", "1")
    part = D.solve_partitioned_local(s, nparts, opts)
    assert part.dist_layout == 1
    assert (part.split_sweeps > 0) == split, part.split_sweeps
    assert part.iterations == one.iterations
    np.testing.assert_array_equal(part.means, one.means)
    np.testing.assert_array_equal(np.asarray(part.max_change_history),
                                  np.asarray(one.max_change_history))


@pytest.mark.parametrize("kind,nparts", [("poisson3d_32", 8), ("poisson2d_256", 3),
                                         ("stencil_random", 4)])
def test_partitions_on_the_diagonal_layout(kind, nparts):
    """Row blocks of stencil graphs agree on the diagonal layout (dist_layout 3): halo =
    {P, x} and the incoming messages on the diagonals that cross the cut; bitwise the
    single-partition solve, including unequal blocks (256 rows in 3) and a stencil with
    random coefficients."""
    from tests.test_dia_gpu import _random_stencil
    if kind == "poisson3d_32":
        s = G.gen_poisson3d(32, 1).system
    elif kind == "poisson2d_256":
        s = G.gen_poisson2d(256, 1).system
    else:  # random coefficients (no edge dropped: the host partitioner's halo is then the
        # whole neighbour row, so local ids keep the diagonal offsets)
        s = _random_stencil(64, 2, 3, drop=0.0)
    opts = G.SolveOptions(schedule="broadcast", epsilon=1e-300, rel_residual_tol=1e-7,
                          max_iter=4000)
    one = G.solve(s, opts)
    part = D.solve_partitioned_local(s, nparts, opts)
    assert part.dist_layout == 3
    assert part.iterations == one.iterations and part.converged == one.converged
    np.testing.assert_array_equal(part.means, one.means)
    np.testing.assert_array_equal(part.precisions, one.precisions)
    np.testing.assert_array_equal(np.asarray(part.max_change_history),
                                  np.asarray(one.max_change_history))


# ---- packed index upload (gabp_graph_create: 32-bit indices over the link) ---------------

def test_packed_index_upload_builds_the_same_graph(monkeypatch):
    """Systems of >= 2^20 pairs send their int64 pair indices packed to 32 bits (host
    threads, chunked under the copies) and widen them on the device: the graph is the one
    the plain upload builds, element for element."""
    s = G.gen_random_sparse(1 << 17, 16, 5).system
    assert s.pair_v.size >= 1 << 20
    g1 = G.build_graph(s)
    monkeypatch.setenv("GABP_NO_PACK", "1")
    g2 = G.build_graph(s)
    try:
        for name in ("src", "dst", "rev", "coeff"):
            np.testing.assert_array_equal(getattr(g1, name), getattr(g2, name), err_msg=name)
    finally:
        g1.close()
        g2.close()


@pytest.mark.parametrize("bad", [-1, 1 << 40])
def test_packed_index_upload_rejects_bad_indices_like_the_plain_one(bad):
    """An index that does not fit 32 bits leaves the packed path; the device validation
    reports it exactly as for a small system."""
    s = G.gen_random_sparse(1 << 17, 16, 5).system
    pi = s.pair_i.copy()
    pi[12345] = bad
    t = G.SymSystem.from_pairs(s.diag, pi, s.pair_j, s.pair_v, s.rhs, validate=False)
    with pytest.raises(ValueError, match="bad off-diagonal"):
        G.build_graph(t)


# ---- cross-check variants stay bitwise equal to the default kernels ----------------------

def test_parallel_one_row_per_warp_equals_four_rows_per_warp(monkeypatch):
    """GABP_ROW_NO_QUAD selects the round-1 warp-per-row kernel (rowpar_kernel): same bits
    as rowquad_kernel on a graph with rows of 0..120 edges (the long-row path included)."""
    rng = np.random.default_rng(3)
    n = 20000
    deg = np.minimum(rng.poisson(14, n) + (rng.random(n) < 0.01) * 90, 120)
    pi = np.repeat(np.arange(n), deg)
    pj = rng.integers(0, n, pi.size)
    keep = pi != pj
    lo, hi = np.minimum(pi[keep], pj[keep]), np.maximum(pi[keep], pj[keep])
    key = np.unique(lo.astype(np.int64) * n + hi)
    pi, pj = key // n, key % n
    pv = rng.uniform(-1.0, 1.0, pi.size)
    pv[pv == 0.0] = 0.5
    absrow = np.bincount(pi, np.abs(pv), n) + np.bincount(pj, np.abs(pv), n)
    s = G.SymSystem.from_pairs(1.2 * absrow + (absrow == 0), pi, pj, pv, rng.standard_normal(n))
    kw = dict(schedule="parallel", gather_mode="rows", epsilon=1e-300, max_iter=12,
              record_means_history=True)
    a = G.solve(s, G.SolveOptions(**kw))
    monkeypatch.setenv("GABP_ROW_NO_QUAD", "1")
    b = G.solve(s, G.SolveOptions(**kw))
    assert a.iterations == b.iterations == 12
    for x, y in zip(a.means_history, b.means_history):
        np.testing.assert_array_equal(_bits(x), _bits(y))
    np.testing.assert_array_equal(_bits(np.asarray(a.max_change_history)),
                                  _bits(np.asarray(b.max_change_history)))
    np.testing.assert_array_equal(_bits(a.precisions), _bits(b.precisions))


def test_dense_two_kernel_sweep_equals_fused_sweep(monkeypatch):
    """GABP_DENSE_TWO_KERNELS selects the column walk + pair tiles: same trajectory as the
    fused one-kernel sweep (K = 300: padded tiles, diagonal tiles, exact zeros of A)."""
    s = G.gen_cdma_detection(512, 300, 0.5, 4)[0].system
    kw = dict(schedule="broadcast", epsilon=1e-300, max_iter=25, record_means_history=True)
    g = G.build_graph(s, dense=True)
    try:
        a = G.solve_graph(g, G.SolveOptions(**kw))
        monkeypatch.setenv("GABP_DENSE_TWO_KERNELS", "1")
        b = G.solve_graph(g, G.SolveOptions(**kw))
    finally:
        g.close()
    assert (a.iterations, a.diverged) == (b.iterations, b.diverged)
    assert len(a.means_history) == len(b.means_history)
    for x, y in zip(a.means_history, b.means_history):
        np.testing.assert_array_equal(_bits(x), _bits(y))
    np.testing.assert_array_equal(_bits(np.asarray(a.max_change_history)),
                                  _bits(np.asarray(b.max_change_history)))
    np.testing.assert_allclose(a.residual_history, b.residual_history, rtol=1e-9, atol=0)
