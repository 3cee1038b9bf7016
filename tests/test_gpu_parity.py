"""CUDA path vs the reference (golden fixtures) and the C oracle -- the parity gate.

Bar: bitwise for messages, marginals, change history and iteration counts (the kernels
use the reference's operation order without FMA contraction); the in-solve residual
history is reduced in a different order and is compared to 1e-9 relative.
"""

import ctypes

import numpy as np
import pytest

import paper_0810_1119_b200 as G
from oracle import oracle
from paper_0810_1119_b200 import _lib
from tests import golden_cases as gc

pytestmark = pytest.mark.gpu
CASES = gc.names()
SCHEDS = ["parallel", "broadcast"]


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    _lib.load()
    assert _lib.device_count() > 0, "no CUDA device: " + _lib.last_error()
    oracle.build()


def _res_close(got, want):
    got = np.asarray(got)
    want = np.asarray(want)
    assert got.shape == want.shape
    fin = np.isfinite(want)
    np.testing.assert_array_equal(np.isfinite(got), fin)
    atol = 1e-12 * float(np.max(want[fin], initial=0.0))
    np.testing.assert_allclose(got[fin], want[fin], rtol=1e-9, atol=atol)


@pytest.mark.parametrize("case", CASES)
def test_graph_build_matches_reference(case):
    rec = gc.load(case)
    g = G.build_graph(gc.system(rec))
    np.testing.assert_array_equal(g.src, rec["src"])
    np.testing.assert_array_equal(g.dst, rec["dst"])
    np.testing.assert_array_equal(g.rev, rec["rev"])
    np.testing.assert_array_equal(g.coeff, rec["coeff"])


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("sched", SCHEDS)
def test_sweep_trace_bitwise(case, sched):
    rec = gc.load(case)
    g = G.build_graph(gc.system(rec))
    st = G.initial_state(g, sched)
    opts = G.SolveOptions(schedule=sched)
    tp, tm, tc = (rec[f"{sched}_trace_prec"], rec[f"{sched}_trace_mean"],
                  rec[f"{sched}_trace_change"])
    for t in range(tp.shape[0]):
        st, change = G.sweep(g, st, opts)
        np.testing.assert_array_equal(st.prec, tp[t])
        np.testing.assert_array_equal(st.mean, tm[t])
        assert change == tc[t]
        assert st.iteration == t + 1
    if int(rec[f"{sched}_trace_singular_at"]) > 0:
        with pytest.raises(G.SingularSubgraphError):
            G.sweep(g, st, opts)


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("sched", SCHEDS)
def test_marginals_bitwise_vs_oracle(case, sched):
    rec = gc.load(case)
    g = G.build_graph(gc.system(rec))
    og = oracle.build_graph(rec["diag"], rec["rhs"], rec["pair_i"], rec["pair_j"],
                            rec["pair_v"])
    st = G.initial_state(g, sched)
    for t in range(rec[f"{sched}_trace_prec"].shape[0]):
        st, _ = G.sweep(g, st, G.SolveOptions(schedule=sched))
        means, precs = G.infer_marginals(g, st)
        om, op = oracle.marginals(og, st.prec, st.mean)
        np.testing.assert_array_equal(means, om)
        np.testing.assert_array_equal(precs, op)


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("sched,mode", [("parallel", "auto"), ("broadcast", "auto"),
                                        ("broadcast", "slice")])
@pytest.mark.parametrize("poll", [0, 1, 3])
def test_solve_matches_reference(case, sched, mode, poll):
    """auto: small graphs solve in one persistent CTA (csrc/small.cu); slice: the same
    fixtures through the sweep-per-launch loop of the slice kernels."""
    rec = gc.load(case)
    tol = float(rec["rel_residual_tol"]) or None
    opts = G.SolveOptions(schedule=sched, epsilon=float(rec["epsilon"]),
                          max_iter=int(rec["max_iter"]), rel_residual_tol=tol,
                          sweeps_per_poll=poll, gather_mode=mode)
    r = G.solve(gc.system(rec), opts)
    assert r.converged == bool(rec[f"{sched}_converged"])
    assert r.diverged == bool(rec[f"{sched}_diverged"])
    assert r.converged != r.diverged
    assert r.iterations == int(rec[f"{sched}_iterations"])
    want = rec[f"{sched}_means"]
    fin = np.isfinite(want)
    np.testing.assert_array_equal(np.isfinite(r.means), fin)
    np.testing.assert_array_equal(r.means[fin], want[fin])
    np.testing.assert_array_equal(r.precisions, rec[f"{sched}_precisions"])
    ch = rec[f"{sched}_change_hist"]
    got = np.asarray(r.max_change_history)
    assert got.shape == ch.shape
    # every entry, the non-finite ones included (NaN when a new message is NaN, as the
    # reference's np.max propagates it; NaN == NaN for assert_array_equal)
    np.testing.assert_array_equal(got, ch)
    _res_close(r.residual_history, rec[f"{sched}_res_hist"])
    assert len(r.residual_history) == len(r.max_change_history)
    if r.means_history:
        assert len(r.means_history) == len(r.max_change_history)
        if r.iterations == len(r.means_history) and r.iterations > 0:
            np.testing.assert_array_equal(r.means_history[-1][fin], want[fin])


def test_toy3_trace_and_report():
    """Reference solver tests test_solve_toy3_counts_and_trace / test_marginals_toy3."""
    sys3 = G.load_instance("toy3").system
    r = G.solve(sys3, G.SolveOptions(schedule="parallel"))
    assert r.converged and not r.diverged and r.iterations == 3
    np.testing.assert_allclose(r.means, [1.0, 2.0, -1.0], atol=1e-14)
    np.testing.assert_allclose(r.precisions, [-12.0, 1.5, 4.0], atol=1e-14)
    assert r.precisions_exact is True
    np.testing.assert_allclose(r.means_history[0], [1.0, 4.0, -2.5], atol=1e-14)
    np.testing.assert_allclose(r.means_history[1], [1.0, 2.0, -1.0], atol=1e-14)
    assert r.messages_sent == 3 * 4


def test_broadcast_message_accounting():
    system = G.gen_random("spd", 10, 17).system
    g = G.build_graph(system)
    naive, _ = G.sweep(g, G.initial_state(g), G.SolveOptions())
    bcast, _ = G.broadcast_sweep(g, G.initial_state(g, "broadcast"))
    assert naive.messages_sent == 90
    assert bcast.messages_sent == 10


def test_sweep_is_functional():
    """sweep returns a new state; the input state is unchanged (solver.py:166-173)."""
    g = G.build_graph(G.load_instance("cdma4").system)
    s0 = G.initial_state(g)
    s1, _ = G.sweep(g, s0, G.SolveOptions())
    s2, _ = G.sweep(g, s1, G.SolveOptions())
    assert np.all(s0.prec == 0.0) and s0.iteration == 0
    assert s1.iteration == 1 and s2.iteration == 2
    assert not np.array_equal(s1.mean, s2.mean)


def test_identity_system_noop():
    ident = G.SymSystem(diag=np.ones(3), offdiag={}, rhs=np.array([1.0, 2.0, 3.0]))
    g = G.build_graph(ident)
    st, change = G.sweep(g, G.initial_state(g), G.SolveOptions())
    assert change == 0.0 and st.prec.size == 0
    means, precs = G.infer_marginals(g, st)
    np.testing.assert_array_equal(means, ident.rhs)
    np.testing.assert_array_equal(precs, np.ones(3))


def test_single_node():
    s = G.SymSystem(diag=np.array([2.0]), offdiag={}, rhs=np.array([3.0]))
    r = G.solve(s)
    assert r.converged and r.iterations == 1
    assert r.means[0] == 1.5


def test_zero_diagonal_rejected():
    s = G.SymSystem(diag=np.array([1.0, 0.0, 1.0]), offdiag={(0, 1): 2.0}, rhs=np.zeros(3))
    with pytest.raises(G.ZeroDiagonalError, match="row 1"):
        G.build_graph(s)


def test_duplicate_pair_rejected_by_device_builder():
    s = G.SymSystem.from_pairs(np.full(3, 4.0), [0, 0], [1, 1], [1.0, 2.0], np.ones(3),
                               validate=False)
    with pytest.raises(ValueError, match="duplicate"):
        G.build_graph(s)


def test_bad_pair_rejected_by_device_builder():
    s = G.SymSystem.from_pairs(np.full(3, 4.0), [1], [0], [1.0], np.ones(3), validate=False)
    with pytest.raises(ValueError, match="bad off-diagonal"):
        G.build_graph(s)


def test_unsorted_pair_order_same_graph():
    """Pair order in the input never changes edge ids or results."""
    base = G.gen_random_sparse(500, 8, 3).system
    perm = np.random.default_rng(0).permutation(base.pair_v.size)
    shuf = G.SymSystem.from_pairs(base.diag, base.pair_i[perm], base.pair_j[perm],
                                  base.pair_v[perm], base.rhs)
    a = G.solve(base, G.SolveOptions(rel_residual_tol=1e-10, epsilon=1e-300))
    b = G.solve(shuf, G.SolveOptions(rel_residual_tol=1e-10, epsilon=1e-300))
    assert a.iterations == b.iterations
    np.testing.assert_array_equal(a.means, b.means)


def test_dense_entry_point_matches_sparse():
    inst, _ = G.gen_cdma_detection(64, 32, 0.5, 2)
    a, b = inst.system.to_dense()
    lib = _lib.load()
    h = ctypes.c_void_p()
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    _lib.check(lib.gabp_graph_create_dense(32, _lib.ptr(a), _lib.ptr(b), 0, ctypes.byref(h)))
    try:
        o = G.solver._options_struct(G.SolveOptions(schedule="broadcast"), 32, None)
        means = np.empty(32)
        rep = _lib.Report()
        _lib.check(lib.gabp_solve(h, ctypes.byref(o), _lib.ptr(means), None, None, None,
                                  ctypes.byref(rep)))
    finally:
        lib.gabp_graph_destroy(h)
    ref = G.solve(inst.system, G.SolveOptions(schedule="broadcast"))
    assert rep.iterations == ref.iterations
    np.testing.assert_array_equal(means, ref.means)


def test_c_abi_solve_system_host_buffers():
    """The one-call drop-in (gabp_solve_system) with host buffers."""
    s = G.gen_poisson2d(32, 0).system
    lib = _lib.load()
    o = G.solver._options_struct(G.SolveOptions(schedule="broadcast", epsilon=1e-300,
                                                rel_residual_tol=1e-8), s.n, None)
    means = np.empty(s.n)
    ch = np.empty(o.max_iter)
    rh = np.empty(o.max_iter)
    rep = _lib.Report()
    _lib.check(lib.gabp_solve_system(s.n, s.pair_v.size, _lib.ptr(s.diag), _lib.ptr(s.rhs),
                                     _lib.ptr(s.pair_i), _lib.ptr(s.pair_j), _lib.ptr(s.pair_v),
                                     0, ctypes.byref(o), _lib.ptr(means), None, _lib.ptr(ch),
                                     _lib.ptr(rh), ctypes.byref(rep)))
    og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
    orc = oracle.solve(og, epsilon=1e-300, schedule="broadcast", rel_residual_tol=1e-8)
    assert rep.converged and rep.iterations == orc.iterations
    np.testing.assert_array_equal(means, orc.means)
    assert rep.final_rel_residual < 1e-8


def test_residual_norm_per_eq_matches_oracle():
    s = G.gen_random_sparse(2000, 16, 5).system
    g = G.build_graph(s)
    x = np.random.default_rng(1).standard_normal(s.n)
    out = ctypes.c_double()
    _lib.check(_lib.load().gabp_residual_norm_per_eq(g.handle, _lib.ptr(x), ctypes.byref(out)))
    og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
    assert out.value == np.sqrt(oracle.residual_sq(og, x)) / s.n


# ---------------------------------------------------------------------------------------
# BASELINE configs at (near) full size: bitwise vs the oracle where it finishes in
# seconds, size-independent properties otherwise.
# ---------------------------------------------------------------------------------------

@pytest.mark.parametrize("sched", SCHEDS)
def test_config1_random_1M_full_solve(sched):
    s = G.gen_random_sparse(1 << 20, 16, 0).system
    opts = G.SolveOptions(schedule=sched, epsilon=1e-300, rel_residual_tol=1e-8)
    r = G.solve(s, opts)
    og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
    orc = oracle.solve(og, epsilon=1e-300, schedule=sched, rel_residual_tol=1e-8)
    assert r.converged and orc.converged
    assert r.iterations == orc.iterations
    np.testing.assert_array_equal(r.means, orc.means)
    np.testing.assert_array_equal(r.precisions, orc.precisions)
    np.testing.assert_array_equal(np.asarray(r.max_change_history), orc.max_change_history)
    _res_close(r.residual_history, orc.residual_history)
    # independent check of the answer
    rel = np.linalg.norm(s.matvec(r.means) - s.rhs) / np.linalg.norm(s.rhs)
    assert rel < 1e-8


def test_config2_poisson_4096_sweeps_vs_oracle():
    """n = 16.8M: five sweeps bitwise against the oracle, then the marginals."""
    s = G.gen_poisson2d(4096, 0).system
    g = G.build_graph(s)
    og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
    st = G.initial_state(g, "broadcast")
    p = np.zeros(g.num_edges)
    m = np.zeros(g.num_edges)
    for _ in range(5):
        st, c = G.broadcast_sweep(g, st)
        p, m, oc, _ = oracle.sweep(og, p, m, "broadcast")
        assert c == oc
    np.testing.assert_array_equal(st.prec, p)
    np.testing.assert_array_equal(st.mean, m)
    means, _ = G.infer_marginals(g, st)
    om, _ = oracle.marginals(og, p, m)
    np.testing.assert_array_equal(means, om)


def test_config3_cdma_full_dense_vs_oracle():
    """K = 4096 users, N = 8192 chips, all K^2 edges, dense kernels: GaBP diverges on this
    instance (K/N = 0.5, sigma^2 = 0.5 is not walk-summable); the run must reproduce the
    oracle's trajectory bitwise -- same sweep of divergence, same last means."""
    inst, _ = G.gen_cdma_detection(8192, 4096, 0.5, 0)
    s = inst.system
    opts = G.SolveOptions(schedule="broadcast", epsilon=1e-300, rel_residual_tol=1e-8,
                          max_iter=2000)
    g = G.build_graph(s)
    assert g.info.is_dense
    r = G.solve_graph(g, opts)
    og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
    orc = oracle.solve(og, epsilon=1e-300, schedule="broadcast", rel_residual_tol=1e-8,
                       max_iter=2000)
    assert r.diverged == orc.diverged and r.converged == orc.converged
    assert r.iterations == orc.iterations
    np.testing.assert_array_equal(np.asarray(r.max_change_history), orc.max_change_history)
    fin = np.isfinite(orc.means)
    np.testing.assert_array_equal(r.means[fin], orc.means[fin])


@pytest.mark.parametrize("K,N,seed", [(32, 64, 2), (200, 400, 5), (300, 1200, 9)])
def test_dense_kernels_bitwise_equal_sparse(K, N, seed):
    inst, _ = G.gen_cdma_detection(N, K, 0.5, seed)
    s = inst.system
    opts = G.SolveOptions(schedule="broadcast", epsilon=1e-300, rel_residual_tol=1e-10,
                          max_iter=400)
    d = G.solve_graph(G.build_graph(s, dense=True), opts)
    sp = G.solve_graph(G.build_graph(s, dense=False), opts)
    assert d.iterations == sp.iterations and d.converged == sp.converged
    np.testing.assert_array_equal(d.means, sp.means)
    np.testing.assert_array_equal(d.precisions, sp.precisions)
    np.testing.assert_array_equal(np.asarray(d.max_change_history),
                                  np.asarray(sp.max_change_history))
    _res_close(d.residual_history, sp.residual_history)


def test_config4_poisson3d_small_slab_vs_oracle():
    s = G.gen_poisson3d(64, 0).system
    r = G.solve(s, G.SolveOptions(schedule="broadcast", max_iter=30, epsilon=1e-300))
    og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
    orc = oracle.solve(og, epsilon=1e-300, max_iter=30, schedule="broadcast")
    assert r.iterations == orc.iterations == 30 and r.diverged and orc.diverged
    np.testing.assert_array_equal(r.means, orc.means)


def _subbox_system(s, p, lo, L):
    """The 3-D grid system restricted to the box [lo, lo + L)^3 (z, y, x), nodes renumbered
    lexicographically -- so every row keeps its neighbours in ascending order."""
    z, y, x = np.meshgrid(*(np.arange(c, c + L) for c in lo), indexing="ij")
    glob = (z * p * p + y * p + x).ravel()
    loc = -np.ones(p ** 3, dtype=np.int64)
    loc[glob] = np.arange(glob.size)
    li, lj = loc[s.pair_i], loc[s.pair_j]
    keep = (li >= 0) & (lj >= 0)
    sub = G.SymSystem.from_pairs(s.diag[glob], li[keep], lj[keep], s.pair_v[keep], s.rhs[glob])
    return sub, glob


def test_config4_full_size_locality_vs_oracle():
    """Config 4 at full size (512^3, 804M directed edges) on one GPU.  After T sweeps from
    zero messages a marginal depends only on the rows within T+1 hops, so on a sub-box
    the oracle (run on the restricted system) must reproduce the full-size marginals bitwise
    wherever the sub-box's cut faces are more than T+1 hops away.  Two boxes: one at the
    domain corner (three true Dirichlet faces), one in the interior."""
    p, T, L = 512, 6, 40
    s = G.gen_poisson3d(p, 0).system
    r = G.solve(s, G.SolveOptions(schedule="broadcast", epsilon=1e-300, max_iter=T,
                                  record_means_history=False))
    assert r.iterations == T
    m = T + 2  # margin from a cut face
    for lo in ((0, 0, 0), (200, 300, 100)):
        sub, glob = _subbox_system(s, p, lo, L)
        og = oracle.build_graph(sub.diag, sub.rhs, sub.pair_i, sub.pair_j, sub.pair_v)
        orc = oracle.solve(og, epsilon=1e-300, max_iter=T, schedule="broadcast")
        assert orc.iterations == T
        k = np.arange(L)
        ok_axis = [(k >= (0 if c == 0 else m)) & (k < L - m) for c in lo]
        inner = (ok_axis[0][:, None, None] & ok_axis[1][None, :, None] &
                 ok_axis[2][None, None, :]).ravel()
        assert inner.sum() > 1000
        np.testing.assert_array_equal(r.means[glob[inner]], orc.means[inner])
        np.testing.assert_array_equal(r.precisions[glob[inner]], orc.precisions[inner])


@pytest.mark.parametrize("case", CASES)
def test_gather_modes_bitwise_identical(case):
    """Broadcast solve with the twin-message gather and with the aggregate recompute
    (sweep.cu): same iterations, means, precisions and change history as the reference."""
    rec = gc.load(case)
    tol = float(rec["rel_residual_tol"]) or None
    out = {}
    for mode in ("message", "recompute", "slice"):
        opts = G.SolveOptions(schedule="broadcast", epsilon=float(rec["epsilon"]),
                              max_iter=int(rec["max_iter"]), rel_residual_tol=tol,
                              gather_mode=mode)
        out[mode] = G.solve(gc.system(rec), opts)
    a = out["message"]
    for b in (out["recompute"], out["slice"]):
        assert a.iterations == b.iterations == int(rec["broadcast_iterations"])
        assert a.converged == b.converged
        np.testing.assert_array_equal(a.means, b.means)
        np.testing.assert_array_equal(a.precisions, b.precisions)
        np.testing.assert_array_equal(np.asarray(a.max_change_history),
                                      np.asarray(b.max_change_history))


@pytest.mark.parametrize("mode", ["message", "recompute", "slice"])
def test_config1_gather_modes(mode):
    s = G.gen_random_sparse(1 << 18, 16, 3).system
    opts = G.SolveOptions(schedule="broadcast", epsilon=1e-300, rel_residual_tol=1e-10,
                          gather_mode=mode)
    r = G.solve(s, opts)
    og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
    orc = oracle.solve(og, epsilon=1e-300, schedule="broadcast", rel_residual_tol=1e-10)
    assert r.iterations == orc.iterations
    np.testing.assert_array_equal(r.means, orc.means)


# ---------------------------------------------------------------------------------------
# multi-rank path: row blocks as in-process partitions on one GPU (same kernels, halo
# lists and decision logic as the NCCL path)
# ---------------------------------------------------------------------------------------

@pytest.mark.parametrize("kind,nparts", [("poisson", 1), ("poisson", 2), ("poisson", 4),
                                         ("random", 3), ("cdma", 2), ("toy", 2),
                                         ("cdma_big", 2)])
def test_partitioned_solve_bitwise_equal_single(kind, nparts):
    from paper_0810_1119_b200 import dist as D
    if kind == "poisson":
        s = G.gen_poisson2d(64, 5).system
    elif kind == "random":
        s = G.gen_random_sparse(20000, 8, 2).system
    elif kind == "cdma":
        s = G.gen_cdma_detection(64, 32, 0.5, 2)[0].system
    elif kind == "cdma_big":  # rows of degree ~400: unstaged (slow) tiles with cut edges
        s = G.gen_cdma_detection(1024, 400, 0.5, 2)[0].system
    else:
        s = G.load_instance("cdma4").system
    opts = G.SolveOptions(schedule="broadcast", epsilon=1e-300, rel_residual_tol=1e-9,
                          max_iter=3000)
    if kind == "toy":
        opts = G.SolveOptions(schedule="broadcast")
    one = G.solve(s, opts)
    part = D.solve_partitioned_local(s, nparts, opts)
    assert part.iterations == one.iterations
    assert part.converged == one.converged
    np.testing.assert_array_equal(part.means, one.means)
    np.testing.assert_array_equal(part.precisions, one.precisions)
    np.testing.assert_array_equal(np.asarray(part.max_change_history),
                                  np.asarray(one.max_change_history))
    _res_close(part.residual_history, one.residual_history)


# ---------------------------------------------------------------------------------------
# slice layout (csrc/slice.cu): degree-sorted 32-row slices, lane per row
# ---------------------------------------------------------------------------------------

def _ragged_system(seed=5):
    """Isolated nodes, a degree-100 hub, a chain and random pairs; n not a multiple of 32."""
    rng = np.random.default_rng(seed)
    n = 1000
    pairs = {}
    for j in range(1, 101):                       # hub 0
        pairs[(0, j)] = rng.uniform(-1, 1)
    for i in range(200, 400):                     # chain
        pairs[(i, i + 1)] = rng.uniform(-1, 1)
    for _ in range(1500):                         # random sparse part
        i, j = sorted(rng.choice(np.arange(400, 980), 2, replace=False))
        pairs[(int(i), int(j))] = rng.uniform(-1, 1)
    # rows 980..999 stay isolated
    pi = np.array([p[0] for p in pairs], dtype=np.int64)
    pj = np.array([p[1] for p in pairs], dtype=np.int64)
    pv = np.array(list(pairs.values()))
    absrow = np.zeros(n)
    np.add.at(absrow, pi, np.abs(pv))
    np.add.at(absrow, pj, np.abs(pv))
    diag = 1.2 * absrow + (absrow == 0)
    rhs = rng.standard_normal(n)
    return G.SymSystem.from_pairs(diag, pi, pj, pv, rhs)


def test_slice_layout_built():
    s = G.gen_poisson2d(33, 0).system
    g = G.build_graph(s)
    # slices of 32 rows, the last group of slices completed with padding slices
    assert (s.n + 31) // 32 <= g.info.num_slices < (s.n + 31) // 32 + 16
    assert g.info.num_slots >= g.num_edges


def test_slice_ragged_vs_tiles_and_oracle():
    s = _ragged_system()
    og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
    orc = oracle.solve(og, epsilon=1e-12, max_iter=200, schedule="broadcast")
    for mode in ("slice", "message", "recompute"):
        r = G.solve(s, G.SolveOptions(schedule="broadcast", epsilon=1e-12, max_iter=200,
                                      gather_mode=mode))
        assert r.iterations == orc.iterations, mode
        assert r.converged == orc.converged
        np.testing.assert_array_equal(r.means, orc.means)
        np.testing.assert_array_equal(r.precisions, orc.precisions)
        np.testing.assert_array_equal(np.asarray(r.max_change_history),
                                      np.asarray(orc.max_change_history))


def test_slice_needs_broadcast_and_layout():
    s = G.gen_poisson2d(8, 0).system
    with pytest.raises(ValueError):
        G.SolveOptions(schedule="serial", gather_mode="slice")
    # a hub longer than the slice limit: tiles only, auto still solves
    n = 5001
    pi = np.zeros(n - 1, dtype=np.int64)
    pj = np.arange(1, n, dtype=np.int64)
    pv = np.full(n - 1, 0.01)
    hub = G.SymSystem.from_pairs(np.full(n, 100.0), pi, pj, pv, np.ones(n))
    g = G.build_graph(hub)
    assert g.info.num_slices == 0
    with pytest.raises(_lib.GabpError):
        G.solve_graph(g, G.SolveOptions(schedule="broadcast", gather_mode="slice"))
    r = G.solve_graph(g, G.SolveOptions(schedule="broadcast", epsilon=1e-12))
    og = oracle.build_graph(hub.diag, hub.rhs, hub.pair_i, hub.pair_j, hub.pair_v)
    orc = oracle.solve(og, epsilon=1e-12, schedule="broadcast")
    assert r.iterations == orc.iterations
    np.testing.assert_array_equal(r.means, orc.means)
    del s


def test_slice_exact_relaunch_zero_rhs():
    """b = 0 on part of the rows makes 0 / A_ij divisions, which leave the fast division
    path: the fast slice launch flags itself and its exact twin redoes the sweep."""
    s = G.gen_poisson2d(40, 1).system
    rhs = s.rhs.copy()
    rhs[: s.n // 2] = 0.0
    s2 = G.SymSystem.from_pairs(s.diag, s.pair_i, s.pair_j, s.pair_v, rhs)
    og = oracle.build_graph(s2.diag, s2.rhs, s2.pair_i, s2.pair_j, s2.pair_v)
    orc = oracle.solve(og, epsilon=1e-10, max_iter=400, schedule="broadcast")
    r = G.solve(s2, G.SolveOptions(schedule="broadcast", epsilon=1e-10, max_iter=400,
                                   gather_mode="slice"))
    assert r.iterations == orc.iterations and r.converged == orc.converged
    np.testing.assert_array_equal(r.means, orc.means)
    np.testing.assert_array_equal(r.precisions, orc.precisions)
    np.testing.assert_array_equal(np.asarray(r.max_change_history),
                                  np.asarray(orc.max_change_history))


@pytest.mark.parametrize("variant", [0, 1, 2])
@pytest.mark.parametrize("which", ["ragged", "random64k", "poisson2d_200"])
def test_slice_kernel_variants_bitwise(variant, which, monkeypatch):
    """Every slice kernel (0 register batches, 1 cp.async ring, 2 TMA ring with dynamic
    work units) gives the oracle's bits; GABP_SLICE_VARIANT is read when the layout is
    built."""
    monkeypatch.setenv("GABP_SLICE_VARIANT", str(variant))
    if which == "ragged":
        s = _ragged_system()
    elif which == "random64k":
        s = G.gen_random_sparse(1 << 16, 16, 3).system
    else:
        s = G.gen_poisson2d(200, 4).system
    g = G.build_graph(s)
    assert int(g.info.slice_variant) == variant
    og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
    orc = oracle.solve(og, epsilon=1e-300, max_iter=60, schedule="broadcast",
                       rel_residual_tol=1e-8)
    r = G.solve_graph(g, G.SolveOptions(schedule="broadcast", epsilon=1e-300, max_iter=60,
                                        rel_residual_tol=1e-8, gather_mode="slice"))
    assert r.iterations == orc.iterations and r.converged == orc.converged
    np.testing.assert_array_equal(r.means, orc.means)
    np.testing.assert_array_equal(r.precisions, orc.precisions)
    np.testing.assert_array_equal(np.asarray(r.max_change_history),
                                  np.asarray(orc.max_change_history))


def test_skewed_degrees_fall_back_to_tiles():
    """One degree-3000 hub among degree-2 rows: padding every row of the hub's group to
    the hub's width would stream mostly padding, so the build keeps the CSR tiles; the
    solve still matches the oracle bitwise."""
    n = 20000
    pi = np.concatenate([np.zeros(3000, dtype=np.int64), np.arange(3001, n - 1)])
    pj = np.concatenate([np.arange(1, 3001), np.arange(3002, n)])
    pv = np.full(pi.size, 0.1)
    s = G.SymSystem.from_pairs(np.full(n, 400.0), pi, pj, pv, np.ones(n))
    g = G.build_graph(s)
    assert g.info.num_slices == 0
    og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
    orc = oracle.solve(og, epsilon=1e-12, schedule="broadcast")
    r = G.solve_graph(g, G.SolveOptions(schedule="broadcast", epsilon=1e-12))
    assert r.iterations == orc.iterations
    np.testing.assert_array_equal(r.means, orc.means)


def _degree_ladder_system(seed=11):
    """Stars of every degree class the warp-per-row kernel distinguishes (0, 1..32 in one
    register slot per lane, 33..64 in two, 65..256 through the strip rounds), hubs joined
    by a chain so the graph is connected, diagonally dominant."""
    rng = np.random.default_rng(seed)
    degs = [1, 2, 7, 8, 9, 31, 32, 33, 40, 63, 64, 65, 100, 128, 200, 255]
    pairs, nxt, hubs = {}, 0, []
    for d in degs:
        h = nxt
        hubs.append(h)
        for k in range(1, d + 1):
            pairs[(h, h + k)] = rng.uniform(-1, 1)
        nxt = h + d + 1
    for a, b in zip(hubs[:-1], hubs[1:]):
        pairs[(a + 1, b + 1)] = rng.uniform(-1, 1)
    n = nxt + 5  # trailing isolated nodes
    pi = np.array([p[0] for p in pairs], dtype=np.int64)
    pj = np.array([p[1] for p in pairs], dtype=np.int64)
    pv = np.array(list(pairs.values()))
    absrow = np.zeros(n)
    np.add.at(absrow, pi, np.abs(pv))
    np.add.at(absrow, pj, np.abs(pv))
    diag = 1.3 * absrow + (absrow == 0)
    return G.SymSystem.from_pairs(diag, pi, pj, pv, rng.standard_normal(n))


@pytest.mark.parametrize("sweep_cap", [1, 2, 3, 5, 60])
def test_parallel_rows_kernel_degree_ladder(sweep_cap):
    """Warp-per-row parallel kernel (rowpar.cu) on every degree class, stopped after each
    of the first sweeps (messages, change history, marginals of every launch kind) and at
    convergence: bitwise equal to the oracle."""
    s = _degree_ladder_system()
    og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
    orc = oracle.solve(og, epsilon=1e-12, max_iter=sweep_cap, schedule="parallel")
    r = G.solve(s, G.SolveOptions(schedule="parallel", epsilon=1e-12, max_iter=sweep_cap,
                                  gather_mode="rows"))
    assert r.iterations == orc.iterations and r.converged == orc.converged
    np.testing.assert_array_equal(r.means, orc.means)
    np.testing.assert_array_equal(r.precisions, orc.precisions)
    np.testing.assert_array_equal(np.asarray(r.max_change_history),
                                  np.asarray(orc.max_change_history))


def test_parallel_rows_kernel_rejects_long_rows():
    n = 400
    pi = np.zeros(300, dtype=np.int64)
    pj = np.arange(1, 301)
    s = G.SymSystem.from_pairs(np.full(n, 100.0), pi, pj, np.full(300, 0.1), np.ones(n))
    with pytest.raises(Exception):
        G.solve(s, G.SolveOptions(schedule="parallel", gather_mode="rows"))


@pytest.mark.parametrize("which", ["ragged", "random64k", "poisson2d_200", "golden"])
def test_parallel_schedule_slice_kernel_bitwise(which):
    """The parallel schedule on the slice groups (exclusion sums over the contiguous
    incoming slots, scattered twin stores) against the oracle and the tile kernel."""
    if which == "ragged":
        systems = [_ragged_system()]
    elif which == "random64k":
        systems = [G.gen_random_sparse(1 << 16, 16, 3).system]
    elif which == "poisson2d_200":
        systems = [G.gen_poisson2d(200, 4).system]
    else:
        systems = [gc.system(gc.load(c)) for c in CASES]
    for s in systems:
        og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
        orc = oracle.solve(og, epsilon=1e-300, max_iter=80, schedule="parallel",
                           rel_residual_tol=1e-8)
        g = G.build_graph(s)
        for mode in ("slice", "message", "rows"):
            if mode == "slice" and int(g.info.num_slices) == 0:
                continue
            if mode == "rows" and int(g.info.max_degree) > 256:
                continue
            r = G.solve_graph(g, G.SolveOptions(schedule="parallel", epsilon=1e-300,
                                                max_iter=80, rel_residual_tol=1e-8,
                                                gather_mode=mode))
            assert r.iterations == orc.iterations and r.converged == orc.converged, mode
            assert r.diverged == orc.diverged
            np.testing.assert_array_equal(r.means, orc.means)
            np.testing.assert_array_equal(r.precisions, orc.precisions)
            np.testing.assert_array_equal(np.asarray(r.max_change_history),
                                          np.asarray(orc.max_change_history))


# ---------------------------------------------------------------------------------------
# serial schedule (solver.py:176-217) as dependency levels (rowpar.cu serial_level_kernel)
# ---------------------------------------------------------------------------------------

@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("tag", ["asc", "custom"])
def test_serial_sweep_trace_vs_reference(case, tag):
    """Device serial sweeps (ascending order, and a custom order with a repeated and a
    missing node) bitwise equal to the reference's own in-place loop."""
    rec = gc.load(case)
    srec = gc.load_serial(case)
    g = G.build_graph(gc.system(rec))
    order = None if tag == "asc" else [int(v) for v in srec["order"]]
    opts = G.SolveOptions(schedule="serial", serial_order=order)
    st = G.initial_state(g, "serial")
    want_p, want_m = srec[f"{tag}_trace_prec"], srec[f"{tag}_trace_mean"]
    want_c = srec[f"{tag}_trace_change"]
    for t in range(want_p.shape[0]):
        st, mc = G.sweep(g, st, opts)
        np.testing.assert_array_equal(st.prec, want_p[t])
        np.testing.assert_array_equal(st.mean, want_m[t])
        assert mc == want_c[t]
    if int(srec[f"{tag}_trace_singular_at"]) > 0:
        with pytest.raises(G.SingularSubgraphError):
            G.sweep(g, st, opts)


@pytest.mark.parametrize("case", CASES)
def test_serial_solve_vs_reference(case):
    rec = gc.load(case)
    srec = gc.load_serial(case)
    tol = float(rec["rel_residual_tol"]) or None
    r = G.solve(gc.system(rec), G.SolveOptions(schedule="serial", epsilon=float(rec["epsilon"]),
                                               max_iter=int(rec["max_iter"]),
                                               rel_residual_tol=tol))
    assert r.converged == bool(srec["serial_converged"])
    assert r.diverged == bool(srec["serial_diverged"])
    assert r.iterations == int(srec["serial_iterations"])
    want = srec["serial_means"]
    fin = np.isfinite(want)
    np.testing.assert_array_equal(np.isfinite(r.means), fin)
    np.testing.assert_array_equal(r.means[fin], want[fin])
    np.testing.assert_array_equal(r.precisions, srec["serial_precisions"])
    np.testing.assert_array_equal(np.asarray(r.max_change_history), srec["serial_change_hist"])
    rh = srec["serial_res_hist"]
    atol = 1e-12 * float(np.max(rh[np.isfinite(rh)], initial=0.0))
    np.testing.assert_allclose(np.asarray(r.residual_history), rh, rtol=1e-9, atol=atol)


@pytest.mark.parametrize("which", ["random64k", "poisson2d_200", "ladder", "ragged"])
def test_serial_large_vs_oracle(which):
    """Many dependency levels and wide levels: device serial solve (ascending and a seeded
    random order) bitwise equal to the sequential C oracle."""
    if which == "random64k":
        s = G.gen_random_sparse(1 << 16, 16, 3).system
    elif which == "poisson2d_200":
        s = G.gen_poisson2d(200, 4).system
    elif which == "ladder":
        s = _degree_ladder_system()
    else:
        s = _ragged_system()
    og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
    rng = np.random.default_rng(7)
    for order in (None, [int(v) for v in rng.permutation(s.n)]):
        orc = oracle.solve_serial(og, epsilon=1e-300, max_iter=12, order=order,
                                  rel_residual_tol=1e-10)
        r = G.solve(s, G.SolveOptions(schedule="serial", epsilon=1e-300, max_iter=12,
                                      serial_order=order, rel_residual_tol=1e-10))
        assert r.iterations == orc.iterations and r.converged == orc.converged
        np.testing.assert_array_equal(r.means, orc.means)
        np.testing.assert_array_equal(r.precisions, orc.precisions)
        np.testing.assert_array_equal(np.asarray(r.max_change_history),
                                      orc.max_change_history)


def test_serial_order_errors():
    s = G.gen_poisson2d(8, 0).system
    with pytest.raises(Exception):
        G.solve(s, G.SolveOptions(schedule="serial", serial_order=[0, 1, s.n]))


@pytest.mark.parametrize("which", ["ladder", "poisson2d_200"])
def test_serial_level_launch_path_vs_oracle(which, monkeypatch):
    """The per-level launch path (CUDA graph of level launches, GABP_SERIAL_LEVEL_LAUNCHES)
    gives the same bits as the cooperative one-launch sweep and the oracle."""
    s = _degree_ladder_system() if which == "ladder" else G.gen_poisson2d(200, 4).system
    og = oracle.build_graph(s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)
    orc = oracle.solve_serial(og, epsilon=1e-300, max_iter=6)
    monkeypatch.setenv("GABP_SERIAL_LEVEL_LAUNCHES", "1")
    r = G.solve(s, G.SolveOptions(schedule="serial", epsilon=1e-300, max_iter=6))
    assert r.iterations == orc.iterations
    np.testing.assert_array_equal(r.means, orc.means)
    np.testing.assert_array_equal(np.asarray(r.max_change_history), orc.max_change_history)
