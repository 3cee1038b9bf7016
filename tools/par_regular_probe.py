"""How much of the four-rows-per-warp kernel's time is SIMD padding: the parallel sweep on a
near-regular random graph (every row 31-32 edges: unions of random permutations) against
BASELINE config 1 (same size, degrees 16 + Poisson-like).  Usage: python tools/par_regular_probe.py"""
import ctypes
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0810_1119_b200 as G  # noqa: E402
from paper_0810_1119_b200 import _lib  # noqa: E402

lib = _lib.load()
n, k = 1 << 20, 16
rng = np.random.default_rng(1)
pi = np.tile(np.arange(n, dtype=np.int64), k)
pj = np.concatenate([rng.permutation(n) for _ in range(k)]).astype(np.int64)
keep = pi != pj
lo, hi = np.minimum(pi[keep], pj[keep]), np.maximum(pi[keep], pj[keep])
key = np.unique(lo * n + hi)
pi, pj = key // n, key % n
pv = rng.uniform(-1.0, 1.0, pi.size)
pv[pv == 0.0] = 0.25
absrow = np.bincount(pi, np.abs(pv), n) + np.bincount(pj, np.abs(pv), n)
s = G.SymSystem.from_pairs(1.1 * absrow, pi, pj, pv, rng.standard_normal(n), validate=False)
c1 = G.gen_random_sparse(n, k, 0).system
# config 1 relabelled by degree (rows of equal block count next to each other): the same
# work, no padding inside a quad -- the most a row permutation in the load stage could win
deg1 = np.bincount(np.concatenate([c1.pair_i, c1.pair_j]), minlength=n)
rank = np.empty(n, dtype=np.int64)
rank[np.argsort(-deg1, kind="stable")] = np.arange(n)
ri, rj = rank[c1.pair_i], rank[c1.pair_j]
inv = np.argsort(rank)
c1s = G.SymSystem.from_pairs(c1.diag[inv], np.minimum(ri, rj), np.maximum(ri, rj), c1.pair_v,
                             c1.rhs[inv], validate=False)
for name, sysm in (("regular-32", s), ("config 1", c1), ("config 1 by degree", c1s)):
    g = G.build_graph(sysm, 0)
    deg = np.bincount(np.concatenate([sysm.pair_i, sysm.pair_j]), minlength=n)
    ms = ctypes.c_double()
    _lib.check(lib.gabp_bench_sweeps(g.handle, 0, 4, 3, ctypes.byref(ms)))
    _lib.check(lib.gabp_bench_sweeps(g.handle, 0, 4, 20, ctypes.byref(ms)))
    E = int(g.info.num_edges)
    print(json.dumps({"graph": name, "directed_edges": E, "deg_min": int(deg.min()),
                      "deg_max": int(deg.max()), "ms_per_sweep": round(ms.value, 4),
                      "ns_per_kilo_edge": round(ms.value * 1e6 / (E / 1e3), 3)}), flush=True)
    g.close()
