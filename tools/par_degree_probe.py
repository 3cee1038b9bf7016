"""Parallel schedule on random graphs of different mean degree: slice-group kernel against
the four-rows-per-warp kernel (gather mode rows).  Usage: python tools/par_degree_probe.py"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0810_1119_b200 as G  # noqa: E402
from paper_0810_1119_b200 import _lib  # noqa: E402

lib = _lib.load()
for k in (2, 4, 6, 8, 12):
    s = G.gen_random_sparse(1 << 19, k, 3).system
    g = G.build_graph(s, 0)
    out = {"k": k, "mean_degree": round(g.num_edges / g.n, 1)}
    for mode, mid in (("slice", 3), ("rows", 4)):
        ms = ctypes.c_double()
        try:
            _lib.check(lib.gabp_bench_sweeps(g.handle, 0, mid, 5, ctypes.byref(ms)))
            _lib.check(lib.gabp_bench_sweeps(g.handle, 0, mid, 20, ctypes.byref(ms)))
            out[mode] = round(ms.value, 4)
        except Exception as e:  # noqa: BLE001
            out[mode] = str(e)[:60]
    g.close()
    print(json.dumps(out), flush=True)
