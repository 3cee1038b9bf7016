"""Host-clock breakdown of the e2e drop-in call on config 1: graph create (H2D + device
build), first solve (workspace allocation + CUDA-graph capture), destroy; then the fused
gabp_solve_system.  Usage: python tools/e2e_breakdown.py [--config 1] [--reps 3]"""
import argparse
import ctypes
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_0810_1119_b200 import _lib, problems  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
s = problems.CONFIGS[a.config][1](0).system
lib = _lib.load()
keep = [bench.pinned_copy(x) for x in (s.diag, s.rhs, s.pair_i, s.pair_j, s.pair_v)]
hd, hr, hi, hj, hv = (k[1] for k in keep)
n = s.n
o = _lib.Options()
o.epsilon = 1e-300
o.max_iter = 10000
o.blowup = 1e10
o.schedule = 2
o.rel_residual_tol = 1e-8
means = bench.pinned_copy(np.empty(n))[1]
ch = np.empty(o.max_iter)
rh = np.empty(o.max_iter)
rep = _lib.Report()
for r in range(a.reps):
    t0 = time.perf_counter()
    h = ctypes.c_void_p()
    _lib.check(lib.gabp_graph_create(n, s.pair_v.size, _lib.ptr(hd), _lib.ptr(hr), _lib.ptr(hi),
                                     _lib.ptr(hj), _lib.ptr(hv), 0, ctypes.byref(h)))
    t1 = time.perf_counter()
    info = _lib.GraphInfo()
    _lib.check(lib.gabp_graph_info(h, ctypes.byref(info)))
    _lib.check(lib.gabp_solve(h, ctypes.byref(o), _lib.ptr(means), None, _lib.ptr(ch),
                              _lib.ptr(rh), ctypes.byref(rep)))
    t2 = time.perf_counter()
    _lib.check(lib.gabp_solve(h, ctypes.byref(o), _lib.ptr(means), None, _lib.ptr(ch),
                              _lib.ptr(rh), ctypes.byref(rep)))
    t3 = time.perf_counter()
    lib.gabp_graph_destroy(h)
    t4 = time.perf_counter()
    _lib.check(lib.gabp_solve_system(n, s.pair_v.size, _lib.ptr(hd), _lib.ptr(hr), _lib.ptr(hi),
                                     _lib.ptr(hj), _lib.ptr(hv), 0, ctypes.byref(o),
                                     _lib.ptr(means), None, _lib.ptr(ch), _lib.ptr(rh),
                                     ctypes.byref(rep)))
    t5 = time.perf_counter()
    print(f"rep {r}: create {1e3*(t1-t0):.1f} ms (device build {info.build_ms:.1f}), "
          f"solve#1 {1e3*(t2-t1):.1f} ms (device {rep.device_ms:.2f}), solve#2 {1e3*(t3-t2):.1f} ms, "
          f"destroy {1e3*(t4-t3):.1f} ms | solve_system {1e3*(t5-t4):.1f} ms")

# the bench's sequence: torch context, a resident graph solved then closed, then e2e calls
import torch  # noqa: E402
import paper_0810_1119_b200 as G  # noqa: E402

torch.cuda.synchronize(0)
g = G.build_graph(s, 0)
_lib.check(lib.gabp_solve_device(g.handle, ctypes.byref(o), None, None, ctypes.byref(rep)))
g.close()
for r in range(5):
    t0 = time.perf_counter()
    _lib.check(lib.gabp_solve_system(n, s.pair_v.size, _lib.ptr(hd), _lib.ptr(hr), _lib.ptr(hi),
                                     _lib.ptr(hj), _lib.ptr(hv), 0, ctypes.byref(o),
                                     _lib.ptr(means), None, _lib.ptr(ch), _lib.ptr(rh),
                                     ctypes.byref(rep)))
    print(f"after torch + resident graph: solve_system {1e3*(time.perf_counter()-t0):.1f} ms")
