"""Steady-state sweep time of a device-generated Poisson grid (grid.py) through
gabp_bench_sweeps: auto mode (diagonal layout when the graph is a stencil) or a forced mode.
Usage: python tools/grid_probe.py --dims 2 --p 4096 [--mode auto|slice] [--sweeps 20]"""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0810_1119_b200 import _lib, grid as GR  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dims", type=int, default=2)
ap.add_argument("--p", type=int, default=4096)
ap.add_argument("--mode", default="auto")
ap.add_argument("--sweeps", type=int, default=20)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
spec = GR.GridSpec(a.dims, a.p, 0)
g = GR.GridGraph(spec, 0)
lib = _lib.load()
ms = ctypes.c_double()
mode = _lib.GATHER_IDS[a.mode]
out = []
for _ in range(a.reps):
    _lib.check(lib.gabp_bench_sweeps(g.handle, 2, mode, a.sweeps, ctypes.byref(ms)))
    out.append(ms.value)
E, n = g.num_edges, g.n
try:
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0)
except OSError:  # (driver-written per pod; absent: the profiling recipe's fallback)
    peak = 6650.0
best = min(out)
print(json.dumps({"grid": spec.name, "mode": a.mode, "dia": int(g.info.dia_diagonals),
                  "ms": [round(v, 4) for v in out],
                  "frac": (48 * E + 52 * n) / (best / 1e3) / 1e9 / peak}))
