"""Run a few sweep-kernel launches of one config for ncu (no timing is reported from
profiled runs).  Usage: python tools/profile_sweep.py --config 1 --sweeps 4"""

import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_0810_1119_b200 as G  # noqa: E402
from paper_0810_1119_b200 import _lib, problems  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--schedule", default="broadcast")
ap.add_argument("--sweeps", type=int, default=4)
ap.add_argument("--gather", default="auto", choices=["auto", "message", "recompute", "slice"])
ap.add_argument("--solve", action="store_true", help="also run one full solve")
args = ap.parse_args()

name, fn = problems.CONFIGS[args.config]
system = fn(0).system
g = G.build_graph(system, 0)
ms = ctypes.c_double()
_lib.check(_lib.load().gabp_bench_sweeps(g.handle, _lib.SCHED_IDS[args.schedule],
                                          _lib.GATHER_IDS[args.gather], args.sweeps,
                                          ctypes.byref(ms)))
print(f"{name} [{args.schedule}/{args.gather}, twin_span {g.info.twin_span:.0f}]: "
      f"{args.sweeps} sweeps, {ms.value:.3f} ms/sweep (unprofiled number only if not under ncu)")
if args.solve:
    r = G.solve_graph(g, G.SolveOptions(schedule=args.schedule, epsilon=1e-300,
                                        rel_residual_tol=1e-8, record_means_history=False,
                                        gather_mode=args.gather))
    print("solve", r.iterations, r.converged, r.device_ms)
