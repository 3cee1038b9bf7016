"""Parallel-schedule probe: back-to-back sweep time per gather mode (device events,
gabp_bench_sweeps) and one full solve per mode, on a BASELINE config.
Usage: python tools/par_probe.py --config 1 [--modes slice,rows,message] [--sweeps 20]"""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0810_1119_b200 as G  # noqa: E402
from paper_0810_1119_b200 import _lib, problems  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--modes", default="slice,rows,message")
ap.add_argument("--sweeps", type=int, default=20)
ap.add_argument("--solve", type=int, default=1)
a = ap.parse_args()
name, fn = problems.CONFIGS[a.config]
s = fn(0).system
g = G.build_graph(s, 0)
lib = _lib.load()
E, n = int(g.info.num_edges), int(g.info.n)
alg = 48.0 * E + 52.0 * n  # algorithmic bytes of one sweep
ref = None
for mode in a.modes.split(","):
    ms = ctypes.c_double()
    gid = _lib.GATHER_IDS[mode]
    _lib.check(lib.gabp_bench_sweeps(g.handle, 0, gid, 3, ctypes.byref(ms)))
    _lib.check(lib.gabp_bench_sweeps(g.handle, 0, gid, a.sweeps, ctypes.byref(ms)))
    line = {"config": a.config, "workload": name, "mode": mode, "ms_per_sweep": ms.value,
            "edge_updates_per_s": E / (ms.value * 1e-3),
            "alg_GBps": alg / (ms.value * 1e-3) / 1e9}
    if a.solve:
        opts = G.SolveOptions(schedule="parallel", epsilon=1e-300, rel_residual_tol=1e-8,
                              max_iter=400, gather_mode=mode, record_means_history=False)
        G.solve_graph(g, opts)
        r = G.solve_graph(g, opts)
        line.update({"solve_ms": r.device_ms, "iterations": r.iterations})
        if ref is None:
            ref = r
        else:
            line["bitwise_vs_first"] = bool(
                r.iterations == ref.iterations and (r.means.view("u8") == ref.means.view("u8")).all()
                and (r.precisions.view("u8") == ref.precisions.view("u8")).all())
    print(json.dumps(line), flush=True)
