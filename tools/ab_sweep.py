"""A/B timing of sweep-kernel builds: each library (GABP_LIB path) in its own process,
alternating, back-to-back steady-state sweeps (gabp_bench_sweeps, CUDA events) on one
config.  Usage: python tools/ab_sweep.py --config 1 --libs lib/a.so lib/b.so [--rounds 3]"""
import argparse
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)

CHILD = r"""
import ctypes, json, os, sys, time
sys.path.insert(0, %r)
import paper_0810_1119_b200 as G
from paper_0810_1119_b200 import _lib, problems
name, fn = problems.CONFIGS[%d]
s = fn(0).system
g = G.build_graph(s, 0)
lib = _lib.load()
ms = ctypes.c_double()
out = []
_lib.check(lib.gabp_bench_sweeps(g.handle, %d, 0, 5, ctypes.byref(ms)))
for _ in range(%d):
    _lib.check(lib.gabp_bench_sweeps(g.handle, %d, 0, %d, ctypes.byref(ms)))
    out.append(ms.value)
E, n = g.num_edges, g.n
print(json.dumps({"lib": os.environ.get("GABP_LIB", "default"), "ms": out, "E": E, "n": n}))
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--libs", nargs="+", required=True)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--sweeps", type=int, default=50)
    ap.add_argument("--schedule", type=int, default=2)
    a = ap.parse_args()
    try:
        peak = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0)
    except OSError:  # (driver-written per pod; absent: the profiling recipe's fallback)
        peak = 6650.0
    res = {}
    for _ in range(a.rounds):
        for lib in a.libs:
            env = dict(os.environ, GABP_LIB=os.path.abspath(lib))
            code = CHILD % (REPO, a.config, a.schedule, a.reps, a.schedule, a.sweeps)
            p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True,
                               text=True)
            if p.returncode:
                print(p.stderr[-2000:], file=sys.stderr)
                continue
            d = json.loads(p.stdout.strip().splitlines()[-1])
            res.setdefault(lib, []).extend(d["ms"])
            E, n = d["E"], d["n"]
    for lib, ms in res.items():
        best = min(ms)
        algo = 48 * E + 52 * n
        print(json.dumps({"lib": lib, "config": a.config, "ms_best": round(best, 4),
                          "ms_median": round(sorted(ms)[len(ms) // 2], 4),
                          "frac_best": round(algo / (best / 1e3) / 1e9 / peak, 4)}))


if __name__ == "__main__":
    main()
