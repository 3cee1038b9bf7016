"""Serial-schedule probe: dependency levels of the ascending order and wall time per
device sweep (gabp_sweep_serial) on a BASELINE config.
Usage: python tools/serial_probe.py --config 1 [--sweeps 3]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0810_1119_b200 as G  # noqa: E402
from paper_0810_1119_b200 import problems, solver  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--sweeps", type=int, default=3)
a = ap.parse_args()
name, fn = problems.CONFIGS[a.config]
s = fn(0).system
g = G.build_graph(s, 0)
st = G.initial_state(g, "serial")
order = solver._order_arg(None)
t0 = time.perf_counter()
_, _, levels = solver._serial_inplace(g, st, order, 1e10)  # builds the level schedule
t_first = time.perf_counter() - t0
t0 = time.perf_counter()
for _ in range(a.sweeps):
    solver._serial_inplace(g, st, order, 1e10)
dt = (time.perf_counter() - t0) / a.sweeps
E = int(g.info.num_edges)
print(json.dumps({"config": a.config, "workload": name, "schedule": "serial (ascending)",
                  "levels": levels, "first_sweep_s_incl_level_build": t_first,
                  "ms_per_sweep": dt * 1e3, "edge_updates_per_s": E / dt}))
