"""A/B of the residual probe: device time and launches of full solves to 1e-8 with and
without it (GABP_NO_PROBE=1 in a second process).
Usage: GABP_HOST_TIMING=1 python tools/probe_ab.py --config 1 [--reps 5]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0810_1119_b200 as G  # noqa: E402
from paper_0810_1119_b200 import problems  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--schedule", default="broadcast")
a = ap.parse_args()
name, fn = problems.CONFIGS[a.config]
s = fn(0).system
g = G.build_graph(s, 0)
opts = G.SolveOptions(schedule=a.schedule, epsilon=1e-300, rel_residual_tol=1e-8, device=0,
                      record_means_history=False)
ms = []
for _ in range(a.reps + 1):
    r = G.solve_graph(g, opts)
    ms.append(r.device_ms)
print(f"{name} {a.schedule} probe={'off' if os.environ.get('GABP_NO_PROBE') else 'on'}: "
      f"{r.iterations} sweeps, launched {r.sweeps_launched}, probes {r.residual_probes}, "
      f"kernels {r.kernel_launches}, device ms "
      f"{' '.join(f'{m:.3f}' for m in ms[1:])}", flush=True)
