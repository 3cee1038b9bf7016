"""Config 0 (Poisson 32^2) solved to 1e-8 through the one-CTA kernel: device time per sweep.
Usage: python tools/small_probe.py [--reps 3]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0810_1119_b200 as G  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--p", type=int, default=32)
a = ap.parse_args()
s = G.gen_poisson2d(a.p, 0).system
g = G.build_graph(s, 0)
opts = G.SolveOptions(schedule="broadcast", epsilon=1e-300, rel_residual_tol=1e-8, device=0,
                      record_means_history=False)
for _ in range(a.reps):
    r = G.solve_graph(g, opts)
    print(f"poisson2d-{a.p}: {r.iterations} sweeps, {r.device_ms:.3f} ms, "
          f"{1e3 * r.device_ms / r.iterations:.2f} us/sweep, launches {r.kernel_launches}",
          flush=True)
