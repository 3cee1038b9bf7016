"""Parallel schedule on a Poisson grid: the diagonal-layout kernel (dia_par_kernel) against
the slice-group kernel (GABP_NO_DIA_PAR=1).  Usage: python tools/dia_par_probe.py [--dims 2
--p 4096 --sweeps 30]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0810_1119_b200 as G  # noqa: E402
from paper_0810_1119_b200 import grid as GR  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dims", type=int, default=2)
ap.add_argument("--p", type=int, default=4096)
ap.add_argument("--sweeps", type=int, default=30)
a = ap.parse_args()
g = GR.GridGraph(GR.GridSpec(a.dims, a.p, 0), 0)
opts = G.SolveOptions(schedule="parallel", epsilon=1e-300, max_iter=a.sweeps, device=0,
                      record_means_history=False)
out = {"grid": f"poisson{a.dims}d-{a.p}", "n": g.n, "directed_edges": g.num_edges}
for label, env in (("dia_par", None), ("slice_par", "1")):
    if env:
        os.environ["GABP_NO_DIA_PAR"] = env
    else:
        os.environ.pop("GABP_NO_DIA_PAR", None)
    G.solve_graph(g, opts)
    r = min((G.solve_graph(g, opts) for _ in range(2)), key=lambda r: r.device_ms)
    ms = r.device_ms / max(r.sweeps_launched, 1)
    algo = 48 * g.num_edges + 52 * g.n
    out[label] = {"ms_per_launch": round(ms, 4), "launches": int(r.sweeps_launched),
                  "alg_GBps": round(algo / ms / 1e6, 1)}
g.close()
print(json.dumps(out))
