"""Config 3 (dense CDMA, K = 4096): capped solves through the fused one-kernel sweep and the
two-kernel sweep (GABP_DENSE_TWO_KERNELS=1); ms per launch.  Usage: python tools/dense_fused_probe.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0810_1119_b200 as G  # noqa: E402
from paper_0810_1119_b200 import problems as P  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
s = G.gen_cdma_detection(2 * K, K, 0.5, 0)[0].system
g = G.build_graph(s, 0)
o = G.SolveOptions(schedule="broadcast", epsilon=1e-300, max_iter=20, device=0,
                   record_means_history=False)
out = {"K": K, "directed_edges": g.num_edges}
algo = 48 * g.num_edges + 52 * g.n
for label, env in (("fused", None), ("two_kernels", "1")):
    if env:
        os.environ["GABP_DENSE_TWO_KERNELS"] = env
    else:
        os.environ.pop("GABP_DENSE_TWO_KERNELS", None)
    G.solve_graph(g, o)
    r = min((G.solve_graph(g, o) for _ in range(3)), key=lambda r: r.device_ms)
    ms = r.device_ms / max(r.sweeps_launched, 1)
    out[label] = {"ms_per_launch": round(ms, 4), "launches": int(r.sweeps_launched),
                  "iterations": int(r.iterations), "frac_6545": round(algo / ms / 1e6 / 6545, 3)}
g.close()
print(json.dumps(out))
