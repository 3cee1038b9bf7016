"""Config 3 (dense CDMA detection, K=4096) through the public solve: convergence and time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_0810_1119_b200 as G
t0 = time.time()
inst, s_true = G.gen_cdma_detection(8192, 4096, 0.5, 0)
print(f"generated in {time.time()-t0:.1f}s, pairs {inst.system.pair_v.size}")
g = G.build_graph(inst.system, 0)
print("graph", g.info.num_edges, "tiles", g.info.num_tiles, "build ms", g.info.build_ms)
for mode in ("auto", "message", "recompute"):
    opts = G.SolveOptions(schedule="broadcast", epsilon=1e-300, rel_residual_tol=1e-8,
                          max_iter=500, record_means_history=False, gather_mode=mode)
    r = G.solve_graph(g, opts)
    print(mode, "conv", r.converged, "iters", r.iterations, "ms", round(r.device_ms, 2),
          "ms/sweep", round(r.device_ms / max(r.sweeps_launched, 1), 3),
          "rel", r.final_rel_residual, "res_hist tail", r.residual_history[-3:])
a, b = inst.system.to_dense()
x = np.linalg.solve(a, b)
print("decisions agree with the decorrelator:", np.array_equal(np.sign(r.means), np.sign(x)),
      "bit errors vs s:", int(np.sum(np.sign(r.means) != s_true)))
