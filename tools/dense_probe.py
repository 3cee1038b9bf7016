"""Short dense (config 3) solve for ncu launch lists."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0810_1119_b200 as G
inst, _ = G.gen_cdma_detection(8192, 4096, 0.5, 0)
g = G.build_graph(inst.system, 0)
r = G.solve_graph(g, G.SolveOptions(schedule="broadcast", epsilon=1e-300, max_iter=6,
                                    record_means_history=False))
print("dense", g.info.is_dense, "iters", r.iterations, "ms", r.device_ms)
