import sys; sys.path.insert(0,'.')
import paper_0810_1119_b200 as G
s = G.gen_poisson2d(32, 0).system
g = G.build_graph(s, 0)
for sched in ("broadcast","parallel"):
    opts = G.SolveOptions(schedule=sched, epsilon=1e-300, rel_residual_tol=1e-8, device=0, record_means_history=False)
    for _ in range(2):
        r = G.solve_graph(g, opts)
    print(sched, r.iterations, f"{r.device_ms:.3f} ms {1e3*r.device_ms/r.iterations:.2f} us/sweep launches {r.kernel_launches}")
