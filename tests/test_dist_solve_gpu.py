"""The torch.distributed entry point (DistributedGraph / solve_distributed) on one GPU:
world_size 1 under the gloo-free single-rank path, result bitwise equal to solve()."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_solve_distributed_single_rank():
    import torch
    import torch.distributed as dist

    import paper_0810_1119_b200 as G
    from paper_0810_1119_b200 import dist as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        s = G.gen_poisson2d(48, 1).system
        opts = G.SolveOptions(schedule="broadcast", epsilon=1e-300, rel_residual_tol=1e-9,
                              max_iter=5000, device=0)
        one = G.solve(s, opts)
        r = D.solve_distributed(s, opts)
        assert r.iterations == one.iterations
        np.testing.assert_array_equal(r.means, one.means)
        dg = D.DistributedGraph(s, device=0)
        r2 = dg.solve(opts)
        r3 = dg.solve(opts)   # repeated solves on one build
        dg.close()
        np.testing.assert_array_equal(r2.means, one.means)
        np.testing.assert_array_equal(r3.means, one.means)
    finally:
        dist.destroy_process_group()
