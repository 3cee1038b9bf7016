"""Device grid generator (grid.py), host-side: the slab parts it forms equal the host
partitioner's (dist.local_part) on the same grid -- pairs, priors, owned range and halo
lists -- so the device-built partitions are the partitions the parity tests check."""

import numpy as np
import pytest

from paper_0810_1119_b200 import dist as D
from paper_0810_1119_b200 import grid as GR
from paper_0810_1119_b200 import problems as P


@pytest.mark.parametrize("dims,p,world", [(2, 16, 1), (2, 16, 4), (2, 9, 3), (3, 8, 1),
                                          (3, 8, 2), (3, 8, 8), (3, 6, 4)])
def test_grid_part_equals_host_partition(dims, p, world):
    spec = GR.GridSpec(dims, p, 0)
    s = (P.gen_poisson2d if dims == 2 else P.gen_poisson3d)(p, 0).system
    bounds = GR.slab_bounds(spec, world)
    assert bounds[0] == 0 and bounds[-1] == spec.n
    assert np.all(np.diff(bounds) % spec.plane == 0)
    rhs = GR.rhs_device(spec, -1)
    total = 0
    for r in range(world):
        gp = GR.grid_part(spec, world, r, -1, rhs)
        lp = D.local_part(s, bounds, r)
        assert (gp.n_local, gp.row_lo, gp.row_hi) == (lp.n_local, lp.row_lo, lp.row_hi)
        got = set(zip(gp.pair_i.numpy().tolist(), gp.pair_j.numpy().tolist()))
        want = set(zip(lp.pair_i.tolist(), lp.pair_j.tolist()))
        assert got == want
        assert len(got) == gp.npairs  # no duplicates
        assert np.all(gp.pair_v.numpy() == -1.0)
        np.testing.assert_array_equal(gp.diag.numpy(), lp.diag)
        np.testing.assert_array_equal(gp.rhs.numpy()[gp.row_lo:gp.row_hi],
                                      rhs.numpy()[gp.lo:gp.hi])
        assert gp.peers == lp.peers
        for q in gp.peers:
            np.testing.assert_array_equal(gp.send_idx[q], lp.send_idx[q])
            np.testing.assert_array_equal(gp.recv_idx[q], lp.recv_idx[q])
        assert gp.halo_bytes_per_sweep() == D.halo_bytes_per_sweep(lp)
        total += gp.hi - gp.lo
    assert total == spec.n
    whole = GR.grid_part(spec, 1, 0, -1, rhs)
    assert whole.npairs == spec.npairs == s.pair_v.size


def test_grid_spec_rejects():
    with pytest.raises(ValueError):
        GR.GridSpec(4, 8)
    with pytest.raises(ValueError):
        GR.slab_bounds(GR.GridSpec(2, 4), 5)
