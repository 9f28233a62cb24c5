"""Host logic of the Signal Tracing Bank's aperture partition, CPU only."""
import numpy as np
import pytest

from paper_2605_29097_b200.training import AperturePatches


@pytest.mark.parametrize("n_u,n_v,pu,pv", [(8, 8, 4, 4), (8, 8, 8, 8), (7, 5, 3, 2), (128, 128, 40, 80)])
def test_patches_partition_the_aperture(n_u, n_v, pu, pv):
    P = AperturePatches(n_u, n_v, pu, pv)
    perm = P.perm.numpy()
    assert sorted(perm.tolist()) == list(range(n_u * n_v))              # every antenna once
    assert P.bounds[0][0] == 0 and P.bounds[-1][1] == n_u * n_v
    assert all(P.bounds[i][1] == P.bounds[i + 1][0] for i in range(P.n_patches - 1))
    for lo, hi in P.bounds:                                              # each patch is a grid box
        u, v = perm[lo:hi] // n_v, perm[lo:hi] % n_v
        assert (u.max() - u.min() + 1) * (v.max() - v.min() + 1) == hi - lo
        assert u.max() - u.min() < pu and v.max() - v.min() < pv


def test_single_patch_is_identity_order():
    P = AperturePatches(8, 8, 8, 8)
    assert P.n_patches == 1 and np.array_equal(P.perm.numpy(), np.arange(64))


def test_paper_patch_size_3200():
    """Baseline patch of 3200 antennas on a 128 x 128 aperture: 40 x 80 boxes."""
    P = AperturePatches(128, 128, 40, 80)
    assert max(hi - lo for lo, hi in P.bounds) == 3200
