"""Device versions of the public building blocks against the reference's own
values (tests/golden/functions.npz from chebyshev.py / kernels.py)."""

import os

import numpy as np
import pytest

import paper_2508_05958_b200 as H

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def g():
    return np.load(os.path.join(GOLD, "functions.npz"))


@pytest.mark.parametrize("p", [1, 2, 3, 6, 8])
def test_cheb_points_and_factor_matrix(p):
    grid = H.cheb_points(0.25, 0.75, p)
    ref = g()[f"cheb_{p}"]
    assert np.abs(grid.nodes - ref).max() <= 2e-16
    fac = H.factor_matrix(g()[f"fac_pts_{p}"], grid)
    assert np.abs(fac - g()[f"fac_{p}"]).max() <= 1e-14
    with pytest.raises(ValueError):
        H.factor_matrix([0.0], grid)


def test_core_tensors():
    nt = [H.cheb_points(0.0, 0.25, 4), H.cheb_points(0.5, 0.75, 4)]
    ns = [H.cheb_points(0.5, 0.75, 4), H.cheb_points(0.0, 0.25, 4)]
    for kern, key in ((H.gaussian(0.7), "core2d_gauss"), (H.slp_2d(), "core2d_slp")):
        c = H.core_tensor(kern, nt, ns)
        ref = g()[key]
        assert np.linalg.norm(c - ref) <= 1e-14 * np.linalg.norm(ref)
    nt3 = [H.cheb_points(0.0, 0.25, 3)] * 3
    ns3 = [H.cheb_points(0.5, 0.75, 3)] * 3
    c = H.core_tensor(H.slp_3d(), nt3, ns3)
    assert np.linalg.norm(c - g()["core3d_slp"]) <= 1e-14 * np.linalg.norm(g()["core3d_slp"])


def test_pairwise_and_singular_rejection():
    x = np.array([[0.0, 0.0, 0.0]])
    y = np.array([[1.0, 2.0, 2.0]])
    assert abs(H.evaluate(H.slp_3d(), x, y) - 1.0 / (4 * np.pi * 3.0)) <= 1e-16
    assert abs(H.evaluate(H.gaussian(1.0), x, x) - 1.0) == 0.0
    with pytest.raises(ValueError, match="diagonal"):
        H.pairwise(H.slp_3d(), x, x)
