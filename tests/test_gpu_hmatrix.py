"""H-matrix baseline against the reference's
construct_hmatrix / hmatrix_matvec fixtures, and TLR == low-rank agreement
(test_operators.py:ecTestHMatrixBaseline in the reference)."""

import os

import numpy as np
import pytest

import paper_2508_05958_b200 as H

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")

CASES = {
    "h2_weak_gauss": (2, 64, 8, 4, H.AdmissibilityRule.weak(), H.gaussian(np.sqrt(2.0)), 41),
    "h3_eta1_slp": (3, 16, 4, 3, H.AdmissibilityRule.strong(1.0), H.slp_3d(), 42),
}


def rel(a, b):
    return np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b))


@pytest.mark.parametrize("key", sorted(CASES))
def test_hmatrix_vs_reference(key):
    g = np.load(os.path.join(GOLD, "hmatrix.npz"))
    d, n, leaf, p, rule, k, seed = CASES[key]
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        cfg = H.BuildConfig(rank=p, leaf_side=leaf, rule=rule, kernel=k, coeff=H.CoefficientFn.constant(0.0))
    grid = H.UniformGrid(d, n)
    hop = H.construct_hmatrix(cfg, grid)
    u = np.random.default_rng(seed).standard_normal(grid.num_points)
    f = H.hmatrix_matvec(hop, u)
    assert rel(f, g[key + "_f"]) <= 1e-12
    top = H.construct(cfg, grid)
    assert np.abs(H.matvec(top, u) - f).max() <= 1e-12 * np.abs(f).max()   # TLR == low-rank
    rep = H.storage_report(hop)
    assert [rep.dense_scalars, rep.factor_scalars, rep.core_scalars, rep.total_scalars] == list(g[key + "_storage"])
    assert rep.total_scalars > H.storage_report(top).total_scalars
    lid = int(g[key + "_adm_leaf"][0])
    blk = hop.payloads[lid]
    assert isinstance(blk, H.LowRankBlock)
    assert rel(H.materialize(blk), g[key + "_adm_mat"]) <= 1e-12
