"""BASELINE config 5 (mapped quasi-uniform grid), CPU side: the reference has
no mapped grid, so the oracle restatement is self-checked (amplitude 0
reproduces the reference-pinned uniform oracle bit for bit; the compressed
operator matches the dense Nystrom matrix to approximation accuracy; the
rectangular-cell quadrature converges), and the C++ list builder's mapped
lists are compared with the oracle's bit for bit."""

import numpy as np
import pytest

import paper_2508_05958_b200 as H
from oracle import htlr_oracle as O


@pytest.mark.parametrize("d,n,leaf", [(3, 16, 4), (3, 24, 6), (2, 32, 4), (3, 48, 6)])
def test_mapped_lists_bit_exact_vs_oracle(d, n, leaf):
    geo = O.MappedGeometry(n, 0.05)
    ref = O.leaves_to_array(O.mapped_block_leaves(geo, d, leaf, "strong", 1.0), d)
    grid = H.MappedGrid(d, n, 0.05)
    bt = H.build_block_cluster_tree(H.build_cluster_tree(grid, leaf), H.AdmissibilityRule.strong(1.0))
    assert np.array_equal(bt.leaf_array, ref)


def test_mapped_geometry_tables_match_device_tables():
    grid = H.MappedGrid(3, 96, 0.05)
    geo = O.MappedGeometry(96, 0.05)
    assert np.array_equal(grid.coords1d(), geo.coords())
    assert np.array_equal(grid.bounds1d(), geo.boundaries())
    assert abs(geo.widths().sum() - 1.0) < 1e-14
    # symmetric map: phi(1 - t) = 1 - phi(t)
    assert np.allclose(geo.boundaries()[::-1], 1.0 - geo.boundaries(), atol=1e-15)


def test_amplitude_zero_reproduces_uniform_oracle():
    k = O.Kernel("slp2d", scale=2 * np.pi)
    u = np.random.default_rng(1).standard_normal(32 ** 2)
    pm = O.MappedProblem(d=2, geo=O.MappedGeometry(32, 0.0), rank=6, leaf_side_max=8, kernel=k,
                         coeff=O.constant_coeff(0.5))
    pu = O.Problem(d=2, n=32, rank=6, leaf_side_max=8, kernel=k, coeff=O.constant_coeff(0.5))
    fm = O.mapped_matvec(pm, u)
    fu = O.matvec(pu, u)
    assert np.linalg.norm(fm - fu) <= 1e-14 * np.linalg.norm(fu)


def test_mapped_operator_matches_dense_nystrom():
    k = O.Kernel("slp2d", scale=2 * np.pi)
    u = np.random.default_rng(2).standard_normal(32 ** 2)
    err = {}
    for amp in (0.0, 0.05):
        pb = O.MappedProblem(d=2, geo=O.MappedGeometry(32, amp), rank=6, leaf_side_max=8, kernel=k,
                             coeff=O.constant_coeff(0.0))
        fm = O.mapped_matvec(pb, u)
        fd = O.mapped_dense_matrix(pb) @ u
        err[amp] = np.linalg.norm(fm - fd) / np.linalg.norm(fd)
    # interpolation error of the same order as on the uniform grid
    assert err[0.05] < 1e-4 and err[0.0] < 1e-4


def test_rectangular_cell_quadrature_converges():
    geo = O.MappedGeometry(12, 0.05)
    k = O.Kernel("slp3d")
    idx = (3, 7, 10)
    a = O.mapped_cell_integral(k, geo, idx, q=10)
    b = O.mapped_cell_integral(k, geo, idx, q=20)
    assert abs(a - b) <= 1e-12 * abs(b)
    # centred cubic cell: equals the reference's cell average times h^d
    g0 = O.MappedGeometry(12, 0.0)
    c = O.mapped_cell_integral(k, g0, idx, q=10)
    assert abs(c - O.cell_average(k, 3, 1 / 12) / 12 ** 3) <= 1e-13 * abs(c)


def test_cfg5_lists_bit_exact_vs_oracle_fixture():
    """BASELINE config 5 at its own size (n = 96, leaf_side 8 -> side-6
    leaves, 2.65 M leaves): the C++ builder's DFS list equals the oracle's
    mapped restatement bit for bit (sha256 of the whole list, the
    (level, kind) histogram, strided rows; tests/golden/make_mapped_fixtures.py).
    Ties of the predicate on the non-dyadic mapped domains (grids.py:153-165)
    are where the two could part."""
    import hashlib
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "mapped.npz"))
    grid = H.MappedGrid(3, 96, 0.05)
    arr = H.build_block_cluster_tree(H.build_cluster_tree(grid, 8), H.AdmissibilityRule.strong(1.0)).leaf_array
    hist = np.zeros((16, 2), dtype=np.int64)
    np.add.at(hist, (arr[:, 2], arr[:, 1]), 1)
    assert np.array_equal(hist, g["cfg5_hist"])
    assert np.array_equal(arr[g["cfg5_spotidx"]], g["cfg5_spot"])
    sha = hashlib.sha256(np.ascontiguousarray(arr, dtype=np.int32).tobytes()).digest()
    assert sha == bytes(g["cfg5_sha"])
