"""The reference's per-block API (htlr.tensor, htlr.blocks builders and
applies), device-backed (csrc/htlr_tensor.cu), against the reference's own
values (tests/golden: functions.npz, cfg1_matvec.npz, hmatrix.npz -- made by
tests/golden/make_golden.py from the reference) and numpy.  Tolerance: 1e-12
relative (fp64), QR factors sign-exact (LAPACK conventions, as numpy)."""

import os

import numpy as np
import pytest

import paper_2508_05958_b200 as H
from oracle import htlr_oracle as O

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def rel(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("shape", [(8, 3), (32, 8), (100, 7), (24, 6), (6, 6), (512, 64)])
def test_qr_matches_numpy_signs_and_values(shape):
    a = np.random.default_rng(shape[0]).standard_normal(shape)
    f = H.qr(a)
    q, r = np.linalg.qr(a, mode="reduced")
    assert rel(f.q, q) <= 1e-12 and rel(f.r, r) <= 1e-12
    assert rel(f.q @ f.r, a) <= 1e-13
    with pytest.raises(ValueError):
        H.qr(a.T if shape[0] > shape[1] else np.zeros((2, 3)))


def test_mode_product_contract_multi_mode_vs_numpy():
    rng = np.random.default_rng(5)
    t = rng.standard_normal((3, 4, 5, 6))
    m = rng.standard_normal((7, 5))
    got = H.mode_product(t, m, 3)
    ref = np.moveaxis(np.tensordot(m, t, axes=([1], [2])), 0, 2)
    assert got.shape == (3, 4, 7, 6) and rel(got, ref) <= 1e-14
    b = rng.standard_normal((6, 4, 2))
    got = H.contract(t, b, [4, 2], [1, 2])
    assert rel(got, np.tensordot(t, b, axes=([3, 1], [0, 1]))) <= 1e-14
    fs = [(rng.standard_normal((2, 3)), 1), (rng.standard_normal((9, 6)), 4)]
    got = H.multi_mode_apply(t, fs)
    ref = t
    for mm, mode in fs:
        ref = np.moveaxis(np.tensordot(mm, ref, axes=([1], [mode - 1])), 0, mode - 1)
    assert rel(got, ref) <= 1e-14
    with pytest.raises(ValueError):
        H.mode_product(t, m, 2)          # extent mismatch
    with pytest.raises(ValueError):
        H.multi_mode_apply(t, [(m, 3), (m, 3)])
    with pytest.raises(ValueError):
        H.contract(t, b, [4], [2])
    v = rng.standard_normal(24)
    assert np.array_equal(H.tensor_to_vec(H.vec_to_tensor(v, (2, 3, 4))), v)
    assert np.array_equal(H.reshape(v, (4, 6)), v.reshape((4, 6), order="F"))


@pytest.mark.parametrize("key,kernel", [("tb2_slp", H.slp_2d()), ("tb2_gauss_sq", H.gaussian(0.5)),
                                        ("tb3_slp", H.slp_3d())])
def test_build_tlr_and_tlr_apply_vs_reference(key, kernel):
    g = np.load(os.path.join(GOLD, "functions.npz"))
    meta = g[key + "_meta"].astype(int)
    d, n, p = meta[:3]
    tb = tuple((int(meta[3 + 2 * a]), int(meta[4 + 2 * a])) for a in range(d))
    sb = tuple((int(meta[3 + 2 * d + 2 * a]), int(meta[4 + 2 * d + 2 * a])) for a in range(d))
    grid = H.UniformGrid(d, n)
    blk = H.build_tlr(kernel, grid, H.IndexBox(tb), H.IndexBox(sb), int(p), grid.h)
    assert rel(blk.core, g[key + "_core"]) <= 1e-12
    for a in range(d):
        for side, facs in (("u", blk.u_factors), ("v", blk.v_factors)):
            ref = g[f"{key}_{side}{a}"]
            if ref.size == 0:
                assert facs[a] is None
            else:
                assert rel(facs[a], ref) <= 1e-12
    assert rel(H.materialize(blk), g[key + "_mat"]) <= 1e-12
    assert rel(H.tlr_apply(blk, g[key + "_seg"]), g[key + "_apply"]) <= 1e-12
    with pytest.raises(ValueError):
        H.tlr_apply(blk, np.zeros(3))
    with pytest.raises(ValueError):
        H.build_tlr(kernel, grid, H.IndexBox(tb), H.IndexBox(tb), int(p), grid.h)   # overlapping domains
    with pytest.raises(NotImplementedError):
        H.build_tlr(kernel, grid, H.IndexBox(tb), H.IndexBox(sb), int(p), grid.h, trim=True)


def test_build_dense_vs_reference_cfg1():
    """The first two leaves of config 1 (tau == sigma with the cell-average
    diagonal and a = 1, and a neighbour pair) against the reference's blocks."""
    g = np.load(os.path.join(GOLD, "cfg1_matvec.npz"))
    grid = H.UniformGrid(2, 64)
    leaves = O.block_leaves(64, 2, 8)
    for lid in (0, 1):
        lf = leaves[lid]
        blk = H.build_dense(H.neg_log_2d(), H.CoefficientFn.constant(1.0), grid, H.IndexBox(lf.tau),
                            H.IndexBox(lf.sigma), grid.h, H.QuadratureConfig())
        assert rel(blk.matrix, g[f"leaf{lid}_dense"]) <= 1e-12


def test_build_lowrank_vs_reference_hmatrix():
    g = np.load(os.path.join(GOLD, "hmatrix.npz"))
    cases = {"h2_weak_gauss": (2, 64, 8, 4, "weak", None, H.gaussian(np.sqrt(2.0))),
             "h3_eta1_slp": (3, 16, 4, 3, "strong", 1.0, H.slp_3d())}
    for key, (d, n, leaf, p, rule, eta, kern) in cases.items():
        lf = O.block_leaves(n, d, leaf, rule, eta)[int(g[key + "_adm_leaf"][0])]
        grid = H.UniformGrid(d, n)
        blk = H.build_lowrank(kern, grid, H.IndexBox(lf.tau), H.IndexBox(lf.sigma), p, grid.h)
        assert rel(H.materialize(blk), g[key + "_adm_mat"]) <= 1e-12
        seg = np.random.default_rng(1).standard_normal(blk.shape[1])
        assert rel(H.lowrank_apply(blk, seg), g[key + "_adm_mat"] @ seg) <= 1e-12
