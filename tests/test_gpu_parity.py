"""GPU parity of the B200 HTLR path against the reference (golden fixtures
generated from the reference itself) and the CPU oracle.

Tolerance (BASELINE north star): relative 2-norm error <= 1e-12 in fp64 for
matvecs and construction; lists bit-exact (tests/test_lists_capi.py)."""

import os

import numpy as np
import pytest

import paper_2508_05958_b200 as H
from paper_2508_05958_b200.configs import WORKLOADS
from oracle import htlr_oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")
TOL = 1e-12

pytestmark = pytest.mark.gpu


def load(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


def rel(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    return np.linalg.norm(a - b) / np.linalg.norm(b)


# ------------------------------------------------------------------ diag

DIAG = {
    "cfg1": (H.neg_log_2d(), 2, 1 / 64),
    "cfg2": (H.inv_r_3d(), 3, 1 / 32),
    "cfg3": (H.inv_r_3d(), 3, 1 / 64),
    "cfg4": (H.gaussian_bw(0.1), 3, 1 / 128),
    "slp2d_h1_16": (H.slp_2d(), 2, 1 / 16),
    "slp3d_h1_16": (H.slp_3d(), 3, 1 / 16),
    "gauss1.4142_2d_h1_32": (H.gaussian(np.sqrt(2.0)), 2, 1 / 32),
    "gauss0.3_3d_h1_8": (H.gaussian(0.3), 3, 1 / 8),
}


@pytest.mark.parametrize("key", sorted(DIAG))
def test_diagonal_entry_device(key):
    k, d, h = DIAG[key]
    val = H.diagonal_entry(k, np.full(d, h / 2), h, H.QuadratureConfig())
    gold = float(load("diag")[key][0])
    assert abs(val - gold) <= 1e-13 * abs(gold)


# ------------------------------------------------------------------ small reference cases

SMALL = {
    "s2_weak_gauss": (2, 32, 16, 8, H.AdmissibilityRule.weak(), H.gaussian(np.sqrt(2.0)), 0.0, 38),
    "s2_strong_slp": (2, 32, 8, 6, H.AdmissibilityRule.strong(np.sqrt(2.0)), H.slp_2d(), 0.5, 39),
    "s2_eta1_slp_sq": (2, 32, 4, 4, H.AdmissibilityRule.strong(1.0), H.slp_2d(), 1.0, 40),
    "s3_eta1_slp": (3, 16, 4, 3, H.AdmissibilityRule.strong(1.0), H.slp_3d(), 0.0, 41),
    "s3_weak_gauss_sq": (3, 16, 4, 4, H.AdmissibilityRule.weak(), H.gaussian(0.4), 2.0, 42),
    "s3_eta1_gauss": (3, 32, 8, 6, H.AdmissibilityRule.strong(1.0), H.gaussian(0.3), 0.0, 43),
    "s2_single_leaf": (2, 4, 4, 4, H.AdmissibilityRule.weak(), H.slp_2d(), 0.0, 37),
}


@pytest.mark.parametrize("key", sorted(SMALL))
def test_small_matvec_vs_reference(key):
    d, n, leaf, rank, rule, k, a, seed = SMALL[key]
    cfg = H.BuildConfig(rank=rank, leaf_side=leaf, rule=rule, kernel=k, coeff=H.CoefficientFn.constant(a))
    grid = H.UniformGrid(d, n)
    op = H.construct(cfg, grid)
    u = np.random.default_rng(seed).standard_normal(grid.num_points)
    f = H.matvec(op, u)
    assert isinstance(f, np.ndarray) and f.shape == u.shape
    assert rel(f, load("small")[key + "_f"]) <= TOL
    rep = H.storage_report(op)
    gold = load("small")[key + "_storage"]
    assert [rep.dense_scalars, rep.factor_scalars, rep.core_scalars, rep.total_scalars] == list(gold)


# ------------------------------------------------------------------ BASELINE configs


def build(name):
    w = WORKLOADS[name]
    return w, H.construct(w.build_config(), w.grid)


def test_cfg1_full_matvec():
    w, op = build("cfg1")
    f = H.matvec(op, w.input())
    assert rel(f, load("cfg1_matvec")["f"]) <= TOL
    assert op.diag_value() == pytest.approx(float(load("diag")["cfg1"][0]), rel=1e-13)


def test_cfg2_full_matvec_repeated():
    w, op = build("cfg2")
    u = w.input()
    gold = load("cfg2_matvec")["f"]
    for _ in range(3):   # the config runs 10 matvecs on one operator
        f = H.matvec(op, u)
        assert rel(f, gold) <= TOL


def _box_rows(n, box):
    mesh = np.meshgrid(*[np.arange(lo, hi) for lo, hi in box], indexing="ij")
    lin = mesh[0] + n * mesh[1] + n * n * mesh[2]
    return lin.ravel(order="F")


def test_cfg3_sampled_rows_16rhs():
    w, op = build("cfg3")
    U = w.input()
    F = H.matmat(op, U)
    g = load("cfg3_sampled")
    for i, box in enumerate(g["boxes"]):
        rows = _box_rows(w.n, box)
        assert rel(F[rows], g["rows"][i]) <= TOL


def test_cfg4_sampled_rows():
    w, op = build("cfg4")
    f = H.matvec(op, w.input())
    g = load("cfg4_sampled")
    for i, box in enumerate(g["boxes"]):
        rows = _box_rows(w.n, box)
        assert rel(f[rows], g["rows"][i][:, 0]) <= TOL


# ------------------------------------------------------------------ construction parity


def _sign_normalise(block):
    """Column signs of every factor -> +, compensated in the core (QR sign
    conventions are only unique up to column signs)."""
    core = block.core.copy()
    d = len(block.u_factors)
    facs = []
    for side, lst in ((0, block.u_factors), (1, block.v_factors)):
        for a, f in enumerate(lst):
            if f is None:
                facs.append(None)
                continue
            idx = np.argmax(np.abs(f), axis=0)
            s = np.sign(f[idx, np.arange(f.shape[1])])
            facs.append(f * s)
            mode = a if side == 0 else d + a
            shape = [1] * (2 * d)
            shape[mode] = len(s)
            core = core * s.reshape(shape)
    return core, facs


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_construction_blocks_vs_reference(name):
    w, op = build(name)
    g = load(name + "_matvec")
    ids = sorted({int(k[4:].split("_")[0]) for k in g.files if k.startswith("leaf")})
    assert ids
    d = w.d
    for lid in ids:
        blk = op.payloads[lid]
        tag = f"leaf{lid}"
        if tag + "_dense" in g.files:
            assert isinstance(blk, H.DenseBlock)
            assert rel(blk.matrix, g[tag + "_dense"]) <= TOL
            continue
        ref = H.TuckerBlock(core=g[tag + "_core"],
                            u_factors=[g[f"{tag}_u{a}"] if g[f"{tag}_u{a}"].size else None for a in range(d)],
                            v_factors=[g[f"{tag}_v{a}"] if g[f"{tag}_v{a}"].size else None for a in range(d)])
        c1, f1 = _sign_normalise(blk)
        c2, f2 = _sign_normalise(ref)
        assert rel(c1, c2) <= TOL
        for a, b in zip(f1, f2):
            assert (a is None) == (b is None)
            if a is not None:
                assert rel(a, b) <= TOL
        assert rel(H.materialize(blk), H.materialize(ref)) <= TOL


# ------------------------------------------------------------------ properties / edge cases


def test_identity_operator():
    """k == 0 (scale 0), a == 1 -> f == u (test_operators.py:71-79)."""
    grid = H.UniformGrid(2, 32)
    cfg = H.BuildConfig(rank=8, leaf_side=16, rule=H.AdmissibilityRule.weak(),
                        kernel=H.gaussian(1.0, scale=0.0), coeff=H.CoefficientFn.constant(1.0))
    op = H.construct(cfg, grid)
    u = np.random.default_rng(35).standard_normal(grid.num_points)
    assert np.abs(H.matvec(op, u) - u).max() <= 1e-14


def test_single_leaf_is_the_dense_block():
    """n <= leaf side: the root is one inadmissible leaf (test_operators.py:
    112-120 / 148-164), so the matvec is that dense block -- K h^d with the
    cell-average diagonal, plus a -- applied to u."""
    for d, n, kd, ko in ((2, 8, H.neg_log_2d(), O.Kernel("slp2d", scale=2 * np.pi)),
                         (3, 8, H.inv_r_3d(), O.Kernel("slp3d", scale=4 * np.pi))):
        cfg = H.BuildConfig(rank=4, leaf_side=8, rule=H.AdmissibilityRule.strong(1.0), kernel=kd,
                            coeff=H.CoefficientFn.constant(0.25))
        op = H.construct(cfg, H.UniformGrid(d, n))
        pb = O.Problem(d=d, n=n, rank=4, leaf_side_max=8, kernel=ko, coeff=O.constant_coeff(0.25))
        full = tuple((0, n) for _ in range(d))
        A = O.dense_block(pb.kernel, pb.coeff, n, full, full, pb.diag())
        u = np.random.default_rng(40 + d).standard_normal(n ** d)
        assert rel(H.matvec(op, u), A @ u) <= 1e-14


def test_zero_input_gives_exact_zero():
    grid = H.UniformGrid(3, 16)
    cfg = H.BuildConfig(rank=4, leaf_side=4, rule=H.AdmissibilityRule.strong(1.0),
                        kernel=H.slp_3d(), coeff=H.CoefficientFn.constant(0.5))
    op = H.construct(cfg, grid)
    assert np.all(H.matvec(op, np.zeros(grid.num_points)) == 0.0)


def test_linearity_and_length_check():
    grid = H.UniformGrid(2, 32)
    cfg = H.BuildConfig(rank=8, leaf_side=16, rule=H.AdmissibilityRule.weak(),
                        kernel=H.gaussian(np.sqrt(2.0)), coeff=H.CoefficientFn.constant(0.0))
    op = H.construct(cfg, grid)
    rng = np.random.default_rng(39)
    u, v = rng.standard_normal((2, grid.num_points))
    lhs = H.matvec(op, 2.0 * u - 0.5 * v)
    rhs = 2.0 * H.matvec(op, u) - 0.5 * H.matvec(op, v)
    assert np.abs(lhs - rhs).max() <= 1e-12 * np.abs(lhs).max()
    with pytest.raises(ValueError):
        H.matvec(op, np.zeros(10))


def test_device_tensor_path_and_matmat_columns():
    import torch
    w, op = build("cfg2")
    rng = np.random.default_rng(5)
    U = rng.standard_normal((w.grid.num_points, 3))
    Ud = torch.from_numpy(U).cuda()
    Fd = H.matmat(op, Ud)
    assert Fd.is_cuda and tuple(Fd.shape) == U.shape
    F = Fd.cpu().numpy()
    for r in range(3):
        assert rel(F[:, r], H.matvec(op, U[:, r])) <= 1e-13


def test_variable_coefficient_vs_oracle():
    grid = H.UniformGrid(2, 16)
    fn = lambda pts: 1.0 + pts[:, 0] * pts[:, 1]   # noqa: E731
    cfg = H.BuildConfig(rank=4, leaf_side=4, rule=H.AdmissibilityRule.strong(1.0),
                        kernel=H.slp_2d(), coeff=H.CoefficientFn(fn))
    op = H.construct(cfg, grid)
    u = np.random.default_rng(3).standard_normal(grid.num_points)
    pb = O.Problem(d=2, n=16, rank=4, leaf_side_max=4, kernel=O.Kernel("slp2d"), coeff=fn)
    assert rel(H.matvec(op, u), O.matvec(pb, u)) <= TOL


ORACLE_CASES = [
    # d, n, leaf, rank, rule, eta, kernel(oracle), kernel(device), a
    (3, 16, 4, 4, "strong", 1.0, O.Kernel("gaussian", sigma=0.25), H.gaussian(0.25), 0.0),
    (3, 16, 8, 5, "strong", 1.5, O.Kernel("slp3d", scale=2.0), H.slp_3d(scale=2.0), 0.25),
    (2, 64, 8, 6, "weak", None, O.Kernel("slp2d"), H.slp_2d(), 0.0),
    (2, 32, 4, 3, "strong", 0.7, O.Kernel("gaussian", sigma=0.2), H.gaussian(0.2), 1.0),
    (3, 24, 6, 6, "weak", None, O.Kernel("slp3d"), H.slp_3d(), 0.0),
]


@pytest.mark.parametrize("case", range(len(ORACLE_CASES)))
def test_random_configs_vs_oracle(case):
    d, n, leaf, rank, rule, eta, ko, kd, a = ORACLE_CASES[case]
    arule = H.AdmissibilityRule.weak() if rule == "weak" else H.AdmissibilityRule.strong(eta)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        cfg = H.BuildConfig(rank=rank, leaf_side=leaf, rule=arule, kernel=kd, coeff=H.CoefficientFn.constant(a))
    op = H.construct(cfg, H.UniformGrid(d, n))
    u = np.random.default_rng(100 + case).standard_normal((n ** d, 2))
    pb = O.Problem(d=d, n=n, rank=rank, leaf_side_max=leaf, kernel=ko, coeff=O.constant_coeff(a),
                   rule=rule, eta=eta)
    assert rel(H.matmat(op, u), O.matvec(pb, u)) <= TOL


def test_rank_above_box_side_raises_like_reference():
    cfg = H.BuildConfig(rank=8, leaf_side=4, rule=H.AdmissibilityRule.strong(1.0),
                        kernel=H.slp_3d(), coeff=H.CoefficientFn.constant(0.0))
    with pytest.raises(ValueError, match="qr requires rows >= cols"):
        H.construct(cfg, H.UniformGrid(3, 16))


# ------------------------------------------------------------------ exact rows / sampled error (8(f) f2)


def test_exact_rows_match_dense_reference_operator():
    """Device exact rows == rows of the reference-built dense operator (small
    grid, oracle dense blocks are the reference's build_dense restated)."""
    grid = H.UniformGrid(2, 16)
    k, a = H.slp_2d(), 0.5
    ev = H.exact_row_evaluator(k, H.CoefficientFn.constant(a), grid, H.QuadratureConfig())
    pb = O.Problem(d=2, n=16, rank=4, leaf_side_max=16, kernel=O.Kernel("slp2d"), coeff=O.constant_coeff(a))
    full = ((0, 16), (0, 16))
    D = O.dense_block(pb.kernel, pb.coeff, 16, full, full, pb.diag())
    u = np.random.default_rng(8).standard_normal(256)
    rows = np.array([0, 17, 100, 255])
    assert rel(ev(rows, u), (D @ u)[rows]) <= 1e-13


def test_exact_rows_mapped_match_oracle_dense():
    grid = H.MappedGrid(2, 16, 0.05)
    ev = H.exact_row_evaluator(H.slp_2d(), H.CoefficientFn.constant(0.0), grid, H.QuadratureConfig())
    pb = O.MappedProblem(d=2, geo=O.MappedGeometry(16, 0.05), rank=4, leaf_side_max=16, kernel=O.Kernel("slp2d"),
                         coeff=O.constant_coeff(0.0))
    D = O.mapped_dense_matrix(pb)
    u = np.random.default_rng(9).standard_normal(256)
    rows = np.array([3, 77, 200])
    assert rel(ev(rows, u), (D @ u)[rows]) <= 1e-12


def test_estimate_rel_error_cfg4_scale():
    """Accuracy (not parity) of config 4 at full scale: 1000 exact rows."""
    w, op = build("cfg4")
    cfg = w.build_config()
    ev = H.exact_row_evaluator(cfg.kernel, cfg.coeff, w.grid, cfg.quadrature)
    err = H.estimate_rel_error_random(op, ev, w.input(), sample_size=1000, seed=1)
    print("cfg4 sampled relative error", err)
    assert err < 1e-3


def test_randomised_parity_sweep():
    """tools/fuzz_parity.py: random dimension / grid (uniform or mapped) /
    leaf side / rank / admissibility / kernel / coefficient / RHS count
    against the oracle's full matvec, all within 1e-12."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "tools/fuzz_parity.py", "2", "12"], cwd=root, capture_output=True,
                         text=True, timeout=1200)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]


def test_field_shaped_input_flattens_in_fortran_order():
    """matvec accepts the grid field as an (n,)*d array and flattens it like
    the reference, u.ravel(order="F") (operators.py:139): first index fastest.
    numpy and torch (host and device) inputs, against the reference fixture."""
    import torch
    w = WORKLOADS["cfg1"]
    op = H.construct(w.build_config(), w.grid)
    u = w.input()
    gold = load("cfg1_matvec")["f"]
    field = u.reshape((64, 64), order="F")
    for x in (field, torch.from_numpy(field), torch.from_numpy(field).cuda()):
        f = H.matvec(op, x)
        f = f.cpu().numpy() if isinstance(f, torch.Tensor) else np.asarray(f)
        assert f.shape == (4096,)
        assert rel(f, gold) <= TOL


def test_cfg4_full_size_properties():
    """BASELINE config 4 at its own size (N = 2,097,152), through properties
    that do not need the reference's (infeasible) full matvec: the operator
    the reference defines is symmetric (uniform weights, a symmetric kernel,
    Tucker blocks whose (tau, sigma) and (sigma, tau) cores are transposes:
    blocks.py:126-164), commutes with the grid's reflections x_a -> 1 - x_a
    (the tree, the lists and the Chebyshev nodes are reflection symmetric) and
    is linear.  Sampled rows of the same matvec are checked against the
    reference's fixture in test_matvec_sampled_rows_vs_reference."""
    import torch
    w, op = build("cfg4")
    assert op.leaf_pass() == "banded"
    n = w.grid.n
    rng = np.random.default_rng(11)
    u, v = (torch.from_numpy(rng.standard_normal(n ** 3)).cuda() for _ in range(2))
    Au, Av = H.matvec(op, u).clone(), H.matvec(op, v).clone()
    # symmetry: <v, A u> = <u, A v>
    s1, s2 = float(torch.dot(v, Au)), float(torch.dot(u, Av))
    scale = float(torch.linalg.norm(v) * torch.linalg.norm(Au))
    assert abs(s1 - s2) <= 1e-12 * scale, (s1, s2)
    # linearity
    lhs = H.matvec(op, 2.0 * u - 0.5 * v)
    assert float(torch.linalg.norm(lhs - (2.0 * Au - 0.5 * Av)) / torch.linalg.norm(lhs)) <= 1e-13
    # reflections: the F-order vector as an (x, y, z) field is u.reshape(z, y, x)
    for dims in ((0,), (1,), (2,), (0, 1, 2)):
        ur = torch.flip(u.reshape(n, n, n), dims).reshape(-1).contiguous()
        Aur = H.matvec(op, ur)
        ref = torch.flip(Au.reshape(n, n, n), dims).reshape(-1)
        assert float(torch.linalg.norm(Aur - ref) / torch.linalg.norm(ref)) <= 1e-12, dims
