"""Pin the CPU oracle (oracle/htlr_oracle.py) against the fixtures generated
from the reference itself (tests/golden/make_golden.py).  CPU only."""

import os

import numpy as np
import pytest

from oracle import htlr_oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


BASE_KERNELS = {
    "cfg1": O.Kernel("slp2d", scale=2 * np.pi),
    "cfg2": O.Kernel("slp3d", scale=4 * np.pi),
    "cfg3": O.Kernel("slp3d", scale=4 * np.pi),
    "cfg4": O.Kernel("gaussian", sigma=0.1 / np.sqrt(2.0)),
}


def rel(a, b):
    return np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b))


# ---------------------------------------------------------------- lists

SMALL_LISTS = {
    "l2_n16_l4_weak": (2, 16, 4, "weak", None),
    "l2_n16_l4_s1.4142": (2, 16, 4, "strong", np.sqrt(2.0)),
    "l2_n32_l16_weak": (2, 32, 16, "weak", None),
    "l2_n64_l8_s1": (2, 64, 8, "strong", 1.0),
    "l3_n16_l4_s1": (3, 16, 4, "strong", 1.0),
    "l3_n32_l8_s1": (3, 32, 8, "strong", 1.0),
    "l3_n24_l6_weak": (3, 24, 6, "weak", None),
    "l2_n4_l4_weak": (2, 4, 4, "weak", None),
}


@pytest.mark.parametrize("key", sorted(SMALL_LISTS))
def test_oracle_lists_bit_exact(key):
    d, n, leaf, rule, eta = SMALL_LISTS[key]
    gold = load("lists")["full_" + key]
    arr = O.leaves_to_array(O.block_leaves(n, d, leaf, rule, eta), d)
    assert arr.shape == gold.shape
    assert np.array_equal(arr, gold)


def test_oracle_lists_cfg3_digest():
    import hashlib
    g = load("lists")
    arr = O.leaves_to_array(O.block_leaves(64, 3, 8, "strong", 1.0), 3).astype(np.int32)
    assert hashlib.sha256(arr.tobytes()).digest() == bytes(g["sha_l3_n64_l8_s1"])


def test_leaf_side_rules():
    assert O.leaf_side(96, 8) == 6
    assert O.leaf_side(32, 5) == 4
    with pytest.raises(ValueError):
        O.leaf_side(10, 4)


# ---------------------------------------------------------------- diag

DIAG_KERNELS = {
    "cfg1": (BASE_KERNELS["cfg1"], 2, 1 / 64),
    "cfg2": (BASE_KERNELS["cfg2"], 3, 1 / 32),
    "cfg3": (BASE_KERNELS["cfg3"], 3, 1 / 64),
    "cfg4": (BASE_KERNELS["cfg4"], 3, 1 / 128),
    "slp2d_h1_16": (O.Kernel("slp2d"), 2, 1 / 16),
    "slp3d_h1_16": (O.Kernel("slp3d"), 3, 1 / 16),
    "gauss1.4142_2d_h1_32": (O.Kernel("gaussian", sigma=np.sqrt(2.0)), 2, 1 / 32),
    "gauss0.3_3d_h1_8": (O.Kernel("gaussian", sigma=0.3), 3, 1 / 8),
}


@pytest.mark.parametrize("key", sorted(DIAG_KERNELS))
def test_oracle_diag(key):
    k, d, h = DIAG_KERNELS[key]
    gold = float(load("diag")[key][0])
    val = O.cell_average(k, d, h)
    # scaled built-ins vs the reference's custom evaluators differ by a few ulp
    assert abs(val - gold) <= 1e-14 * abs(gold)


# ---------------------------------------------------------------- building blocks


@pytest.mark.parametrize("p", [1, 2, 3, 6, 8])
def test_oracle_cheb_and_factors(p):
    g = load("functions")
    nodes = O.cheb_nodes(0.25, 0.75, p)
    assert np.array_equal(nodes, g[f"cheb_{p}"])
    fac = O.lagrange_matrix(g[f"fac_pts_{p}"], nodes)
    assert np.array_equal(fac, g[f"fac_{p}"])


def test_oracle_cores():
    g = load("functions")
    nt = [O.cheb_nodes(0.0, 0.25, 4), O.cheb_nodes(0.5, 0.75, 4)]
    ns = [O.cheb_nodes(0.5, 0.75, 4), O.cheb_nodes(0.0, 0.25, 4)]
    assert np.array_equal(O.kernel_core(O.Kernel("gaussian", sigma=0.7), nt, ns), g["core2d_gauss"])
    assert np.array_equal(O.kernel_core(O.Kernel("slp2d"), nt, ns), g["core2d_slp"])
    nt3 = [O.cheb_nodes(0.0, 0.25, 3)] * 3
    ns3 = [O.cheb_nodes(0.5, 0.75, 3)] * 3
    assert np.array_equal(O.kernel_core(O.Kernel("slp3d"), nt3, ns3), g["core3d_slp"])


TUCKER = {
    "tb2_slp": O.Kernel("slp2d"),
    "tb2_gauss_sq": O.Kernel("gaussian", sigma=0.5),
    "tb3_slp": O.Kernel("slp3d"),
}


@pytest.mark.parametrize("key", sorted(TUCKER))
def test_oracle_tucker_block(key):
    g = load("functions")
    meta = g[key + "_meta"]
    d, n, p = int(meta[0]), int(meta[1]), int(meta[2])
    rr = [int(v) for v in meta[3:]]
    tau = tuple((rr[2 * a], rr[2 * a + 1]) for a in range(d))
    sig = tuple((rr[2 * d + 2 * a], rr[2 * d + 2 * a + 1]) for a in range(d))
    blk = O.tucker_block(TUCKER[key], n, tau, sig, p)
    assert rel(blk.core, g[key + "_core"]) <= 1e-13
    for a in range(d):
        for side, facs in (("u", blk.ufac), ("v", blk.vfac)):
            ref = g[f"{key}_{side}{a}"]
            if ref.size == 0:
                assert facs[a] is None
            else:
                assert rel(facs[a], ref) <= 1e-13
    assert rel(O.materialize_tucker(blk), g[key + "_mat"]) <= 1e-13
    assert rel(O.tucker_apply(blk, g[key + "_seg"]), g[key + "_apply"]) <= 1e-13


# ---------------------------------------------------------------- matvecs

SMALL = {
    "s2_weak_gauss": (2, 32, 16, 8, "weak", None, O.Kernel("gaussian", sigma=np.sqrt(2.0)), 0.0, 38),
    "s2_strong_slp": (2, 32, 8, 6, "strong", np.sqrt(2.0), O.Kernel("slp2d"), 0.5, 39),
    "s2_eta1_slp_sq": (2, 32, 4, 4, "strong", 1.0, O.Kernel("slp2d"), 1.0, 40),
    "s3_eta1_slp": (3, 16, 4, 3, "strong", 1.0, O.Kernel("slp3d"), 0.0, 41),
    "s3_weak_gauss_sq": (3, 16, 4, 4, "weak", None, O.Kernel("gaussian", sigma=0.4), 2.0, 42),
    "s2_single_leaf": (2, 4, 4, 4, "weak", None, O.Kernel("slp2d"), 0.0, 37),
}


@pytest.mark.parametrize("key", sorted(SMALL))
def test_oracle_small_matvec(key):
    d, n, leaf, rank, rule, eta, k, a, seed = SMALL[key]
    pb = O.Problem(d=d, n=n, rank=rank, leaf_side_max=leaf, kernel=k,
                   coeff=O.constant_coeff(a), rule=rule, eta=eta)
    u = np.random.default_rng(seed).standard_normal(pb.num_points)
    f = O.matvec(pb, u)
    assert rel(f, load("small")[key + "_f"]) <= 1e-13


def test_oracle_cfg1_full_matvec():
    pb = O.Problem(d=2, n=64, rank=8, leaf_side_max=8, kernel=BASE_KERNELS["cfg1"],
                   coeff=O.constant_coeff(1.0))
    u = np.random.default_rng(0).uniform(-1, 1, pb.num_points)
    f = O.matvec(pb, u)
    assert rel(f, load("cfg1_matvec")["f"]) <= 1e-13


def test_oracle_sampled_equals_full_rows():
    """The sampled-target restriction reproduces the full matvec's rows."""
    pb = O.Problem(d=2, n=32, rank=4, leaf_side_max=4, kernel=O.Kernel("slp2d"),
                   coeff=O.constant_coeff(1.0))
    u = np.random.default_rng(40).standard_normal(pb.num_points)
    full = O.matvec(pb, u)
    boxes = [((0, 4), (0, 4)), ((12, 16), (20, 24))]
    rows = O.sampled_matvec(pb, u, boxes)
    for i, bx in enumerate(boxes):
        assert np.array_equal(rows[i, :, 0], full[O.box_linear_indices(32, bx)])


def test_oracle_storage_counts_cfg1():
    leaves = O.block_leaves(64, 2, 8, "strong", 1.0)
    pb = O.Problem(d=2, n=64, rank=8, leaf_side_max=8, kernel=BASE_KERNELS["cfg1"],
                   coeff=O.constant_coeff(1.0))
    c = O.storage_counts(pb, leaves)
    gold = load("cfg1_matvec")["storage"]
    assert [c["dense"], c["factors"], c["cores"], c["total"]] == list(gold)
