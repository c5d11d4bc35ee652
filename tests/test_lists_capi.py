"""CPU tests of the C-ABI library: it loads, exports every symbol the header
declares, and its host list builder reproduces the reference's DFS leaf
lists bit for bit (golden fixtures from the reference).  No device work."""

import hashlib
import os
import re

import numpy as np
import pytest

import paper_2508_05958_b200 as H
from paper_2508_05958_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def gold_lists():
    return np.load(os.path.join(GOLD, "lists.npz"))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "htlr_b200.h")).read()
    return sorted(set(re.findall(r"\b(htlr_[a-z_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _lib.lib()
    declared = header_symbols()
    assert declared, "no declarations parsed"
    bound = {name for name, _, _ in _lib.SYMBOLS}
    for name in declared:
        assert hasattr(lib, name), name
        assert name in bound, f"{name} declared but not bound in _lib.SYMBOLS"


def rule_of(eta):
    return H.AdmissibilityRule.weak() if eta < 0 else H.AdmissibilityRule.strong(float(eta))


def all_list_keys():
    g = gold_lists()
    return sorted(k[len("meta_"):] for k in g.files if k.startswith("meta_"))


@pytest.mark.parametrize("key", all_list_keys())
def test_lists_bit_exact_vs_reference(key):
    g = gold_lists()
    d, n, leaf, eta, count = g["meta_" + key]
    d, n, leaf, count = int(d), int(n), int(leaf), int(count)
    grid = H.UniformGrid(d, n)
    tree = H.build_cluster_tree(grid, leaf)
    bt = H.build_block_cluster_tree(tree, rule_of(eta))
    arr = bt.leaf_array
    assert arr.shape == (count, 3 + 4 * d)
    assert hashlib.sha256(np.ascontiguousarray(arr, dtype=np.int32).tobytes()).digest() == bytes(g["sha_" + key])
    if "full_" + key in g.files:
        assert np.array_equal(arr, g["full_" + key])
    else:
        assert np.array_equal(arr[g["spotidx_" + key]], g["spot_" + key])
    hist = np.zeros((16, 2), dtype=np.int64)
    np.add.at(hist, (arr[:, 2], arr[:, 1]), 1)
    assert np.array_equal(hist, g["hist_" + key])


def test_leaf_objects_match_reference_semantics():
    grid = H.UniformGrid(2, 16)
    tree = H.build_cluster_tree(grid, 4)
    bt = H.build_block_cluster_tree(tree, H.AdmissibilityRule.strong(np.sqrt(2.0)))
    # at most 9 dense blocks per leaf row, reached by interior rows (test_grids.py:147-158)
    counts = {}
    for lf in bt.leaves:
        if lf.kind == H.INADMISSIBLE:
            counts[lf.tau.box.ranges] = counts.get(lf.tau.box.ranges, 0) + 1
    assert max(counts.values()) == 9
    # leaves partition all index pairs exactly once (test_grids.py:167-183)
    cov = np.zeros((256, 256), dtype=np.int8)
    for lf in bt.leaves:
        cov[np.ix_(lf.tau.box.linear_indices(16), lf.sigma.box.linear_indices(16))] += 1
    assert np.all(cov == 1)


def test_block_tree_root_rebuilds_internal_nodes():
    grid = H.UniformGrid(2, 16)
    bt = H.build_block_cluster_tree(H.build_cluster_tree(grid, 4), H.AdmissibilityRule.weak())
    seen = []

    def walk(node):
        if node.children:
            assert node.kind == H.grids.INTERNAL
            for c in node.children:
                walk(c)
        else:
            seen.append(node.leaf_id)

    walk(bt.root)
    assert seen == list(range(len(bt.leaves)))


def test_tiny_problem_single_dense_root():
    grid = H.UniformGrid(2, 4)
    bt = H.build_block_cluster_tree(H.build_cluster_tree(grid, 4), H.AdmissibilityRule.weak())
    assert len(bt.leaves) == 1 and bt.leaves[0].kind == H.INADMISSIBLE
    assert bt.root.leaf_id == 0


def test_invalid_inputs_raise_value_error():
    with pytest.raises(ValueError):
        H.UniformGrid(4, 8)
    with pytest.raises(ValueError):
        H.build_cluster_tree(H.UniformGrid(2, 10), 4)
    with pytest.raises(ValueError):
        H.AdmissibilityRule.strong(0.0)
    with pytest.raises(ValueError):
        H.BuildConfig(rank=0, leaf_side=8, rule=H.AdmissibilityRule.weak(),
                      kernel=H.gaussian(1.0), coeff=H.CoefficientFn.constant(0.0))
    with pytest.warns(UserWarning, match="recommended range"):
        H.BuildConfig(rank=4, leaf_side=16, rule=H.AdmissibilityRule.weak(),
                      kernel=H.gaussian(1.0), coeff=H.CoefficientFn.constant(0.0))


def test_custom_kernels_are_rejected_not_emulated():
    k = H.custom(lambda x, y: np.zeros(np.broadcast(x, y).shape[:-1]))
    cfg = H.BuildConfig(rank=4, leaf_side=4, rule=H.AdmissibilityRule.weak(), kernel=k,
                        coeff=H.CoefficientFn.constant(1.0))
    with pytest.raises(ValueError, match="B200"):
        H.construct(cfg, H.UniformGrid(2, 8))


def test_host_only_plan_refuses_device_work():
    import ctypes
    L = _lib.lib()
    desc = _lib.HtlrDesc(d=2, n=16, leaf_side_max=4, rank=4, rule=1, eta=1.0, kernel=0, sigma=1.0,
                         scale=1.0, quad_q=10, corner_subdivision=0, coeff_const=0.0)
    plan = ctypes.c_void_p()
    _lib.check(L.htlr_plan_create(ctypes.byref(desc), -1, ctypes.byref(plan)))
    try:
        _lib.check(L.htlr_build_lists(plan))
        out = np.zeros(5, dtype=np.int64)
        _lib.check(L.htlr_storage(plan, out.ctypes.data))
        assert out[3] == out[0] + out[1] + out[2]
        with pytest.raises(ValueError, match="host-only"):
            _lib.check(L.htlr_construct(plan, None))
    finally:
        L.htlr_plan_destroy(plan)


def test_storage_accounting_matches_reference_cfg1():
    import ctypes
    L = _lib.lib()
    desc = _lib.HtlrDesc(d=2, n=64, leaf_side_max=8, rank=8, rule=1, eta=1.0, kernel=1, sigma=0.0,
                         scale=1.0, quad_q=10, corner_subdivision=1, coeff_const=1.0)
    plan = ctypes.c_void_p()
    _lib.check(L.htlr_plan_create(ctypes.byref(desc), -1, ctypes.byref(plan)))
    try:
        _lib.check(L.htlr_build_lists(plan))
        out = np.zeros(5, dtype=np.int64)
        _lib.check(L.htlr_storage(plan, out.ctypes.data))
    finally:
        L.htlr_plan_destroy(plan)
    gold = np.load(os.path.join(GOLD, "cfg1_matvec.npz"))["storage"]
    assert list(out[:4]) == list(gold)


def _gaussian_host_plan(n, eta=1.0):
    """Host-only plan of a separable-eligible problem (Gaussian, p = leaf side
    = 8, 3-D): the kind whose levels 3 and 4 can be built analytically."""
    import ctypes
    from paper_2508_05958_b200.operators import _desc
    cfg = H.BuildConfig(rank=8, leaf_side=8, rule=H.AdmissibilityRule.strong(eta), kernel=H.gaussian(0.1),
                        coeff=H.CoefficientFn.constant(0.0))
    plan = ctypes.c_void_p()
    _lib.check(_lib.lib().htlr_plan_create(ctypes.byref(_desc(cfg, H.UniformGrid(3, n))), -1, ctypes.byref(plan)))
    return plan


def _tree_info(plan):
    import ctypes
    depth, side = ctypes.c_int32(), ctypes.c_int32()
    nl, na, nn = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _lib.check(_lib.lib().htlr_tree_info(plan, ctypes.byref(depth), ctypes.byref(side), ctypes.byref(nl),
                                         ctypes.byref(na), ctypes.byref(nn)))
    return depth.value, side.value, nl.value, na.value, nn.value


@pytest.mark.parametrize("n", [64, 128])
def test_analytic_banded_levels_equal_the_dfs_lists(n, monkeypatch):
    """Uniform grid, n a power of two, eta = 1: the plan proves the banded
    product-set structure per (level, offset) and builds no pair lists below
    level 2 (htlr_plan.cu analytic_bands_ok).  Its leaf counts (from the
    product sets) and its lazily built DFS list must equal the plan that
    walks the whole DFS (HTLR_ANALYTIC=0) and the reference fixture."""
    from paper_2508_05958_b200.grids import export_leaf_array
    L = _lib.lib()
    info, arrs = {}, {}
    for mode in ("1", "0"):
        monkeypatch.setenv("HTLR_ANALYTIC", mode)
        plan = _gaussian_host_plan(n)
        try:
            _lib.check(L.htlr_build_lists(plan))
            info[mode] = _tree_info(plan)          # before any export: the analytic counts
            arrs[mode] = export_leaf_array(plan, 3)
            assert _tree_info(plan) == info[mode]  # after the lazy DFS
        finally:
            L.htlr_plan_destroy(plan)
    assert info["1"] == info["0"]
    assert np.array_equal(arrs["1"], arrs["0"])
    g = gold_lists()
    key = [k for k in all_list_keys() if tuple(int(v) for v in g["meta_" + k][:3]) == (3, n, 8)
           and float(g["meta_" + k][3]) == 1.0]
    assert key, "no reference fixture for this tree"
    assert hashlib.sha256(np.ascontiguousarray(arrs["1"], dtype=np.int32).tobytes()).digest() == bytes(g["sha_" + key[0]])


def test_analytic_banded_levels_need_eta_one():
    """eta = 2 has other near sets: the per-offset check fails, the plan walks
    the DFS (and still reproduces the reference's list)."""
    from paper_2508_05958_b200.grids import export_leaf_array
    L = _lib.lib()
    plan = _gaussian_host_plan(64, eta=2.0)
    try:
        _lib.check(L.htlr_build_lists(plan))
        arr = export_leaf_array(plan, 3)
    finally:
        L.htlr_plan_destroy(plan)
    grid = H.UniformGrid(3, 64)
    ref = H.build_block_cluster_tree(H.build_cluster_tree(grid, 8), H.AdmissibilityRule.strong(2.0)).leaf_array
    assert np.array_equal(arr, ref)
