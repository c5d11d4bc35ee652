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
