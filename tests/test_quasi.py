"""Quasi-uniform triangle pipeline against fixtures generated
by the reference's quasi.py (tests/golden/make_golden.py gen_quasi)."""

import os

import numpy as np
import pytest

import paper_2508_05958_b200 as H

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold():
    return np.load(os.path.join(GOLD, "quasi.npz"))


def mesh(key):
    g = gold()
    return H.TriMesh(vertices=g[key + "_vertices"], triangles=g[key + "_triangles"])


def test_structured_mesh_matches_reference_fixture():
    m = H.structured_trimesh(8)
    g = gold()
    assert np.array_equal(m.vertices, g["structured_vertices"])
    assert np.array_equal(m.triangles, g["structured_triangles"])
    assert abs(m.areas.sum() - 1.0) < 1e-14


def test_mesh_io_roundtrip(tmp_path):
    m = mesh("jittered")
    p = tmp_path / "m.txt"
    H.save_mesh(m, p)
    m2 = H.load_mesh(p)
    assert np.array_equal(m.vertices, m2.vertices) and np.array_equal(m.triangles, m2.triangles)
    bad = tmp_path / "bad.txt"
    bad.write_text("3 1\n0 0\n1 0\n")
    with pytest.raises(ValueError):
        H.load_mesh(bad)


def test_mesh_validation():
    with pytest.raises(ValueError):
        H.TriMesh(vertices=[[0, 0], [1, 0], [0, 1]], triangles=[[0, 1, 5]])
    with pytest.raises(ValueError):   # covers half the square only
        H.TriMesh(vertices=[[0, 0], [1, 0], [0, 1]], triangles=[[0, 1, 2]])


def test_valid_uniform_side():
    assert H.quasi.valid_uniform_side(30, 4) == 32
    assert H.quasi.valid_uniform_side(16, 4) == 16


@pytest.mark.gpu
def test_overlap_area_known_values():
    g = gold()
    for cell, ref in zip(g["ov_cells"], g["ov_areas"]):
        assert abs(H.overlap_area(g["ov_tri"], tuple(cell)) - ref) <= 1e-15


@pytest.mark.gpu
@pytest.mark.parametrize("key", ["structured", "jittered"])
def test_transfer_matrices_and_pipeline_vs_reference(key):
    g = gold()
    m = mesh(key)
    cfg = H.BuildConfig(rank=4, leaf_side=4, rule=H.AdmissibilityRule.weak(),
                        kernel=H.gaussian(np.sqrt(2.0)), coeff=H.CoefficientFn.constant(0.0))
    pipe = H.build_pipeline(m, cfg, 2.0)
    assert pipe.m_side == int(g[key + "_m_side"][0])
    assert np.abs(pipe.to_uniform.toarray() - g[key + "_S"]).max() <= 1e-12
    assert np.abs(pipe.to_quasi.toarray() - g[key + "_T"]).max() <= 1e-12
    f = H.apply_pipeline(pipe, g[key + "_u"])
    ref = g[key + "_f"]
    assert np.linalg.norm(f - ref) / np.linalg.norm(ref) <= 1e-12
    with pytest.raises(ValueError):
        H.apply_pipeline(pipe, np.zeros(3))
