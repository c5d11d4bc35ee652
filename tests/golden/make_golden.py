"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Run in the build container (where the read-only reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [name ...]

It imports the reference package ``htlr`` and calls only its public/stock
functions (construct, matvec, build_tlr, build_dense, tlr_apply, cheb_points,
factor_matrix, core_tensor, diagonal_entry, build_cluster_tree,
build_block_cluster_tree).  The fixtures are the parity pin for both the CPU
oracle (oracle/htlr_oracle.py) and the CUDA path; nothing at test time reads
/root/reference.

BASELINE.json kernels are expressed in the reference exactly as SURVEY.md
8(c) prescribes: -log r and 1/r as translation-invariant custom KernelSpecs,
exp(-r^2/0.01) as gaussian(0.1/sqrt(2)).

Configs 3 and 4 are too large for the full reference operator (130 GB /
5.3 TB), so their matvec rows come from the sampled-target restriction: walk
the reference's DFS leaf list, keep the leaves whose tau contains a chosen
leaf box, build each payload with the reference's builders and accumulate
exactly as operators.py:146-155 does.  That restriction is bit-identical to
the full reference matvec on those rows (checked on config 2 by
`check_sampled`).
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

import htlr  # noqa: E402  (the reference, via PYTHONPATH)
from htlr import blocks as rblocks  # noqa: E402
from htlr import grids as rgrids  # noqa: E402
from htlr import operators as rops  # noqa: E402


def k_neglog():
    return htlr.KernelSpec(kind="custom", evaluator=lambda x, y: -0.5 * np.log(((x - y) ** 2).sum(-1)),
                           smooth_at_diagonal=False, translation_invariant=True)


def k_invr():
    return htlr.KernelSpec(kind="custom", evaluator=lambda x, y: 1.0 / np.sqrt(((x - y) ** 2).sum(-1)),
                           smooth_at_diagonal=False, translation_invariant=True)


def k_gauss_baseline():
    return htlr.gaussian(0.1 / np.sqrt(2.0))


# name -> (d, n, leaf, rank, kernel factory, a, seed/input spec)
BASELINE = {
    "cfg1": dict(d=2, n=64, leaf=8, rank=8, kernel=k_neglog, a=1.0),
    "cfg2": dict(d=3, n=32, leaf=8, rank=6, kernel=k_invr, a=0.0),
    "cfg3": dict(d=3, n=64, leaf=8, rank=6, kernel=k_invr, a=0.0),
    "cfg4": dict(d=3, n=128, leaf=8, rank=8, kernel=k_gauss_baseline, a=0.0),
}


def baseline_input(name: str, N: int) -> np.ndarray:
    """BASELINE.json seeds, F-order grid linearisation."""
    if name == "cfg1":
        return np.random.default_rng(0).uniform(-1, 1, N)
    if name == "cfg2":
        return np.random.default_rng(1).uniform(-1, 1, N)
    if name == "cfg3":
        return np.random.default_rng(2).standard_normal((N, 16))
    if name == "cfg4":
        return np.random.default_rng(3).uniform(-1, 1, N)
    raise KeyError(name)


def make_cfg(spec, rule=None):
    return htlr.BuildConfig(rank=spec["rank"], leaf_side=spec["leaf"],
                            rule=rule or htlr.AdmissibilityRule.strong(1.0),
                            kernel=spec["kernel"](), coeff=htlr.CoefficientFn.constant(spec["a"]))


def leaves_array(btree, d):
    rows = []
    for lf in btree.leaves:
        kind = 0 if lf.kind == rgrids.ADMISSIBLE else 1
        rows.append([lf.leaf_id, kind, lf.level]
                    + [v for r in lf.tau.box.ranges for v in r]
                    + [v for r in lf.sigma.box.ranges for v in r])
    return np.asarray(rows, dtype=np.int32).reshape(-1, 3 + 4 * d)


def list_digest(arr: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr, dtype=np.int32).tobytes()).hexdigest()


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} B)", flush=True)


# ---------------------------------------------------------------- lists


def gen_lists():
    """Bit-exact DFS leaf lists: full arrays for small trees, sha256 + level
    histograms + strided spot rows for the big ones."""
    out = {}
    cases = [
        ("l2_n16_l4_weak", 2, 16, 4, htlr.AdmissibilityRule.weak()),
        ("l2_n16_l4_s1.4142", 2, 16, 4, htlr.AdmissibilityRule.strong(np.sqrt(2.0))),
        ("l2_n32_l16_weak", 2, 32, 16, htlr.AdmissibilityRule.weak()),
        ("l2_n64_l8_s1", 2, 64, 8, htlr.AdmissibilityRule.strong(1.0)),     # cfg1 tree
        ("l3_n16_l4_s1", 3, 16, 4, htlr.AdmissibilityRule.strong(1.0)),
        ("l3_n32_l5_s1", 3, 32, 5, htlr.AdmissibilityRule.strong(1.0)),
        ("l3_n32_l8_s1", 3, 32, 8, htlr.AdmissibilityRule.strong(1.0)),     # cfg2 tree
        ("l3_n24_l6_weak", 3, 24, 6, htlr.AdmissibilityRule.weak()),
        ("l2_n4_l4_weak", 2, 4, 4, htlr.AdmissibilityRule.weak()),
        ("l3_n64_l8_s1", 3, 64, 8, htlr.AdmissibilityRule.strong(1.0)),     # cfg3 tree
        ("l3_n128_l8_s1", 3, 128, 8, htlr.AdmissibilityRule.strong(1.0)),   # cfg4 tree
        ("l3_n96_l8_s1", 3, 96, 8, htlr.AdmissibilityRule.strong(1.0)),     # cfg5 tree (side 6)
    ]
    meta = []
    for key, d, n, leaf, rule in cases:
        t0 = time.time()
        grid = htlr.UniformGrid(d, n)
        btree = htlr.build_block_cluster_tree(htlr.build_cluster_tree(grid, leaf), rule)
        arr = leaves_array(btree, d)
        digest = list_digest(arr)
        hist = np.zeros((16, 2), dtype=np.int64)
        for lvl, kind in zip(arr[:, 2], arr[:, 1]):
            hist[lvl, kind] += 1
        if len(arr) <= 5000:
            out["full_" + key] = arr
        else:
            out["spot_" + key] = arr[:: max(1, len(arr) // 997)]
            out["spotidx_" + key] = np.arange(0, len(arr), max(1, len(arr) // 997))
        out["hist_" + key] = hist
        out["sha_" + key] = np.frombuffer(bytes.fromhex(digest), dtype=np.uint8)
        eta = rule.eta if rule.kind == "strong" else -1.0
        meta.append([d, n, leaf, eta, len(arr)])
        out["meta_" + key] = np.asarray([d, n, leaf, eta, len(arr)], dtype=np.float64)
        print(f"lists {key}: {len(arr)} leaves in {time.time() - t0:.1f}s", flush=True)
    save("lists", **out)


# ---------------------------------------------------------------- diag


def gen_diag():
    out = {}
    cases = {
        "cfg1": (k_neglog(), 2, 1 / 64),
        "cfg2": (k_invr(), 3, 1 / 32),
        "cfg3": (k_invr(), 3, 1 / 64),
        "cfg4": (k_gauss_baseline(), 3, 1 / 128),
        "slp2d_h1_16": (htlr.slp_2d(), 2, 1 / 16),
        "slp3d_h1_16": (htlr.slp_3d(), 3, 1 / 16),
        "gauss1.4142_2d_h1_32": (htlr.gaussian(np.sqrt(2.0)), 2, 1 / 32),
        "gauss0.3_3d_h1_8": (htlr.gaussian(0.3), 3, 1 / 8),
    }
    for key, (k, d, h) in cases.items():
        center = np.full(d, 0.5 * h)
        out[key] = np.asarray([htlr.diagonal_entry(k, center, h, htlr.QuadratureConfig())])
        print(f"diag {key} = {out[key][0]!r}")
    save("diag", **out)


# ---------------------------------------------------------------- functions


def gen_functions():
    """Known-answer data for the interpolation building blocks."""
    rng = np.random.default_rng(1234)
    out = {}
    for p in (1, 2, 3, 6, 8):
        g = htlr.cheb_points(0.25, 0.75, p)
        out[f"cheb_{p}"] = g.nodes
        pts = np.sort(rng.uniform(0.25, 0.75, 13))
        out[f"fac_pts_{p}"] = pts
        out[f"fac_{p}"] = htlr.factor_matrix(pts, g)
    # cores on a 2-D and a 3-D box pair
    gt = [htlr.cheb_points(0.0, 0.25, 4), htlr.cheb_points(0.5, 0.75, 4)]
    gs = [htlr.cheb_points(0.5, 0.75, 4), htlr.cheb_points(0.0, 0.25, 4)]
    out["core2d_gauss"] = htlr.core_tensor(htlr.gaussian(0.7), gt, gs)
    out["core2d_slp"] = htlr.core_tensor(htlr.slp_2d(), gt, gs)
    gt3 = [htlr.cheb_points(0.0, 0.25, 3)] * 3
    gs3 = [htlr.cheb_points(0.5, 0.75, 3)] * 3
    out["core3d_slp"] = htlr.core_tensor(htlr.slp_3d(), gt3, gs3)
    # Tucker blocks (reference-native kernels), sign-normalised factors
    tcases = {
        "tb2_slp": (htlr.slp_2d(), 2, 32, ((0, 8), (0, 8)), ((16, 24), (8, 16)), 6),
        "tb2_gauss_sq": (htlr.gaussian(0.5), 2, 32, ((0, 8), (0, 8)), ((16, 24), (8, 16)), 8),
        "tb3_slp": (htlr.slp_3d(), 3, 16, ((0, 4), (0, 4), (0, 4)), ((8, 12), (4, 8), (0, 4)), 3),
    }
    for key, (k, d, n, tb, sb, p) in tcases.items():
        grid = htlr.UniformGrid(d, n)
        blk = htlr.build_tlr(k, grid, htlr.IndexBox(tb), htlr.IndexBox(sb), p, grid.h)
        out[key + "_core"] = blk.core
        out[key + "_mat"] = htlr.materialize(blk)
        for a in range(d):
            for side, facs in (("u", blk.u_factors), ("v", blk.v_factors)):
                out[f"{key}_{side}{a}"] = facs[a] if facs[a] is not None else np.zeros((0, 0))
        seg = rng.standard_normal(int(np.prod([hi - lo for lo, hi in sb])))
        out[key + "_seg"] = seg
        out[key + "_apply"] = htlr.tlr_apply(blk, seg)
        out[key + "_meta"] = np.asarray([d, n, p] + [v for r in tb for v in r] + [v for r in sb for v in r])
    save("functions", **out)


# ---------------------------------------------------------------- small full matvecs


SMALL = {
    # key: (d, n, leaf, rank, rule, kernel, a, seed)
    "s2_weak_gauss": (2, 32, 16, 8, ("weak", None), lambda: htlr.gaussian(np.sqrt(2.0)), 0.0, 38),
    "s2_strong_slp": (2, 32, 8, 6, ("strong", np.sqrt(2.0)), htlr.slp_2d, 0.5, 39),
    "s2_eta1_slp_sq": (2, 32, 4, 4, ("strong", 1.0), htlr.slp_2d, 1.0, 40),
    "s3_eta1_slp": (3, 16, 4, 3, ("strong", 1.0), htlr.slp_3d, 0.0, 41),
    "s3_weak_gauss_sq": (3, 16, 4, 4, ("weak", None), lambda: htlr.gaussian(0.4), 2.0, 42),
    "s3_eta1_gauss": (3, 32, 8, 6, ("strong", 1.0), lambda: htlr.gaussian(0.3), 0.0, 43),
    "s2_single_leaf": (2, 4, 4, 4, ("weak", None), htlr.slp_2d, 0.0, 37),
}


def gen_small():
    out = {}
    for key, (d, n, leaf, rank, (rk, eta), kf, a, seed) in SMALL.items():
        t0 = time.time()
        rule = htlr.AdmissibilityRule.weak() if rk == "weak" else htlr.AdmissibilityRule.strong(eta)
        cfg = htlr.BuildConfig(rank=rank, leaf_side=leaf, rule=rule, kernel=kf(),
                               coeff=htlr.CoefficientFn.constant(a))
        grid = htlr.UniformGrid(d, n)
        op = htlr.construct(cfg, grid)
        u = np.random.default_rng(seed).standard_normal(grid.num_points)
        out[key + "_f"] = htlr.matvec(op, u)
        rep = htlr.storage_report(op)
        out[key + "_storage"] = np.asarray([rep.dense_scalars, rep.factor_scalars, rep.core_scalars,
                                            rep.total_scalars], dtype=np.int64)
        print(f"small {key}: {time.time() - t0:.1f}s", flush=True)
    save("small", **out)


# ---------------------------------------------------------------- BASELINE configs


def full_matvec(name):
    spec = BASELINE[name]
    grid = htlr.UniformGrid(spec["d"], spec["n"])
    cfg = make_cfg(spec)
    t0 = time.time()
    op = htlr.construct(cfg, grid, threads=os.cpu_count() or 1)
    t1 = time.time()
    u = baseline_input(name, grid.num_points)
    f = htlr.matvec(op, u)
    t2 = time.time()
    print(f"{name}: construct {t1 - t0:.1f}s matvec {t2 - t1:.2f}s", flush=True)
    return op, u, f


def pick_blocks(op, per_level=2):
    """A few payloads per (level, kind), factors sign-normalised."""
    chosen = {}
    for lf in op.block_tree.leaves:
        key = (lf.level, lf.kind)
        chosen.setdefault(key, [])
        if len(chosen[key]) < per_level:
            chosen[key].append(lf)
    return [lf for v in chosen.values() for lf in v]


def gen_cfg(name, with_blocks=True):
    op, u, f = full_matvec(name)
    d = op.grid.d
    out = {"f": f}
    if with_blocks:
        for lf in pick_blocks(op, per_level=1 if name == "cfg2" else 2):
            pl = op.payloads[lf.leaf_id]
            tag = f"leaf{lf.leaf_id}"
            if isinstance(pl, rblocks.DenseBlock):
                out[tag + "_dense"] = pl.matrix
            else:
                out[tag + "_core"] = pl.core
                for a in range(d):
                    for side, facs in (("u", pl.u_factors), ("v", pl.v_factors)):
                        out[f"{tag}_{side}{a}"] = facs[a] if facs[a] is not None else np.zeros((0, 0))
    rep = htlr.storage_report(op)
    out["storage"] = np.asarray([rep.dense_scalars, rep.factor_scalars, rep.core_scalars,
                                 rep.total_scalars], dtype=np.int64)
    save(name + "_matvec", **out)


def sampled_rows(name, target_boxes):
    """Reference sampled-target restriction (see module docstring)."""
    spec = BASELINE[name]
    grid = htlr.UniformGrid(spec["d"], spec["n"])
    cfg = make_cfg(spec)
    t0 = time.time()
    btree = htlr.build_block_cluster_tree(htlr.build_cluster_tree(grid, cfg.leaf_side), cfg.rule)
    print(f"{name}: tree {time.time() - t0:.1f}s, {len(btree.leaves)} leaves", flush=True)
    diag = rops._cached_diag(cfg, grid)
    u = baseline_input(name, grid.num_points)
    U = u.reshape(grid.num_points, -1)
    R = U.shape[1]
    shape = (grid.n,) * grid.d
    uts = [U[:, r].reshape(shape, order="F") for r in range(R)]
    fts = [np.zeros(shape) for _ in range(R)]
    tb = [htlr.IndexBox(t) for t in target_boxes]

    def contains(outer, inner):
        return all(a <= c and e <= b for (a, b), (c, e) in zip(outer.ranges, inner.ranges))

    nleaf = 0
    for leaf in btree.leaves:
        if not any(contains(leaf.tau.box, t) for t in tb):
            continue
        nleaf += 1
        if leaf.kind == rgrids.ADMISSIBLE:
            block = rblocks.build_tlr(cfg.kernel, grid, leaf.tau.box, leaf.sigma.box, cfg.rank, grid.h)
        else:
            block = rblocks.build_dense(cfg.kernel, cfg.coeff, grid, leaf.tau.box, leaf.sigma.box,
                                        grid.h, cfg.quadrature, diag_value=diag)
        for r in range(R):
            seg = uts[r][leaf.sigma.box.slices].ravel(order="F")
            if isinstance(block, rblocks.DenseBlock):
                res = block.matrix @ seg
            else:
                res = rblocks.tlr_apply(block, seg)
            fts[r][leaf.tau.box.slices] += res.reshape(leaf.tau.box.sizes, order="F")
    rows = np.zeros((len(tb), tb[0].num_points, R))
    for i, t in enumerate(tb):
        for r in range(R):
            rows[i, :, r] = fts[r][t.slices].ravel(order="F")
    print(f"{name}: sampled {len(tb)} boxes via {nleaf} leaves in {time.time() - t0:.1f}s", flush=True)
    return rows


def boxes(side, idx_list, d=3):
    return [tuple((i * side, (i + 1) * side) for i in idx) for idx in idx_list]


SAMPLES = {
    "cfg2": boxes(8, [(0, 0, 0), (1, 2, 3), (3, 0, 1)]),
    "cfg3": boxes(8, [(0, 0, 0), (3, 0, 0), (3, 3, 0), (3, 4, 3), (7, 7, 7)]),
    "cfg4": boxes(8, [(0, 0, 0), (7, 8, 0), (7, 8, 9), (15, 3, 12)]),
}


def gen_sampled(name):
    rows = sampled_rows(name, SAMPLES[name])
    save(name + "_sampled", rows=rows, boxes=np.asarray(SAMPLES[name], dtype=np.int64))


def check_sampled():
    """The sampled restriction equals the full reference matvec bit for bit
    (config 2)."""
    data = np.load(os.path.join(HERE, "cfg2_matvec.npz"))
    rows = sampled_rows("cfg2", SAMPLES["cfg2"])
    f = data["f"]
    n = 32
    for i, bx in enumerate(SAMPLES["cfg2"]):
        mesh = np.meshgrid(*[np.arange(lo, hi) for lo, hi in bx], indexing="ij")
        lin = (mesh[0] + n * mesh[1] + n * n * mesh[2]).ravel(order="F")
        diff = np.abs(rows[i, :, 0] - f[lin]).max()
        print(f"sampled vs full cfg2 box {i}: max |diff| = {diff!r}")
        assert diff == 0.0


# ---------------------------------------------------------------- quasi-uniform pipeline (8(f) f3)


def jittered_mesh(k, seed):
    """Structured mesh with interior vertices moved (still a valid cover)."""
    from htlr import quasi as rq
    m = rq.structured_trimesh(k)
    v = m.vertices.copy()
    rng = np.random.default_rng(seed)
    interior = (v[:, 0] > 0) & (v[:, 0] < 1) & (v[:, 1] > 0) & (v[:, 1] < 1)
    v[interior] += rng.uniform(-0.25, 0.25, (interior.sum(), 2)) / k
    return rq.TriMesh(vertices=v, triangles=m.triangles)


def gen_quasi():
    from htlr import quasi as rq
    out = {}
    cfg = htlr.BuildConfig(rank=4, leaf_side=4, rule=htlr.AdmissibilityRule.weak(),
                           kernel=htlr.gaussian(np.sqrt(2.0)), coeff=htlr.CoefficientFn.constant(0.0))
    for key, mesh in (("structured", rq.structured_trimesh(8)), ("jittered", jittered_mesh(8, 5))):
        out[key + "_vertices"] = mesh.vertices
        out[key + "_triangles"] = mesh.triangles
        pipe = rq.build_pipeline(mesh, cfg, 2.0)
        out[key + "_m_side"] = np.asarray([pipe.m_side])
        out[key + "_S"] = pipe.to_uniform.matrix.toarray()
        out[key + "_T"] = pipe.to_quasi.matrix.toarray()
        u = np.random.default_rng(11).standard_normal(mesh.num_triangles)
        out[key + "_u"] = u
        out[key + "_f"] = rq.apply_pipeline(pipe, u)
    tri = np.array([[0.1, 0.05], [0.9, 0.3], [0.35, 0.95]])
    cells = [(0.0, 0.0, 0.5, 0.5), (0.25, 0.25, 0.75, 0.75), (0.5, 0.0, 1.0, 0.5), (0.9, 0.9, 1.0, 1.0)]
    out["ov_tri"] = tri
    out["ov_cells"] = np.asarray(cells)
    out["ov_areas"] = np.asarray([rq.overlap_area(tri, c) for c in cells])
    save("quasi", **out)


def gen_hmatrix():
    """H-matrix baseline (construct_hmatrix / hmatrix_matvec) on small grids."""
    out = {}
    cases = {
        "h2_weak_gauss": (2, 64, 8, 4, htlr.AdmissibilityRule.weak(), htlr.gaussian(np.sqrt(2.0)), 41),
        "h3_eta1_slp": (3, 16, 4, 3, htlr.AdmissibilityRule.strong(1.0), htlr.slp_3d(), 42),
    }
    for key, (d, n, leaf, p, rule, k, seed) in cases.items():
        cfg = htlr.BuildConfig(rank=p, leaf_side=leaf, rule=rule, kernel=k, coeff=htlr.CoefficientFn.constant(0.0))
        grid = htlr.UniformGrid(d, n)
        hop = htlr.construct_hmatrix(cfg, grid)
        u = np.random.default_rng(seed).standard_normal(grid.num_points)
        out[key + "_f"] = htlr.hmatrix_matvec(hop, u)
        rep = htlr.storage_report(hop)
        out[key + "_storage"] = np.asarray([rep.dense_scalars, rep.factor_scalars, rep.core_scalars,
                                            rep.total_scalars], dtype=np.int64)
        for lf in hop.block_tree.leaves:
            if lf.kind == rgrids.ADMISSIBLE:
                out[key + "_adm_leaf"] = np.asarray([lf.leaf_id])
                out[key + "_adm_mat"] = htlr.materialize(hop.payloads[lf.leaf_id])
                break
    save("hmatrix", **out)


def main(argv):
    jobs = {
        "hmatrix": gen_hmatrix,
        "quasi": gen_quasi,
        "lists": gen_lists, "diag": gen_diag, "functions": gen_functions, "small": gen_small,
        "cfg1": lambda: gen_cfg("cfg1"), "cfg2": lambda: gen_cfg("cfg2"),
        "cfg2_sampled_check": check_sampled,
        "cfg3": lambda: gen_sampled("cfg3"), "cfg4": lambda: gen_sampled("cfg4"),
    }
    names = argv or list(jobs)
    for nm in names:
        jobs[nm]()


if __name__ == "__main__":
    main(sys.argv[1:])
