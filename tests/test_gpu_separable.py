"""GPU parity of the separable-core formulation (htlr_sep.cu): a Gaussian
kernel on a uniform 3-D grid with p = leaf side = 8 applies every block as
the Kronecker product of three 8 x 8 per-axis factors.  Same operator as the
reference's dense cores (blocks.py:126-227), so the bar is the same: relative
2-norm error <= 1e-12 against the oracle / the reference's fixtures (the
config-4 fixture is checked in test_gpu_parity.py), and against the
dense-core GEMM path of this package (HTLR_SEPARABLE=0)."""

import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2508_05958_b200 as H
from oracle import htlr_oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-12
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rel(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def make(n, sigma=0.1, scale=1.0, a=0.0):
    cfg = H.BuildConfig(rank=8, leaf_side=8, rule=H.AdmissibilityRule.strong(1.0),
                        kernel=H.gaussian(sigma, scale=scale), coeff=H.CoefficientFn.constant(a))
    return H.construct(cfg, H.UniformGrid(3, n))


def problem(n, sigma=0.1, scale=1.0, a=0.0):
    return O.Problem(d=3, n=n, rank=8, leaf_side_max=8, kernel=O.Kernel("gaussian", sigma=sigma, scale=scale),
                     coeff=O.constant_coeff(a))


BOXES = {
    32: [((0, 8), (0, 8), (0, 8)), ((8, 16), (16, 24), (24, 32)), ((16, 24), (8, 16), (8, 16))],
    64: [((0, 8), (0, 8), (0, 8)), ((24, 32), (40, 48), (56, 64)), ((32, 40), (32, 40), (24, 32))],
}


@pytest.mark.parametrize("n,sigma,scale,a", [(32, 0.15, 1.3, 0.7), (64, 0.1, 1.0, 0.0)])
def test_separable_sampled_rows_vs_oracle(n, sigma, scale, a):
    """Corner, edge and interior leaf boxes (every kind: near blocks with the
    self-block diagonal correction, leaf-level square cores, and at n = 64 the
    QR-factored level-2 cores) with two right-hand sides."""
    op = make(n, sigma, scale, a)
    assert op.formulation() == "separable"
    U = np.random.default_rng(n).standard_normal((n ** 3, 2))
    F = H.matmat(op, U)
    rows = O.sampled_matvec(problem(n, sigma, scale, a), U, BOXES[n])
    for i, bx in enumerate(BOXES[n]):
        assert rel(F[O.box_linear_indices(n, bx)], rows[i]) <= TOL


def test_separable_blocks_vs_oracle():
    """Construction parity: the exported separable blocks (Kronecker products
    of the device-built per-axis factors) against the oracle's Tucker / dense
    blocks, per (kind, level), after QR sign normalisation."""
    n = 64
    op = make(n, 0.1, 1.0, 0.25)
    pb = problem(n, 0.1, 1.0, 0.25)
    leaves = O.block_leaves(n, 3, 8)
    diag = pb.diag()
    picked = {}
    for lf in leaves:
        key = (lf.kind, lf.tau[0][1] - lf.tau[0][0])
        picked.setdefault(key, []).append(lf)
    rng = np.random.default_rng(5)
    chosen = []
    for key, lst in sorted(picked.items()):
        for j in rng.choice(len(lst), size=min(3, len(lst)), replace=False):
            chosen.append(lst[int(j)])
    selfs = [lf for lf in leaves if lf.kind != O.ADM and lf.tau == lf.sigma][:2]
    assert len(chosen) >= 6
    for lf in chosen + selfs:
        got = op.payloads[lf.leaf_id]
        ref = O.build_payload(pb, lf, diag)
        if isinstance(ref, O.Tucker):
            assert rel(H.materialize(got), O.materialize_tucker(ref)) <= TOL
        else:
            assert rel(got.matrix, ref) <= TOL


_DENSE_SCRIPT = r"""
import sys
import numpy as np
import paper_2508_05958_b200 as H
from paper_2508_05958_b200.configs import WORKLOADS
w = WORKLOADS["cfg4"]
op = H.construct(w.build_config(), w.grid)
np.save(sys.argv[1], H.matvec(op, w.input()))
print(op.formulation())
"""


def test_cfg4_separable_equals_dense_cores(tmp_path):
    """BASELINE config 4 through both formulations: the separable default and
    the dense-core GEMM path (HTLR_SEPARABLE=0, its own process)."""
    from paper_2508_05958_b200.configs import WORKLOADS
    w = WORKLOADS["cfg4"]
    op = H.construct(w.build_config(), w.grid)
    assert op.formulation() == "separable"
    f = H.matvec(op, w.input())
    out = tmp_path / "f.npy"
    r = subprocess.run([sys.executable, "-c", _DENSE_SCRIPT, str(out)], check=True, cwd=ROOT, capture_output=True,
                       text=True, env={**os.environ, "PYTHONPATH": ROOT, "HTLR_SEPARABLE": "0"}, timeout=900)
    assert r.stdout.strip().splitlines()[-1] == "dense"
    err = rel(f, np.load(out))
    print("cfg4 separable vs dense cores", err)
    assert err <= 1e-13


_CHUNK_SCRIPT = r"""
import sys
import numpy as np
import paper_2508_05958_b200 as H
cfg = H.BuildConfig(rank=8, leaf_side=8, rule=H.AdmissibilityRule.strong(1.0), kernel=H.gaussian(0.1),
                    coeff=H.CoefficientFn.constant(0.0))
op = H.construct(cfg, H.UniformGrid(3, 64))
assert op.formulation() == "separable"
U = np.random.default_rng(64).standard_normal((64 ** 3, 2))
np.save(sys.argv[1], H.matmat(op, U))
"""


_NB = {"HTLR_SEP_BAND": "0"}   # the cooperative / per-warp leaf passes instead of the banded sweeps


@pytest.mark.parametrize("env", [{**_NB, "HTLR_SEP_BLOCK": "0", "HTLR_SEP_CHUNK": "1"},
                                 {**_NB, "HTLR_SEP_BLOCK": "0", "HTLR_SEP_CHUNK": "9"},
                                 {**_NB, "HTLR_SEP_BLOCK": "0", "HTLR_SEP_CHUNK": "100000"},
                                 {**_NB, "HTLR_SEP_COLS": "1"}, {**_NB, "HTLR_SEP_COLS": "7"},
                                 {**_NB, "HTLR_SEP_COLS": "1000"},
                                 {**_NB},
                                 {"HTLR_GRAPHS": "0"}])
def test_separable_item_splits(tmp_path, env):
    """Leaf pass by per-warp items (cut at every group, at a few groups, or
    one item per target list) or by cooperative per-parent CTAs (one column,
    a few, or all columns per CTA), and direct launches: identical operator."""
    out = tmp_path / "f.npy"
    subprocess.run([sys.executable, "-c", _CHUNK_SCRIPT, str(out)], check=True, cwd=ROOT,
                   env={**os.environ, "PYTHONPATH": ROOT, **env}, timeout=600)
    F = np.load(out)
    U = np.random.default_rng(64).standard_normal((64 ** 3, 2))
    bx = BOXES[64]
    rows = O.sampled_matvec(problem(64), U, bx)
    for i, b in enumerate(bx):
        assert rel(F[O.box_linear_indices(64, b)], rows[i]) <= TOL


def test_non_separable_configs_keep_dense_cores():
    """1/r kernels, p != 8 and 2-D problems keep the dense-core path."""
    cfg = H.BuildConfig(rank=6, leaf_side=8, rule=H.AdmissibilityRule.strong(1.0), kernel=H.gaussian(0.1),
                        coeff=H.CoefficientFn.constant(0.0))
    assert H.construct(cfg, H.UniformGrid(3, 32)).formulation() == "dense"
    cfg = H.BuildConfig(rank=8, leaf_side=8, rule=H.AdmissibilityRule.strong(1.0), kernel=H.inv_r_3d(),
                        coeff=H.CoefficientFn.constant(0.0))
    assert H.construct(cfg, H.UniformGrid(3, 32)).formulation() == "dense"


def test_out_buffer_host_and_device():
    """matvec / matmat write into a caller's float64 tensor (pinned host or
    device) and return it; a wrong shape raises ValueError.  (Accumulation
    order across CTAs is not fixed -- fp64 RED -- so repeated matvecs agree to
    rounding, not bitwise.)"""
    import torch
    op = make(32, 0.15, 1.3, 0.7)
    u = np.random.default_rng(3).standard_normal(32 ** 3)
    ref = H.matvec(op, u)
    pin = torch.empty(32 ** 3, dtype=torch.float64).pin_memory()
    got = H.matvec(op, torch.from_numpy(u).pin_memory(), out=pin)
    assert got is pin and rel(pin.numpy(), ref) <= 1e-14
    dev = torch.empty((32 ** 3, 1), dtype=torch.float64, device="cuda")
    assert H.matmat(op, torch.from_numpy(u).reshape(-1, 1).cuda(), out=dev) is dev
    assert rel(dev.cpu().numpy()[:, 0], ref) <= 1e-14
    with pytest.raises(ValueError):
        H.matvec(op, u, out=torch.empty(7, dtype=torch.float64))


@pytest.mark.parametrize("n,a,R", [(64, 0.0, 1), (64, 0.4, 2), (128, 0.0, 1)])
def test_host_vector_path_matches_device(n, a, R):
    """Pinned host vectors go through htlr_matvec_host: for separable plans
    the PCIe copies are overlapped with the device work (z halves, two
    streams); the result equals the device-vector matvec (to rounding: RED
    accumulation order), on repeated calls (graph replay) and for R > 1."""
    import torch
    op = make(n, 0.1, 1.0, a)
    U = np.random.default_rng(n + R).standard_normal((n ** 3, R))
    ref = H.matmat(op, torch.from_numpy(U).cuda()).cpu().numpy()
    up = torch.from_numpy(U if R > 1 else U[:, 0].copy()).pin_memory()
    out = torch.empty(up.shape, dtype=torch.float64).pin_memory()
    for _ in range(3):
        got = (H.matmat if R > 1 else H.matvec)(op, up, out=out)
        assert got is out
        assert rel(got.numpy().reshape(-1, R), ref) <= 1e-14
    got2 = (H.matmat if R > 1 else H.matvec)(op, up)   # fresh pinned result (another graph)
    assert got2.is_pinned() and rel(got2.numpy().reshape(-1, R), ref) <= 1e-14


def test_host_vector_path_banded_pipeline():
    """Banded plans (n >= 64) stream u in and f out in z slabs around the
    per-slab upward / downward launches (htlr_matvec_host, HostPipe): 4 slabs
    of upward8, the passes, 4 of downward8 -- the result equals the device
    matvec, for R = 1 and R = 3 (slabs of point-major rows)."""
    import torch
    op = make(64, 0.1, 1.0, 0.2)
    assert op.leaf_pass() == "banded"
    for R in (1, 3):
        U = np.random.default_rng(40 + R).standard_normal((64 ** 3, R))
        ref = H.matmat(op, torch.from_numpy(U).cuda()).cpu().numpy()
        up = torch.from_numpy(U).pin_memory()
        out = torch.empty(up.shape, dtype=torch.float64).pin_memory()
        for _ in range(2):
            H.matmat(op, up, out=out)
            assert rel(out.numpy(), ref) <= 1e-14
        assert op.last_launch_count() >= 8


def test_graph_cache_rotating_device_buffers():
    """Device vectors: graphs are keyed by the caller's (u, f); beyond 4 per
    shape the least recently used graph is re-pointed (cudaGraphExecUpdate)
    instead of re-instantiated.  Six rotating buffer pairs, two rounds: every
    result is the reference's."""
    import torch
    op = make(64, 0.1, 1.0, 0.3)
    rng = np.random.default_rng(11)
    us = [torch.from_numpy(rng.standard_normal(64 ** 3)).cuda() for _ in range(6)]
    fs = [torch.empty(64 ** 3, dtype=torch.float64, device="cuda") for _ in range(6)]
    refs = [H.matvec(op, u.cpu().numpy()) for u in us]
    for _ in range(2):
        for u, f, ref in zip(us, fs, refs):
            H.matvec(op, u, out=f)
            assert rel(f.cpu().numpy(), ref) <= 1e-13


def test_host_vector_path_dense_plan_and_unpinned_rejected():
    """A dense-core plan takes the plain H2D / matvec / D2H route; the C ABI
    rejects pageable host pointers with a ValueError."""
    import ctypes
    import torch
    from paper_2508_05958_b200 import _lib
    cfg = H.BuildConfig(rank=6, leaf_side=8, rule=H.AdmissibilityRule.strong(1.0), kernel=H.inv_r_3d(),
                        coeff=H.CoefficientFn.constant(0.0))
    op = H.construct(cfg, H.UniformGrid(3, 32))
    u = np.random.default_rng(9).uniform(-1, 1, 32 ** 3)
    ref = H.matvec(op, torch.from_numpy(u).cuda()).cpu().numpy()
    got = H.matvec(op, torch.from_numpy(u).pin_memory())
    assert rel(got.numpy(), ref) <= 1e-14
    f = np.zeros_like(u)
    with pytest.raises(ValueError):
        _lib.check(_lib.lib().htlr_matvec_host(op._plan, ctypes.c_void_p(u.ctypes.data),
                                               ctypes.c_void_p(f.ctypes.data), 1, None))


@pytest.mark.parametrize("rule,eta", [("weak", None), ("strong", 2.0), ("strong", 0.7)])
def test_separable_other_admissibility(rule, eta):
    """Other admissibility rules change the offset sets and column lengths:
    the plan stays separable where the 4-bit offset codes fit (falling back to
    per-warp items when a column exceeds the cooperative layout) or keeps the
    dense cores; either way the oracle's rows are reproduced."""
    n = 32
    adm = H.AdmissibilityRule.weak() if rule == "weak" else H.AdmissibilityRule.strong(eta)
    cfg = H.BuildConfig(rank=8, leaf_side=8, rule=adm, kernel=H.gaussian(0.12), coeff=H.CoefficientFn.constant(0.3))
    op = H.construct(cfg, H.UniformGrid(3, n))
    print(rule, eta, op.formulation())
    U = np.random.default_rng(21).standard_normal((n ** 3, 2))
    F = H.matmat(op, U)
    pb = O.Problem(d=3, n=n, rank=8, leaf_side_max=8, kernel=O.Kernel("gaussian", sigma=0.12),
                   coeff=O.constant_coeff(0.3), rule=rule, eta=eta)
    rows = O.sampled_matvec(pb, U, BOXES[32])
    for i, bx in enumerate(BOXES[32]):
        assert rel(F[O.box_linear_indices(n, bx)], rows[i]) <= TOL


def test_separable_random_sweep():
    """Random separable-eligible problems (3-D Gaussian, p = leaf side = 8):
    grid size, admissibility rule and eta, sigma, kernel scale, coefficient
    and RHS count drawn at random; rows of random leaf boxes against the
    oracle.  (The weak rule once exposed a self-correction bug that the
    BASELINE configs could not.)"""
    rng = np.random.default_rng(2024)
    for case in range(8):
        n = int(rng.choice([16, 32, 32]))
        rule = str(rng.choice(["weak", "strong"]))
        eta = float(rng.choice([0.5, 0.7, 1.0, 1.5, 2.0, 3.0])) if rule == "strong" else None
        sig = float(rng.choice([0.05, 0.1, 0.3]))
        scale = float(rng.choice([1.0, 0.7]))
        a = float(rng.choice([0.0, 0.4]))
        R = int(rng.choice([1, 2, 3]))
        adm = H.AdmissibilityRule.weak() if rule == "weak" else H.AdmissibilityRule.strong(eta)
        cfg = H.BuildConfig(rank=8, leaf_side=8, rule=adm, kernel=H.gaussian(sig, scale=scale),
                            coeff=H.CoefficientFn.constant(a))
        op = H.construct(cfg, H.UniformGrid(3, n))
        U = rng.standard_normal((n ** 3, R))
        F = H.matmat(op, U)
        pb = O.Problem(d=3, n=n, rank=8, leaf_side_max=8, kernel=O.Kernel("gaussian", sigma=sig, scale=scale),
                       coeff=O.constant_coeff(a), rule=rule, eta=eta)
        m = n // 8
        boxes = []
        for _ in range(2):
            c = rng.integers(0, m, size=3)
            boxes.append(tuple((int(8 * q), int(8 * q + 8)) for q in c))
        rows = O.sampled_matvec(pb, U, boxes)
        for i, bx in enumerate(boxes):
            err = rel(F[O.box_linear_indices(n, bx)], rows[i])
            assert err <= TOL, (case, n, rule, eta, sig, scale, a, R, op.formulation(), err)


_BAND_SCRIPT = r"""
import sys
import numpy as np
import paper_2508_05958_b200 as H
n, R, a = int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4])
cfg = H.BuildConfig(rank=8, leaf_side=8, rule=H.AdmissibilityRule.strong(1.0), kernel=H.gaussian(0.1, scale=1.3),
                    coeff=H.CoefficientFn.constant(a))
op = H.construct(cfg, H.UniformGrid(3, n))
print(op.leaf_pass())
U = np.random.default_rng(n + R).standard_normal((n ** 3, R))
np.save(sys.argv[1], H.matmat(op, U))
"""


@pytest.mark.parametrize("n,R,a", [(64, 3, 0.25), (64, 1, 0.5), (128, 1, 0.0), (128, 2, 0.0)])
def test_banded_leaf_pass_equals_cooperative(tmp_path, n, R, a):
    """The banded passes (line sweeps over the box grid: C10^3 - C4^3 - C5^3
    + C2^3 (+ E5^3 - E2^3 at the leaf level), htlr_sep.cu; the leaf level and
    level 3) against the cooperative per-pair passes (HTLR_SEP_BAND=0), each
    in its own process: the same blocks summed in another order, so equal to
    rounding."""
    outs = {}
    for band in ("1", "0"):
        out = tmp_path / f"f{band}.npy"
        r = subprocess.run([sys.executable, "-c", _BAND_SCRIPT, str(out), str(n), str(R), str(a)], check=True,
                           cwd=ROOT, capture_output=True, text=True,
                           env={**os.environ, "PYTHONPATH": ROOT, "HTLR_SEP_BAND": band}, timeout=900)
        kind = r.stdout.strip().splitlines()[-1]
        # banded from 8 leaf boxes per axis on (n = 32 keeps the cooperative pass)
        assert kind == ("banded" if band == "1" and n >= 64 else "cooperative")
        outs[band] = np.load(out)
    err = rel(outs["1"], outs["0"])
    print(f"n={n} R={R} banded vs cooperative", err)
    assert err <= 1e-13


def test_banded_only_for_eta_one():
    """Other admissibility rules break the product-set structure: the plan's
    list check keeps the cooperative pass."""
    for rule in (H.AdmissibilityRule.strong(2.0), H.AdmissibilityRule.weak()):
        cfg = H.BuildConfig(rank=8, leaf_side=8, rule=rule, kernel=H.gaussian(0.1),
                            coeff=H.CoefficientFn.constant(0.0))
        op = H.construct(cfg, H.UniformGrid(3, 64))
        assert op.leaf_pass() != "banded"
    op = make(64)
    assert op.leaf_pass() == "banded"


@pytest.mark.parametrize("n,R,a", [(64, 2, 0.25), (128, 1, 0.0)])
def test_analytic_banded_plan_equals_listed_plan(tmp_path, n, R, a):
    """A plan whose banded levels were proven per offset (no pair lists below
    level 2, htlr_plan.cu analytic_bands_ok) against the plan that builds the
    lists and checks them pair by pair (HTLR_ANALYTIC=0): the same kernels on
    the same tables, equal up to the order of the upward pass's fp64 REDs."""
    outs = {}
    for mode in ("1", "0"):
        out = tmp_path / f"f{mode}.npy"
        r = subprocess.run([sys.executable, "-c", _BAND_SCRIPT, str(out), str(n), str(R), str(a)], check=True,
                           cwd=ROOT, capture_output=True, text=True,
                           env={**os.environ, "PYTHONPATH": ROOT, "HTLR_ANALYTIC": mode}, timeout=900)
        assert r.stdout.strip().splitlines()[-1] == "banded"
        outs[mode] = np.load(out)
    err = rel(outs["1"], outs["0"])
    print(f"n={n} R={R} analytic vs listed plan", err)
    assert err <= 1e-14


def test_banded_random_sweep_vs_oracle():
    """The banded path itself under random parameters: 3-D Gaussian, eta = 1,
    n = 64 (8 leaf boxes per axis: the leaf pass runs as banded sweeps over
    analytically built levels), sigma, kernel scale, coefficient and RHS
    count drawn at random; rows of random leaf boxes -- a corner box always
    among them, where every band is cut by the domain -- against the oracle,
    through the device path and through the host pipeline."""
    import torch
    rng = np.random.default_rng(77)
    n = 64
    for case in range(4):
        sig = float(rng.choice([0.04, 0.1, 0.25]))
        scale = float(rng.choice([1.0, 0.6]))
        a = float(rng.choice([0.0, 0.35]))
        R = int(rng.choice([1, 1, 2, 3]))
        cfg = H.BuildConfig(rank=8, leaf_side=8, rule=H.AdmissibilityRule.strong(1.0),
                            kernel=H.gaussian(sig, scale=scale), coeff=H.CoefficientFn.constant(a))
        op = H.construct(cfg, H.UniformGrid(3, n))
        assert op.leaf_pass() == "banded"
        U = rng.standard_normal((n ** 3, R))
        F = H.matmat(op, U)
        pb = O.Problem(d=3, n=n, rank=8, leaf_side_max=8, kernel=O.Kernel("gaussian", sigma=sig, scale=scale),
                       coeff=O.constant_coeff(a))
        corner = tuple((0, 8) if rng.integers(0, 2) else (n - 8, n) for _ in range(3))
        c = rng.integers(0, n // 8, size=3)
        boxes = [corner, tuple((int(8 * q), int(8 * q + 8)) for q in c)]
        rows = O.sampled_matvec(pb, U, boxes)
        for i, bx in enumerate(boxes):
            err = rel(F[O.box_linear_indices(n, bx)], rows[i])
            assert err <= TOL, (case, sig, scale, a, R, bx, err)
        # the same operator through pinned host vectors (the slab pipeline)
        Up = torch.from_numpy(U).pin_memory()
        Fp = H.matmat(op, Up).numpy()
        assert rel(Fp, F) <= 1e-13, (case, "host pipeline")


@pytest.mark.parametrize("n,R,a", [(64, 1, 0.5), (64, 3, 0.25), (128, 1, 0.0), (128, 2, 0.75)])
def test_direct_f_equals_downward_after_leaf_pass(n, R, a):
    """Unsharded banded matvec: by default the plane kernel and the cube
    downward pass both add their share into a zeroed f with fp64 REDs
    (htlr_matvec.cu mv_remote, "Direct f"), so the downward pass runs beside the
    leaf y-x sweep and Y is never written.  HTLR_FDIRECT=0 keeps Y and the
    downward pass after it.  0 + a + b has the same value in either order, so
    the two differ only through the upward pass's unordered REDs (and, with a
    coefficient, the a u term joining the expansion first instead of last):
    equal to rounding.  (Fresh vectors each time: graphs are keyed by the
    caller's vectors, so each call captures under its own setting.)"""
    import torch
    op = make(n, a=a)
    assert op.leaf_pass() == "banded"
    rng = np.random.default_rng(n + R)
    U = rng.standard_normal((n ** 3, R)) if R > 1 else rng.standard_normal(n ** 3)
    outs = {}
    old = os.environ.get("HTLR_FDIRECT")
    try:
        for mode in ("0", "1"):
            os.environ["HTLR_FDIRECT"] = mode
            u = torch.from_numpy(U).cuda()
            apply = H.matmat if R > 1 else H.matvec
            f = apply(op, u)
            f2 = apply(op, u)   # replay of the captured graph
            torch.cuda.synchronize()
            assert rel(f2.cpu().numpy(), f.cpu().numpy()) <= 1e-14
            outs[mode] = f.cpu().numpy()
    finally:
        if old is None:
            os.environ.pop("HTLR_FDIRECT", None)
        else:
            os.environ["HTLR_FDIRECT"] = old
    assert rel(outs["1"], outs["0"]) <= 1e-14
    # and against the oracle's rows of corner, edge and interior leaf boxes
    if n == 64:
        U2 = U.reshape(n ** 3, -1)
        rows = O.sampled_matvec(problem(n, a=a), U2, BOXES[64])
        F = outs["1"].reshape(n ** 3, -1)
        for i, bx in enumerate(BOXES[64]):
            assert rel(F[O.box_linear_indices(n, bx)], rows[i]) <= TOL
