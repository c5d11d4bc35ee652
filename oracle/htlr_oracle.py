"""CPU oracle for the HTLR hot path.  TEST INFRASTRUCTURE ONLY.

This module is the parity checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and the
``--impl reference`` arm) may import it.  The product package
``paper_2508_05958_b200`` never imports anything under ``oracle/``.

It restates, in plain numpy, the algorithm of the reference package ``htlr``
(``/root/reference/pkg/src/htlr``) on the hot path named by BASELINE.json:
cluster tree + block cluster tree (``grids.py``), kernel evaluation and the
diagonal cell quadrature (``kernels.py``), Chebyshev nodes / Lagrange factors /
kernel cores (``chebyshev.py``), Tucker and dense leaf payloads
(``blocks.py``), and the leaf-by-leaf matvec (``operators.py``).  Every
function cites the reference lines it follows.

Parity pin: ``tests/golden/make_golden.py`` imports the reference itself (in
the build container, where ``/root/reference`` exists) and writes the
fixtures under ``tests/golden/``; ``tests/test_oracle_golden.py`` checks this
restatement against every fixture (lists bit-exact, diagonal constants and
matvec results to rounding).  The reference computes with numpy/OpenBLAS
(unvendored, pinned only as ``numpy>=1.24``, ``scipy>=1.10`` in
``pkg/pyproject.toml:10-13``); the fixtures were produced with numpy 2.3.5.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

ADM = 0     # grids.py:377 ADMISSIBLE
NEAR = 1    # grids.py:378 INADMISSIBLE

# --------------------------------------------------------------------------
# kernels (kernels.py:33-117).  `scale` multiplies the reference formula; the
# BASELINE.json kernels are -log r = 2*pi*slp2d, 1/r = 4*pi*slp3d and
# exp(-r^2/s^2) = gaussian(s/sqrt(2)).
# --------------------------------------------------------------------------


@dataclass(frozen=True)
class Kernel:
    kind: str                      # "gaussian" | "slp2d" | "slp3d"
    sigma: float = 0.0
    scale: float = 1.0

    @property
    def smooth_at_diagonal(self) -> bool:      # kernels.py:50-70
        return self.kind == "gaussian"


def kernel_values(k: Kernel, x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """k(x, y) over broadcast point arrays with a trailing coordinate axis
    (kernels.py:88-103)."""
    diff = x - y
    r2 = np.sum(diff * diff, axis=-1)
    if k.kind == "gaussian":
        out = np.exp(-r2 / (2.0 * k.sigma * k.sigma))
    elif k.kind == "slp2d":
        if np.any(r2 == 0.0):
            raise ValueError("SLP kernel evaluated on the diagonal")
        out = -0.5 * np.log(r2) / (2.0 * np.pi)
    elif k.kind == "slp3d":
        r = np.sqrt(r2)
        if np.any(r == 0.0):
            raise ValueError("SLP kernel evaluated on the diagonal")
        out = 1.0 / (4.0 * np.pi * r)
    else:
        raise ValueError(f"unknown kernel kind {k.kind!r}")
    return out if k.scale == 1.0 else k.scale * out


def kernel_pairs(k: Kernel, xs: np.ndarray, ys: np.ndarray) -> np.ndarray:
    """(m1, d) x (m2, d) -> (m1, m2) (kernels.py:113-117)."""
    return kernel_values(k, xs[:, None, :], ys[None, :, :])


def kernel_pairs_self(k: Kernel, pts: np.ndarray, diag: np.ndarray) -> np.ndarray:
    """Square block of a point set with itself; coincident pairs are kept off
    the singular formula (r^2 := 1) and then overwritten by `diag`
    (kernels.py:120-149)."""
    diff = pts[:, None, :] - pts[None, :, :]
    r2 = np.sum(diff * diff, axis=-1)
    idx = np.arange(len(pts))
    if k.kind == "gaussian":
        out = np.exp(-r2 / (2.0 * k.sigma * k.sigma))
    else:
        r2[idx, idx] = 1.0
        if k.kind == "slp2d":
            out = -0.5 * np.log(r2) / (2.0 * np.pi)
        else:
            out = 1.0 / (4.0 * np.pi * np.sqrt(r2))
    if k.scale != 1.0:
        out = k.scale * out
    out[idx, idx] = diag
    return out


# -- diagonal cell average (kernels.py:195-265) -----------------------------

GRADING = 3   # kernels.py:28 RADIAL_GRADING


def _gl01(q: int):
    """Gauss-Legendre rule mapped to [0, 1] (kernels.py:195-198)."""
    x, w = np.polynomial.legendre.leggauss(q)
    return 0.5 * (x + 1.0), 0.5 * w


def _tensor_weights(ws: Sequence[np.ndarray]) -> np.ndarray:
    """Outer product of per-axis weights in 'ij' order (kernels.py:200-207)."""
    out = np.ones([len(w) for w in ws])
    for ax, w in enumerate(ws):
        shape = [1] * len(ws)
        shape[ax] = len(w)
        out = out * w.reshape(shape)
    return out


def cell_average(k: Kernel, d: int, h: float, q: int = 10,
                 corner_subdivision: bool = True) -> float:
    """Average of k(0, .) over the width-h cell centred at the origin
    (translation-invariant kernels, kernels.py:252-265 with center := 0)."""
    if h <= 0:
        raise ValueError("cell width must be positive")
    center = np.zeros(d)
    gx, gw = _gl01(q)
    if k.smooth_at_diagonal or not corner_subdivision:
        # kernels.py:210-219: plain tensor rule over the cell
        axes = [center[a] - h / 2 + h * gx for a in range(d)]
        mesh = np.meshgrid(*axes, indexing="ij")
        w = _tensor_weights([h * gw] * d)
        pts = np.stack([m.ravel() for m in mesh], axis=-1)
        vals = kernel_values(k, np.broadcast_to(center, pts.shape), pts)
        return float(np.sum(vals * w.ravel())) / h ** d
    # kernels.py:222-249: 2^d corner sub-cells x d Duffy pyramids, cubic
    # radial grading toward the singular centre
    half = h / 2.0
    rad = gx ** GRADING
    rad_w = GRADING * gx ** (GRADING - 1) * gw
    total = 0.0
    for corner in np.ndindex(*([2] * d)):
        sgn = np.array([1.0 if c else -1.0 for c in corner])
        for axis in range(d):
            nodes = [rad if a == axis else gx for a in range(d)]
            mesh = np.meshgrid(*nodes, indexing="ij")
            w = _tensor_weights([rad_w if a == axis else gw for a in range(d)])
            t = mesh[axis]
            z = np.empty(t.shape + (d,))
            for a in range(d):
                z[..., a] = half * t if a == axis else half * t * mesh[a]
            pts = (center + sgn * z).reshape(-1, d)
            jac = half ** d * t ** (d - 1)
            vals = kernel_values(k, np.broadcast_to(center, pts.shape), pts)
            total += float(np.sum(vals * (jac * w).ravel()))
    return total / h ** d


# --------------------------------------------------------------------------
# grid, cluster tree, block cluster tree (grids.py:18-296)
# --------------------------------------------------------------------------

Ranges = tuple  # tuple of (lo, hi) per dimension, half-open, 0-based


def grid_points(n: int, ranges: Ranges) -> np.ndarray:
    """Cell-centred points (i + 1/2) h of an index box, first index fastest
    (grids.py:39-50)."""
    h = 1.0 / n
    axes = [(np.arange(lo, hi) + 0.5) * h for lo, hi in ranges]
    mesh = np.meshgrid(*axes, indexing="ij")
    return np.stack([m.ravel(order="F") for m in mesh], axis=-1)


def box_linear_indices(n: int, ranges: Ranges) -> np.ndarray:
    """F-order global ids of the points of an index box (grids.py:82-92)."""
    mesh = np.meshgrid(*[np.arange(lo, hi, dtype=np.int64) for lo, hi in ranges], indexing="ij")
    lin = np.zeros_like(mesh[0])
    stride = 1
    for m in mesh:
        lin = lin + m * stride
        stride *= n
    return lin.ravel(order="F")


def leaf_side(n: int, leaf_side_max: int) -> int:
    """Exact repeated halving down to the threshold (grids.py:196-207)."""
    if leaf_side_max < 1:
        raise ValueError("leaf threshold must be positive")
    side = n
    while side > leaf_side_max:
        if side % 2:
            raise ValueError(f"grid side {n} cannot be halved evenly down to "
                             f"the leaf threshold {leaf_side_max}")
        side //= 2
    return side


@dataclass
class Cluster:
    ranges: Ranges
    level: int
    kids: list = field(default_factory=list)


def cluster_tree(n: int, d: int, leaf_side_max: int) -> Cluster:
    """Midpoint 2^d split, children in ndindex order (last dim fastest),
    leaf iff max side <= threshold (grids.py:210-234)."""
    leaf_side(n, leaf_side_max)

    def grow(ranges: Ranges, level: int) -> Cluster:
        node = Cluster(ranges, level)
        if max(hi - lo for lo, hi in ranges) <= leaf_side_max:
            return node
        halves = [((lo, (lo + hi) // 2), ((lo + hi) // 2, hi)) for lo, hi in ranges]
        for combo in np.ndindex(*([2] * d)):
            node.kids.append(grow(tuple(halves[a][combo[a]] for a in range(d)), level + 1))
        return node

    return grow(tuple((0, n) for _ in range(d)), 0)


def domain(n: int, ranges: Ranges):
    """Real box covered by the cells (grids.py:237-242): (lo*h, hi*h)."""
    h = 1.0 / n
    return tuple((lo * h, hi * h) for lo, hi in ranges)


def admissible(rule: str, eta: Optional[float], dt, ds) -> bool:
    """Weak: zero-volume overlap; strong: diam^2 <= eta^2 dist^2 (1+1e-12),
    evaluated in the reference's operation order (grids.py:110-127,153-165)."""
    if rule == "weak":
        return _overlap_volume(dt, ds) == 0.0
    dist = 0.0
    for (a1, b1), (a2, b2) in zip(dt, ds):
        gap = max(a1 - b2, a2 - b1, 0.0)
        dist += gap * gap
    diam_t = 0
    for a, b in dt:
        diam_t = diam_t + (b - a) ** 2
    diam_s = 0
    for a, b in ds:
        diam_s = diam_s + (b - a) ** 2
    diam = max(float(diam_t), float(diam_s))
    return diam <= eta * eta * dist * (1.0 + 1e-12)


@dataclass
class Leaf:
    leaf_id: int
    kind: int
    level: int
    tau: Ranges
    sigma: Ranges


def block_leaves(n: int, d: int, leaf_side_max: int, rule: str = "strong",
                 eta: Optional[float] = 1.0) -> list:
    """DFS leaf list of the block cluster tree: admissible first, then
    leaf-leaf -> dense, else recurse sigma-children outer / tau-children
    inner; leaf_id in creation order (grids.py:268-296)."""
    root = cluster_tree(n, d, leaf_side_max)
    out: list = []

    def visit(t: Cluster, s: Cluster, level: int):
        if admissible(rule, eta, domain(n, t.ranges), domain(n, s.ranges)):
            out.append(Leaf(len(out), ADM, level, t.ranges, s.ranges))
            return
        if not t.kids or not s.kids:
            assert not t.kids and not s.kids
            out.append(Leaf(len(out), NEAR, level, t.ranges, s.ranges))
            return
        for sk in s.kids:
            for tk in t.kids:
                visit(tk, sk, level + 1)

    import sys
    sys.setrecursionlimit(max(10000, sys.getrecursionlimit()))
    visit(root, root, 0)
    return out


def leaves_to_array(leaves: list, d: int) -> np.ndarray:
    """Leaf list as int64 rows: leaf_id, kind, level, tau lo/hi per dim,
    sigma lo/hi per dim (the export format of htlr_export_lists)."""
    arr = np.empty((len(leaves), 3 + 4 * d), dtype=np.int64)
    for i, lf in enumerate(leaves):
        arr[i, 0] = lf.leaf_id
        arr[i, 1] = lf.kind
        arr[i, 2] = lf.level
        arr[i, 3:3 + 2 * d] = np.asarray(lf.tau, dtype=np.int64).ravel()
        arr[i, 3 + 2 * d:] = np.asarray(lf.sigma, dtype=np.int64).ravel()
    return arr


# --------------------------------------------------------------------------
# Chebyshev interpolation (chebyshev.py:31-85)
# --------------------------------------------------------------------------


def cheb_nodes(lo: float, hi: float, p: int) -> np.ndarray:
    """First-kind nodes in decreasing order (chebyshev.py:31-38)."""
    t = np.arange(1, p + 1)
    return 0.5 * (hi - lo) * np.cos((2 * t - 1) * np.pi / (2 * p)) + 0.5 * (hi + lo)


def lagrange_matrix(x: np.ndarray, nodes: np.ndarray) -> np.ndarray:
    """L[i, t] = prod_{j != t} (x_i - xi_j) / (xi_t - xi_j), product taken in
    ascending j (chebyshev.py:52-66)."""
    p = len(nodes)
    out = np.empty((len(x), p))
    for t in range(p):
        others = np.array([j for j in range(p) if j != t], dtype=np.int64)
        out[:, t] = np.prod((x[:, None] - nodes[None, others]) / (nodes[t] - nodes[others]), axis=1)
    return out


def kernel_core(k: Kernel, nodes_t: Sequence[np.ndarray], nodes_s: Sequence[np.ndarray]) -> np.ndarray:
    """k at all tensor node pairs, order-2d tensor with target modes first
    (chebyshev.py:69-85)."""
    def tensor_pts(nodes):
        mesh = np.meshgrid(*nodes, indexing="ij")
        return np.stack([m.ravel(order="F") for m in mesh], axis=-1)
    vals = kernel_pairs(k, tensor_pts(nodes_t), tensor_pts(nodes_s))
    shape = tuple(len(a) for a in nodes_t) + tuple(len(a) for a in nodes_s)
    return vals.ravel(order="F").reshape(shape, order="F")


# --------------------------------------------------------------------------
# tensor helpers (tensor.py:35-132)
# --------------------------------------------------------------------------


def mode_mul(t: np.ndarray, m: np.ndarray, mode: int) -> np.ndarray:
    """Contract axis `mode` (1-based) of t with the columns of m
    (tensor.py:35-52)."""
    moved = np.moveaxis(t, mode - 1, 0)
    out = np.tensordot(m, moved, axes=([1], [0]))
    return np.moveaxis(out, 0, mode - 1)


# --------------------------------------------------------------------------
# leaf payloads (blocks.py:89-227) and their application (blocks.py:230-286)
# --------------------------------------------------------------------------


@dataclass
class Tucker:
    core: np.ndarray
    ufac: list     # per-dim (s x p) orthonormal factor or None (square)
    vfac: list


def tucker_block(k: Kernel, n: int, tau: Ranges, sigma: Ranges, p: int) -> Tucker:
    """Interpolate over the box pair, QR every non-square factor, fold h^d and
    the triangular factors (raw factor when square) into the core in the
    interleaved order u1, v1, u2, v2, ... (blocks.py:89-106,126-164)."""
    d = len(tau)
    h = 1.0 / n
    dt, ds = domain(n, tau), domain(n, sigma)
    if _overlap_volume(dt, ds) > 0.0:
        raise ValueError("interpolation blocks require disjoint domains")
    nt = [cheb_nodes(lo, hi, p) for lo, hi in dt]
    ns = [cheb_nodes(lo, hi, p) for lo, hi in ds]
    raw_u = [lagrange_matrix((np.arange(*tau[a]) + 0.5) * h, nt[a]) for a in range(d)]
    raw_v = [lagrange_matrix((np.arange(*sigma[a]) + 0.5) * h, ns[a]) for a in range(d)]
    core = h ** d * kernel_core(k, nt, ns)
    ufac, vfac = [], []
    for a in range(d):
        for raw, facs, mode in ((raw_u[a], ufac, a + 1), (raw_v[a], vfac, d + a + 1)):
            if raw.shape[0] < raw.shape[1]:
                raise ValueError(f"qr requires rows >= cols, got shape {raw.shape}")
            if raw.shape[0] == raw.shape[1]:
                facs.append(None)
                core = mode_mul(core, raw, mode)
            else:
                q, r = np.linalg.qr(raw, mode="reduced")
                facs.append(q)
                core = mode_mul(core, r, mode)
    return Tucker(core, ufac, vfac)


def _overlap_volume(dt, ds) -> float:
    vol = 1.0
    for (a1, b1), (a2, b2) in zip(dt, ds):
        length = min(b1, b2) - max(a1, a2)
        if length <= 0.0:
            return 0.0
        vol *= length
    return vol


def dense_block(k: Kernel, coeff: Callable[[np.ndarray], np.ndarray], n: int,
                tau: Ranges, sigma: Ranges, diag: float) -> np.ndarray:
    """a(x_i) 1[i=j] + K_ij h^d; the tau == sigma diagonal is the cached cell
    average (blocks.py:190-227, operators.py:95-99)."""
    d = len(tau)
    h = 1.0 / n
    xs = grid_points(n, tau)
    ys = grid_points(n, sigma)
    if tau == sigma:
        mat = kernel_pairs_self(k, xs, np.full(len(xs), diag)) * h ** d
        idx = np.arange(len(xs))
        mat[idx, idx] += np.asarray(coeff(xs), dtype=np.float64)
        return mat
    return kernel_pairs(k, xs, ys) * h ** d


def tucker_apply(b: Tucker, seg: np.ndarray) -> np.ndarray:
    """V^T mode products, core contraction over the source modes, U mode
    products (blocks.py:230-259)."""
    d = len(b.ufac)
    core_shape = b.core.shape
    cols = tuple(f.shape[0] if f is not None else core_shape[d + a] for a, f in enumerate(b.vfac))
    w = np.reshape(seg, cols, order="F")
    for a, f in enumerate(b.vfac):
        if f is not None:
            w = mode_mul(w, f.T, a + 1)
    hvec = np.tensordot(b.core, w, axes=(list(range(d, 2 * d)), list(range(d))))
    for a, f in enumerate(b.ufac):
        if f is not None:
            hvec = mode_mul(hvec, f, a + 1)
    return hvec.ravel(order="F")


def materialize_tucker(b: Tucker) -> np.ndarray:
    """Full matrix of a Tucker block (blocks.py:267-286)."""
    d = len(b.ufac)
    full = b.core
    for a, f in enumerate(b.ufac):
        if f is not None:
            full = mode_mul(full, f, a + 1)
    for a, f in enumerate(b.vfac):
        if f is not None:
            full = mode_mul(full, f, d + a + 1)
    rows = int(np.prod(full.shape[:d]))
    return full.reshape(rows, -1, order="F")


# --------------------------------------------------------------------------
# operator + matvec (operators.py:95-161)
# --------------------------------------------------------------------------


@dataclass
class Problem:
    d: int
    n: int
    rank: int
    leaf_side_max: int
    kernel: Kernel
    coeff: Callable[[np.ndarray], np.ndarray]
    rule: str = "strong"
    eta: Optional[float] = 1.0
    q: int = 10

    @property
    def h(self) -> float:
        return 1.0 / self.n

    @property
    def num_points(self) -> int:
        return self.n ** self.d

    def diag(self) -> float:
        """operators.py:95-99 (cell centred at the origin: translation-invariant)."""
        return cell_average(self.kernel, self.d, self.h, self.q)


def constant_coeff(c: float):
    return lambda pts: np.full(len(pts), float(c))


def build_payload(pb: Problem, leaf: Leaf, diag: float):
    if leaf.kind == ADM:
        return tucker_block(pb.kernel, pb.n, leaf.tau, leaf.sigma, pb.rank)
    return dense_block(pb.kernel, pb.coeff, pb.n, leaf.tau, leaf.sigma, diag)


def apply_payload(payload, seg: np.ndarray) -> np.ndarray:
    if isinstance(payload, Tucker):
        return tucker_apply(payload, seg)
    return payload @ seg


def _slices(ranges: Ranges):
    return tuple(slice(lo, hi) for lo, hi in ranges)


def matvec(pb: Problem, u: np.ndarray, leaves: Optional[list] = None,
           payloads: Optional[list] = None) -> np.ndarray:
    """f = A u accumulated leaf by leaf in DFS order (operators.py:138-161).
    `u` may be (N,) or (N, R); columns are independent right-hand sides."""
    u = np.asarray(u, dtype=np.float64)
    cols = u.reshape(pb.num_points, -1)
    if cols.shape[0] != pb.num_points:
        raise ValueError("vector length mismatch")
    if leaves is None:
        leaves = block_leaves(pb.n, pb.d, pb.leaf_side_max, pb.rule, pb.eta)
    diag = pb.diag()
    shape = (pb.n,) * pb.d
    out = np.zeros_like(cols)
    for r in range(cols.shape[1]):
        ut = cols[:, r].reshape(shape, order="F")
        ft = np.zeros(shape)
        for lf in leaves:
            pl = payloads[lf.leaf_id] if payloads is not None else build_payload(pb, lf, diag)
            seg = ut[_slices(lf.sigma)].ravel(order="F")
            res = apply_payload(pl, seg)
            ft[_slices(lf.tau)] += res.reshape([hi - lo for lo, hi in lf.tau], order="F")
        out[:, r] = ft.ravel(order="F")
    return out.reshape(u.shape)


def _contains(outer: Ranges, inner: Ranges) -> bool:
    return all(lo_o <= lo_i and hi_i <= hi_o for (lo_o, hi_o), (lo_i, hi_i) in zip(outer, inner))


def sampled_matvec(pb: Problem, u: np.ndarray, targets: Sequence[Ranges],
                   leaves: Optional[list] = None) -> np.ndarray:
    """Rows of f = A u on the given leaf target boxes only: iterate the DFS
    leaves, keep those whose tau contains a target box, build and apply them
    exactly as operators.py:146-155 does.  Accumulation per row follows the
    same DFS order as the full matvec, so the sampled rows equal the full
    reference matvec's rows bit for bit.  Returns an array
    (len(targets), box points, R)."""
    u = np.asarray(u, dtype=np.float64)
    cols = u.reshape(pb.num_points, -1)
    if leaves is None:
        leaves = block_leaves(pb.n, pb.d, pb.leaf_side_max, pb.rule, pb.eta)
    diag = pb.diag()
    shape = (pb.n,) * pb.d
    R = cols.shape[1]
    uts = [cols[:, r].reshape(shape, order="F") for r in range(R)]
    acc = {}
    for lf in leaves:
        hit = [i for i, tb in enumerate(targets) if _contains(lf.tau, tb)]
        if not hit:
            continue
        pl = build_payload(pb, lf, diag)
        tsz = [hi - lo for lo, hi in lf.tau]
        for r in range(R):
            seg = uts[r][_slices(lf.sigma)].ravel(order="F")
            res = apply_payload(pl, seg).reshape(tsz, order="F")
            for i in hit:
                sub = tuple(slice(lo - tlo, hi - tlo) for (lo, hi), (tlo, _) in zip(targets[i], lf.tau))
                key = (i, r)
                if key not in acc:
                    acc[key] = np.zeros([hi - lo for lo, hi in targets[i]])
                acc[key] += res[sub]
    npts = int(np.prod([hi - lo for lo, hi in targets[0]]))
    out = np.zeros((len(targets), npts, R))
    for (i, r), v in acc.items():
        out[i, :, r] = v.ravel(order="F")
    return out


def storage_counts(pb: Problem, leaves: list) -> dict:
    """Scalar counts by category for the reference's per-leaf storage
    (blocks.py:289-299, operators.py:175-197)."""
    p, d = pb.rank, pb.d
    dense = factors = cores = 0
    for lf in leaves:
        nt = int(np.prod([hi - lo for lo, hi in lf.tau]))
        ns = int(np.prod([hi - lo for lo, hi in lf.sigma]))
        if lf.kind == NEAR:
            dense += nt * ns
            continue
        cores += p ** (2 * d)
        for lo, hi in lf.tau + lf.sigma:
            if hi - lo != p:
                factors += (hi - lo) * p
    return {"dense": dense, "factors": factors, "cores": cores,
            "total": dense + factors + cores}


# --------------------------------------------------------------------------
# BASELINE config 5: mapped quasi-uniform tensor grid.  The reference cannot
# represent it (UniformGrid only, grids.py:18-43), so this restatement is the
# oracle (parity UNPINNED by the reference; pinned instead by the
# amplitude-0 limit, which reproduces the reference's uniform results, and by
# dense-vs-HTLR agreement).  It follows the reference's algorithm with the
# mapped geometry substituted:
#   points x_i = phi((i + 1/2)/n), cell [phi(i/n), phi((i+1)/n)], weight
#   w_i = prod_a (cell width)  (grids.py:39-50, 237-242 with phi applied);
#   domain boxes from the cell boundaries; Chebyshev nodes on the mapped
#   intervals (chebyshev.py:31-85); Tucker blocks as blocks.py:126-164 with the
#   source weights folded into the source factors instead of h^d;
#   dense blocks K_ij w_j with the diagonal = integral of k(x_i, .) over the
#   (off-centre, rectangular) cell: kernels.py:222-249 generalised to 2^d
#   rectangular corner boxes.
# phi(t) = t + A sin(2 pi t) / (2 pi)  (BASELINE.json configs[4]).
# --------------------------------------------------------------------------


@dataclass(frozen=True)
class MappedGeometry:
    n: int
    amplitude: float = 0.05

    def phi(self, t: float) -> float:
        return t + self.amplitude * math.sin(2 * math.pi * t) / (2 * math.pi)

    def boundaries(self) -> np.ndarray:
        return np.array([self.phi(i / self.n) for i in range(self.n + 1)])

    def coords(self) -> np.ndarray:
        return np.array([self.phi((i + 0.5) / self.n) for i in range(self.n)])

    def widths(self) -> np.ndarray:
        b = self.boundaries()
        return b[1:] - b[:-1]


def mapped_points(geo: MappedGeometry, ranges: Ranges) -> np.ndarray:
    x = geo.coords()
    mesh = np.meshgrid(*[x[lo:hi] for lo, hi in ranges], indexing="ij")
    return np.stack([m.ravel(order="F") for m in mesh], axis=-1)


def mapped_weights(geo: MappedGeometry, ranges: Ranges) -> np.ndarray:
    c = geo.widths()
    w = np.ones(1)
    for lo, hi in ranges:    # F-order tensor product: first index fastest
        w = np.outer(c[lo:hi], w).ravel()
    return w


def mapped_domain(geo: MappedGeometry, ranges: Ranges):
    b = geo.boundaries()
    return tuple((b[lo], b[hi]) for lo, hi in ranges)


def mapped_block_leaves(geo: MappedGeometry, d: int, leaf_side_max: int, rule: str = "strong",
                        eta: Optional[float] = 1.0) -> list:
    """grids.py:268-296 on the mapped domains."""
    root = cluster_tree(geo.n, d, leaf_side_max)
    out: list = []

    def visit(t: Cluster, s: Cluster, level: int):
        if admissible(rule, eta, mapped_domain(geo, t.ranges), mapped_domain(geo, s.ranges)):
            out.append(Leaf(len(out), ADM, level, t.ranges, s.ranges))
            return
        if not t.kids or not s.kids:
            out.append(Leaf(len(out), NEAR, level, t.ranges, s.ranges))
            return
        for sk in s.kids:
            for tk in t.kids:
                visit(tk, sk, level + 1)

    visit(root, root, 0)
    return out


def mapped_tucker_block(k: Kernel, geo: MappedGeometry, tau: Ranges, sigma: Ranges, p: int) -> Tucker:
    d = len(tau)
    x = geo.coords()
    c = geo.widths()
    dt, ds = mapped_domain(geo, tau), mapped_domain(geo, sigma)
    if _overlap_volume(dt, ds) > 0.0:
        raise ValueError("interpolation blocks require disjoint domains")
    nt = [cheb_nodes(lo, hi, p) for lo, hi in dt]
    ns = [cheb_nodes(lo, hi, p) for lo, hi in ds]
    raw_u = [lagrange_matrix(x[tau[a][0]:tau[a][1]], nt[a]) for a in range(d)]
    raw_v = [c[sigma[a][0]:sigma[a][1], None] * lagrange_matrix(x[sigma[a][0]:sigma[a][1]], ns[a])
             for a in range(d)]
    core = kernel_core(k, nt, ns)
    ufac, vfac = [], []
    for a in range(d):
        for raw, facs, mode in ((raw_u[a], ufac, a + 1), (raw_v[a], vfac, d + a + 1)):
            if raw.shape[0] < raw.shape[1]:
                raise ValueError(f"qr requires rows >= cols, got shape {raw.shape}")
            if raw.shape[0] == raw.shape[1]:
                facs.append(None)
                core = mode_mul(core, raw, mode)
            else:
                q, r = np.linalg.qr(raw, mode="reduced")
                facs.append(q)
                core = mode_mul(core, r, mode)
    return Tucker(core, ufac, vfac)


def mapped_cell_integrals(k: Kernel, geo: MappedGeometry, idx: np.ndarray, q: int = 10) -> np.ndarray:
    """Integral of k(x_i, .) over the rectangular cell of each point (rows of
    the multi-index array `idx`), split at x_i into 2^d corner boxes, each
    integrated with the d-pyramid Duffy rule and cubic radial grading of
    kernels.py:222-249 (there: equal corner boxes of side h/2)."""
    idx = np.atleast_2d(np.asarray(idx, dtype=np.int64))
    npts, d = idx.shape
    b = geo.boundaries()
    x = geo.coords()
    gx, gw = _gl01(q)
    rad = gx ** GRADING
    rad_w = GRADING * gx ** (GRADING - 1) * gw
    total = np.zeros(npts)
    for corner in np.ndindex(*([2] * d)):
        ext = np.stack([(b[idx[:, a] + 1] - x[idx[:, a]]) if corner[a] else (x[idx[:, a]] - b[idx[:, a]])
                        for a in range(d)], axis=-1)                       # (npts, d)
        for axis in range(d):
            nodes = [rad if a == axis else gx for a in range(d)]
            mesh = np.meshgrid(*nodes, indexing="ij")
            w = _tensor_weights([rad_w if a == axis else gw for a in range(d)]).ravel()
            t = mesh[axis].ravel()
            unit = np.stack([t if a == axis else t * mesh[a].ravel() for a in range(d)], axis=-1)   # (m, d)
            pts = ext[:, None, :] * unit[None, :, :]                          # (npts, m, d)
            jac = np.prod(ext, axis=1)[:, None] * t[None, :] ** (d - 1)
            vals = kernel_values(k, np.zeros_like(pts), pts)
            total += np.sum(vals * (jac * w[None, :]), axis=1)
    return total


def mapped_cell_integral(k: Kernel, geo: MappedGeometry, idx, q: int = 10) -> float:
    return float(mapped_cell_integrals(k, geo, np.asarray([idx]), q)[0])


def mapped_dense_block(k: Kernel, coeff, geo: MappedGeometry, tau: Ranges, sigma: Ranges,
                       q: int = 10) -> np.ndarray:
    xs = mapped_points(geo, tau)
    ys = mapped_points(geo, sigma)
    w = mapped_weights(geo, sigma)
    if tau == sigma:
        d = len(tau)
        diag = mapped_cell_integrals(k, geo, np.asarray(_box_multi_indices(tau)), q)
        mat = kernel_pairs_self(k, xs, np.zeros(len(xs))) * w[None, :]
        i = np.arange(len(xs))
        mat[i, i] = diag + np.asarray(coeff(xs), dtype=np.float64)
        return mat
    return kernel_pairs(k, xs, ys) * w[None, :]


def _box_multi_indices(ranges: Ranges):
    """Multi-indices of a box in F-order (first index fastest)."""
    mesh = np.meshgrid(*[np.arange(lo, hi) for lo, hi in ranges], indexing="ij")
    return list(zip(*[m.ravel(order="F") for m in mesh]))


@dataclass
class MappedProblem:
    d: int
    geo: MappedGeometry
    rank: int
    leaf_side_max: int
    kernel: Kernel
    coeff: Callable[[np.ndarray], np.ndarray]
    rule: str = "strong"
    eta: Optional[float] = 1.0
    q: int = 10

    @property
    def n(self) -> int:
        return self.geo.n

    @property
    def num_points(self) -> int:
        return self.geo.n ** self.d


def mapped_matvec(pb: MappedProblem, u: np.ndarray, leaves: Optional[list] = None) -> np.ndarray:
    """Leaf-by-leaf matvec on the mapped grid (operators.py:138-161)."""
    u = np.asarray(u, dtype=np.float64)
    cols = u.reshape(pb.num_points, -1)
    if leaves is None:
        leaves = mapped_block_leaves(pb.geo, pb.d, pb.leaf_side_max, pb.rule, pb.eta)
    shape = (pb.n,) * pb.d
    out = np.zeros_like(cols)
    payloads = []
    for lf in leaves:
        if lf.kind == ADM:
            payloads.append(mapped_tucker_block(pb.kernel, pb.geo, lf.tau, lf.sigma, pb.rank))
        else:
            payloads.append(mapped_dense_block(pb.kernel, pb.coeff, pb.geo, lf.tau, lf.sigma, pb.q))
    for r in range(cols.shape[1]):
        ut = cols[:, r].reshape(shape, order="F")
        ft = np.zeros(shape)
        for lf, pl in zip(leaves, payloads):
            seg = ut[_slices(lf.sigma)].ravel(order="F")
            res = apply_payload(pl, seg)
            ft[_slices(lf.tau)] += res.reshape([hi - lo for lo, hi in lf.tau], order="F")
        out[:, r] = ft.ravel(order="F")
    return out.reshape(u.shape)


def mapped_sampled_matvec(pb: MappedProblem, u: np.ndarray, targets: Sequence[Ranges],
                          leaves: Optional[list] = None) -> np.ndarray:
    """`sampled_matvec` on the mapped grid: rows of the target leaf boxes
    only, from the leaves whose tau contains one, in DFS order (the same
    restriction of operators.py:146-155).  Returns (len(targets), points, R)."""
    u = np.asarray(u, dtype=np.float64)
    cols = u.reshape(pb.num_points, -1)
    if leaves is None:
        leaves = mapped_block_leaves(pb.geo, pb.d, pb.leaf_side_max, pb.rule, pb.eta)
    shape = (pb.n,) * pb.d
    R = cols.shape[1]
    uts = [cols[:, r].reshape(shape, order="F") for r in range(R)]
    acc = {}
    for lf in leaves:
        hit = [i for i, tb in enumerate(targets) if _contains(lf.tau, tb)]
        if not hit:
            continue
        if lf.kind == ADM:
            pl = mapped_tucker_block(pb.kernel, pb.geo, lf.tau, lf.sigma, pb.rank)
        else:
            pl = mapped_dense_block(pb.kernel, pb.coeff, pb.geo, lf.tau, lf.sigma, pb.q)
        tsz = [hi - lo for lo, hi in lf.tau]
        for r in range(R):
            res = apply_payload(pl, uts[r][_slices(lf.sigma)].ravel(order="F")).reshape(tsz, order="F")
            for i in hit:
                sub = tuple(slice(lo - tlo, hi - tlo) for (lo, hi), (tlo, _) in zip(targets[i], lf.tau))
                acc.setdefault((i, r), np.zeros([hi - lo for lo, hi in targets[i]]))
                acc[(i, r)] += res[sub]
    npts = int(np.prod([hi - lo for lo, hi in targets[0]]))
    out = np.zeros((len(targets), npts, R))
    for (i, r), v in acc.items():
        out[i, :, r] = v.ravel(order="F")
    return out


def mapped_dense_matrix(pb: MappedProblem) -> np.ndarray:
    """Full Nystrom matrix on the mapped grid (small n; exactness check of the
    compressed operator)."""
    full = tuple((0, pb.n) for _ in range(pb.d))
    return mapped_dense_block(pb.kernel, pb.coeff, pb.geo, full, full, pb.q)


# --------------------------------------------------------------------------
# The reference's matvec *call structure*, operation for operation -- what the
# `bench.py --impl reference` arm times (the reference is pure Python and
# cannot travel to the GPU box).  `tucker_apply` / `matvec` above compute the
# same values with fewer wrapper layers; these keep every conversion,
# validation and axis move of the reference's per-leaf path, so the Python
# overhead per block is the reference's:
#   tensor.mode_product / contract / reshape / multi_mode_apply
#       (tensor.py:27-32, 35-52, 55-86, 89-104, 118-132),
#   blocks.tlr_apply (blocks.py:230-259),
#   operators._hierarchical_matvec (operators.py:138-156).
# --------------------------------------------------------------------------


def _rl_array(t) -> np.ndarray:
    arr = np.asarray(t, dtype=np.float64)                  # tensor.py:27-32
    if arr.ndim == 0:
        raise ValueError("tensor must have order >= 1")
    return arr


def rl_mode_product(t, m, mode: int) -> np.ndarray:
    """tensor.py:35-52: validated tensordot over `mode`, new axis moved back."""
    t = _rl_array(t)
    m = np.asarray(m, dtype=np.float64)
    if m.ndim != 2 or not 1 <= mode <= t.ndim or m.shape[1] != t.shape[mode - 1]:
        raise ValueError("mode_product: bad factor or mode")
    return np.moveaxis(np.tensordot(m, t, axes=([1], [mode - 1])), 0, mode - 1)


def rl_contract(a, b, dims_a, dims_b) -> np.ndarray:
    """tensor.py:55-86: validated tensordot over 1-based dimension lists."""
    a, b = _rl_array(a), _rl_array(b)
    dims_a, dims_b = list(dims_a), list(dims_b)
    if len(dims_a) != len(dims_b) or len(set(dims_a)) != len(dims_a) or len(set(dims_b)) != len(dims_b):
        raise ValueError("contract: bad dimension lists")
    for da, db in zip(dims_a, dims_b):
        if not (1 <= da <= a.ndim and 1 <= db <= b.ndim) or a.shape[da - 1] != b.shape[db - 1]:
            raise ValueError("contract: extent mismatch")
    return np.tensordot(a, b, axes=([x - 1 for x in dims_a], [x - 1 for x in dims_b]))


def rl_vec_to_tensor(v, shape) -> np.ndarray:
    """tensor.py:89-100: F-order reshape after a float64 ravel."""
    flat = _rl_array(np.asarray(v, dtype=np.float64).ravel(order="F"))
    shape = tuple(int(s) for s in shape)
    if int(np.prod(shape)) != flat.size:
        raise ValueError("reshape: size mismatch")
    return np.reshape(flat, shape, order="F")


def rl_multi_mode_apply(t, factors) -> np.ndarray:
    """tensor.py:118-132: sequential mode products over distinct modes."""
    if len({mode for _, mode in factors}) != len(factors):
        raise ValueError("multi_mode_apply requires distinct modes")
    out = _rl_array(t)
    for m, mode in factors:
        out = rl_mode_product(out, m, mode)
    return out


def rl_tlr_apply(b: Tucker, seg) -> np.ndarray:
    """blocks.py:230-259: V^T mode products (square factors skipped), core
    contraction over the source modes, U mode products, F-order flatten."""
    seg = np.asarray(seg, dtype=np.float64).ravel(order="F")
    d = len(b.ufac)
    cols = [f.shape[0] if f is not None else b.core.shape[d + a] for a, f in enumerate(b.vfac)]
    if seg.size != int(np.prod(cols)):
        raise ValueError("segment length does not match the block")
    w = rl_vec_to_tensor(seg, cols)
    w = rl_multi_mode_apply(w, [(f.T, a + 1) for a, f in enumerate(b.vfac) if f is not None])
    hh = rl_contract(b.core, w, list(range(d + 1, 2 * d + 1)), list(range(1, d + 1)))
    ff = rl_multi_mode_apply(hh, [(f, a + 1) for a, f in enumerate(b.ufac) if f is not None])
    return _rl_array(ff).ravel(order="F")


def rl_leaf(u_tensor: np.ndarray, f_tensor: np.ndarray, lf: Leaf, payload) -> None:
    """One iteration of the leaf loop of operators.py:146-155."""
    seg = u_tensor[_slices(lf.sigma)].ravel(order="F")
    out = payload @ seg if not isinstance(payload, Tucker) else rl_tlr_apply(payload, seg)
    f_tensor[_slices(lf.tau)] += out.reshape([hi - lo for lo, hi in lf.tau], order="F")


def rl_matvec(n: int, d: int, leaves: list, payloads, u) -> np.ndarray:
    """operators.py:138-156: F-order u -> (n,)*d tensor, the DFS leaf loop,
    F-order f.  `payloads[i]` belongs to `leaves[i]`."""
    u = np.asarray(u, dtype=np.float64).ravel(order="F")
    if u.size != n ** d:
        raise ValueError(f"vector length {u.size} != {n ** d}")
    ut = u.reshape((n,) * d, order="F")
    ft = np.zeros((n,) * d)
    for lf, pl in zip(leaves, payloads):
        rl_leaf(ut, ft, lf, pl)
    return ft.ravel(order="F")


def leaf_key(lf: Leaf) -> tuple:
    """Payload identity on a uniform grid with a translation-invariant kernel:
    (kind, level, box sizes, source - target offset) -- equal keys give equal
    blocks (the factors depend on the box size only, the core and the dense
    block on the offset; the tau == sigma diagonal is the same cell average)."""
    return (lf.kind, lf.level, tuple(hi - lo for lo, hi in lf.tau), tuple(hi - lo for lo, hi in lf.sigma),
            tuple(s[0] - t[0] for t, s in zip(lf.tau, lf.sigma)))


def shared_payloads(pb: Problem, leaves: list) -> list:
    """Payload per leaf, one object per leaf_key (uniform grids): the
    reference builds every leaf's block separately; the loop applies the same
    values, and configs 2-4 would not fit in host memory otherwise."""
    diag = pb.diag()
    cache: dict = {}
    out = []
    for lf in leaves:
        key = leaf_key(lf)
        if key not in cache:
            cache[key] = build_payload(pb, lf, diag)
        out.append(cache[key])
    return out
