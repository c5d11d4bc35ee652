"""Uniform grids, cluster trees and block cluster trees (drop-in for
``htlr.grids``, /root/reference/pkg/src/htlr/grids.py).

Value types and the cluster tree are small host objects, as in the
reference.  The block cluster tree -- the interaction lists of the hot path
-- is built by the C++ list builder of the B200 library (bit-exact with
grids.py:268-296) and exposed both as the reference's ``leaves`` list of
``BlockNode`` objects (materialised lazily) and as a packed int32 array
(``BlockClusterTree.leaf_array``).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import Iterator, Optional

import numpy as np

from . import _lib

ADMISSIBLE = "admissible"       # grids.py:377
INADMISSIBLE = "inadmissible"   # grids.py:378
INTERNAL = "internal"           # grids.py:379


@dataclass(frozen=True)
class UniformGrid:
    """Cell-centred grid on [0,1]^d with points (i + 1/2) h, h = 1/n
    (grids.py:18-50)."""

    d: int
    n: int

    def __post_init__(self):
        if self.d not in (2, 3):
            raise ValueError("only d = 2 and d = 3 are supported")
        if self.n < 1:
            raise ValueError("n must be positive")

    @property
    def h(self) -> float:
        return 1.0 / self.n

    @property
    def num_points(self) -> int:
        return self.n ** self.d

    def coords1d(self, lo: int = 0, hi: Optional[int] = None) -> np.ndarray:
        top = self.n if hi is None else hi
        return (np.arange(lo, top) + 0.5) * self.h

    def points(self, box: "IndexBox") -> np.ndarray:
        """(count, d) coordinates of a box, first index fastest."""
        axes = [self.coords1d(lo, hi) for lo, hi in box.ranges]
        grids = np.meshgrid(*axes, indexing="ij")
        return np.stack([g.ravel(order="F") for g in grids], axis=-1)


@dataclass(frozen=True)
class MappedGrid:
    """Quasi-uniform tensor grid of BASELINE config 5 (not representable by
    the reference's UniformGrid): per dimension x_i = phi((i + 1/2)/n) with
    phi(t) = t + A sin(2 pi t) / (2 pi), cell i = [phi(i/n), phi((i+1)/n)],
    Nystrom weight = product of the cell widths.  Same interface as
    UniformGrid; A = 0 is the uniform grid."""

    d: int
    n: int
    amplitude: float = 0.05

    def __post_init__(self):
        if self.d not in (2, 3):
            raise ValueError("only d = 2 and d = 3 are supported")
        if self.n < 1:
            raise ValueError("n must be positive")

    @property
    def num_points(self) -> int:
        return self.n ** self.d

    def phi(self, t: float) -> float:
        return t + self.amplitude * math.sin(2 * math.pi * t) / (2 * math.pi)

    def coords1d(self, lo: int = 0, hi: Optional[int] = None) -> np.ndarray:
        top = self.n if hi is None else hi
        return np.array([self.phi((i + 0.5) / self.n) for i in range(lo, top)])

    def bounds1d(self) -> np.ndarray:
        return np.array([self.phi(i / self.n) for i in range(self.n + 1)])

    def points(self, box: "IndexBox") -> np.ndarray:
        axes = [self.coords1d(lo, hi) for lo, hi in box.ranges]
        grids = np.meshgrid(*axes, indexing="ij")
        return np.stack([g.ravel(order="F") for g in grids], axis=-1)


@dataclass(frozen=True)
class IndexBox:
    """Half-open 0-based index ranges per dimension (grids.py:53-92)."""

    ranges: tuple

    def __post_init__(self):
        for lo, hi in self.ranges:
            if hi <= lo:
                raise ValueError("index ranges must be nonempty")
            if lo < 0:
                raise ValueError("index ranges must be nonnegative")

    @property
    def d(self) -> int:
        return len(self.ranges)

    @property
    def sizes(self) -> tuple:
        return tuple(hi - lo for lo, hi in self.ranges)

    @property
    def num_points(self) -> int:
        return int(np.prod(self.sizes))

    @property
    def slices(self) -> tuple:
        return tuple(slice(lo, hi) for lo, hi in self.ranges)

    def linear_indices(self, n: int) -> np.ndarray:
        grids = np.meshgrid(*[np.arange(lo, hi) for lo, hi in self.ranges], indexing="ij")
        lin = np.zeros_like(grids[0])
        for a, g in enumerate(grids):
            lin = lin + g * n ** a
        return lin.ravel(order="F")


@dataclass(frozen=True)
class DomainBox:
    """Product of real intervals (grids.py:95-127)."""

    intervals: tuple

    def __post_init__(self):
        for a, b in self.intervals:
            if not a < b:
                raise ValueError("intervals must have positive length")

    @property
    def d(self) -> int:
        return len(self.intervals)

    def diameter_sq(self) -> float:
        return float(sum((b - a) ** 2 for a, b in self.intervals))

    def distance_sq(self, other: "DomainBox") -> float:
        acc = 0.0
        for (a1, b1), (a2, b2) in zip(self.intervals, other.intervals):
            g = max(a1 - b2, a2 - b1, 0.0)
            acc += g * g
        return acc

    def overlap_volume(self, other: "DomainBox") -> float:
        vol = 1.0
        for (a1, b1), (a2, b2) in zip(self.intervals, other.intervals):
            ext = min(b1, b2) - max(a1, a2)
            if ext <= 0.0:
                return 0.0
            vol *= ext
        return vol


@dataclass(frozen=True)
class AdmissibilityRule:
    """Weak or strong(eta) admissibility (grids.py:130-150)."""

    kind: str
    eta: Optional[float] = None

    def __post_init__(self):
        if self.kind not in ("weak", "strong"):
            raise ValueError("kind must be 'weak' or 'strong'")
        if self.kind == "strong" and (self.eta is None or self.eta <= 0):
            raise ValueError("strong admissibility needs eta > 0")

    @staticmethod
    def weak() -> "AdmissibilityRule":
        return AdmissibilityRule(kind="weak")

    @staticmethod
    def strong(eta: float) -> "AdmissibilityRule":
        return AdmissibilityRule(kind="strong", eta=eta)


def is_admissible(rule: AdmissibilityRule, btau: DomainBox, bsigma: DomainBox) -> bool:
    """Scalar predicate, same arithmetic as grids.py:153-165 (the list builder
    evaluates it in C++ with the identical operation order)."""
    if rule.kind == "weak":
        return btau.overlap_volume(bsigma) == 0.0
    lhs = max(btau.diameter_sq(), bsigma.diameter_sq())
    return lhs <= rule.eta * rule.eta * btau.distance_sq(bsigma) * (1.0 + 1e-12)


@dataclass
class ClusterNode:
    box: IndexBox
    level: int
    children: list = field(default_factory=list)

    @property
    def is_leaf(self) -> bool:
        return not self.children


@dataclass
class ClusterTree:
    grid: UniformGrid
    root: ClusterNode
    leaf_side: int
    depth: int

    def leaves(self) -> Iterator[ClusterNode]:
        todo = [self.root]
        while todo:
            node = todo.pop()
            if node.is_leaf:
                yield node
            else:
                todo.extend(node.children[::-1])

    def node(self, level: int, coords) -> ClusterNode:
        """Cluster at `level` with integer box coordinates `coords`."""
        cur = self.root
        for lv in range(1, level + 1):
            shift = level - lv
            idx = 0
            for a in range(self.grid.d):
                idx = idx * 2 + ((coords[a] >> shift) & 1)
            cur = cur.children[idx]
        return cur


def leaf_side_for(n: int, leaf_side_max: int) -> int:
    """Leaf side reached by exact halving (grids.py:196-207)."""
    side = n
    while side > leaf_side_max:
        if side % 2:
            raise ValueError(f"grid side {n} cannot be halved evenly down to the leaf "
                             f"threshold {leaf_side_max}")
        side //= 2
    return side


def build_cluster_tree(grid: UniformGrid, leaf_side_max: int) -> ClusterTree:
    """2^d midpoint tree; children in np.ndindex order (grids.py:210-234)."""
    if leaf_side_max < 1:
        raise ValueError("leaf threshold must be positive")
    side = leaf_side_for(grid.n, leaf_side_max)
    depth = int(round(math.log2(grid.n / side))) if grid.n > side else 0
    combos = list(np.ndindex(*([2] * grid.d)))

    def grow(box: IndexBox, level: int) -> ClusterNode:
        node = ClusterNode(box=box, level=level)
        if max(box.sizes) > leaf_side_max:
            mids = [(lo + hi) // 2 for lo, hi in box.ranges]
            for combo in combos:
                rng = tuple((lo, mid) if c == 0 else (mid, hi)
                            for (lo, hi), mid, c in zip(box.ranges, mids, combo))
                node.children.append(grow(IndexBox(rng), level + 1))
        return node

    root = grow(IndexBox(tuple((0, grid.n) for _ in range(grid.d))), 0)
    return ClusterTree(grid=grid, root=root, leaf_side=side, depth=depth)


def domain_of(grid, box: IndexBox) -> DomainBox:
    """grids.py:237-242 (cell images for a MappedGrid)."""
    if any(hi > grid.n for _, hi in box.ranges):
        raise ValueError("index box exceeds the grid")
    if isinstance(grid, MappedGrid):
        return DomainBox(tuple((grid.phi(lo / grid.n), grid.phi(hi / grid.n)) for lo, hi in box.ranges))
    return DomainBox(tuple((lo * grid.h, hi * grid.h) for lo, hi in box.ranges))


@dataclass
class BlockNode:
    tau: ClusterNode
    sigma: ClusterNode
    kind: str
    level: int
    children: list = field(default_factory=list)
    leaf_id: int = -1


class _LeafList:
    """Sequence view of the packed leaf array as BlockNode objects."""

    def __init__(self, bct: "BlockClusterTree"):
        self._bct = bct
        self._cache = None

    def _all(self):
        if self._cache is None:
            self._cache = [self._bct._leaf(i) for i in range(len(self))]
        return self._cache

    def __len__(self):
        return int(self._bct.leaf_array.shape[0])

    def __getitem__(self, i):
        if self._cache is not None:
            return self._cache[i]
        if isinstance(i, slice):
            return [self._bct._leaf(j) for j in range(*i.indices(len(self)))]
        if i < 0:
            i += len(self)
        return self._bct._leaf(i)

    def __iter__(self):
        return iter(self._all())


class BlockClusterTree:
    """Block cluster tree with the reference's attribute names
    (grids.py:250-265).  ``leaf_array`` rows: [leaf_id, kind(0 adm/1 inadm),
    level, tau lo/hi per dim, sigma lo/hi per dim]."""

    def __init__(self, grid: UniformGrid, rule: AdmissibilityRule, tree: ClusterTree,
                 leaf_array: np.ndarray):
        self.grid = grid
        self.rule = rule
        self.cluster_tree = tree
        self.leaf_array = leaf_array
        self.leaves = _LeafList(self)
        self._root = None

    def _cluster(self, level: int, ranges) -> ClusterNode:
        side = self.grid.n >> level
        return self.cluster_tree.node(level, [lo // side for lo, _ in ranges])

    def _leaf(self, i: int) -> BlockNode:
        row = self.leaf_array[i]
        d = self.grid.d
        lvl = int(row[2])
        tr = [(int(row[3 + 2 * a]), int(row[4 + 2 * a])) for a in range(d)]
        sr = [(int(row[3 + 2 * d + 2 * a]), int(row[4 + 2 * d + 2 * a])) for a in range(d)]
        return BlockNode(tau=self._cluster(lvl, tr), sigma=self._cluster(lvl, sr),
                         kind=ADMISSIBLE if row[1] == 0 else INADMISSIBLE, level=lvl,
                         leaf_id=int(row[0]))

    @property
    def root(self) -> BlockNode:
        """Internal nodes rebuilt from the DFS leaf list (children appear in
        the reference's sigma-outer / tau-inner creation order)."""
        if self._root is None:
            root = BlockNode(self.cluster_tree.root, self.cluster_tree.root, INTERNAL, 0)
            nodes = {(0, id(root.tau), id(root.sigma)): root}
            for lf in self.leaves:
                if lf.level == 0:
                    root = lf
                    nodes = {}
                    break
                chain = []
                t, s = lf.tau, lf.sigma
                for lvl in range(lf.level - 1, -1, -1):
                    side = self.grid.n >> lvl
                    tp = self.cluster_tree.node(lvl, [lo // side for lo, _ in t.box.ranges])
                    sp = self.cluster_tree.node(lvl, [lo // side for lo, _ in s.box.ranges])
                    chain.append((lvl, tp, sp))
                    t, s = tp, sp
                parent = None
                child = lf
                for lvl, tp, sp in chain:
                    key = (lvl, id(tp), id(sp))
                    node = nodes.get(key)
                    fresh = node is None
                    if fresh:
                        node = BlockNode(tp, sp, INTERNAL, lvl)
                        nodes[key] = node
                    if not node.children or node.children[-1] is not child:
                        node.children.append(child)
                    if not fresh:
                        break
                    child = node
            self._root = root
        return self._root


def grid_kind(grid) -> tuple:
    """(grid_kind, amplitude) of the C ABI descriptor."""
    if isinstance(grid, MappedGrid):
        return 1, float(grid.amplitude)
    return 0, 0.0


def _host_plan(d: int, n: int, leaf_side_max: int, rule: AdmissibilityRule, grid=None):
    L = _lib.lib()
    gk, amp = grid_kind(grid)
    desc = _lib.HtlrDesc(d=d, n=n, leaf_side_max=leaf_side_max, rank=1,
                         rule=_lib.HTLR_RULE_WEAK if rule.kind == "weak" else _lib.HTLR_RULE_STRONG,
                         eta=float(rule.eta or 0.0), kernel=_lib.HTLR_KERNEL_GAUSSIAN, sigma=1.0,
                         scale=1.0, quad_q=10, corner_subdivision=1, coeff_const=0.0,
                         grid_kind=gk, amplitude=amp)
    plan = ctypes.c_void_p()
    _lib.check(L.htlr_plan_create(ctypes.byref(desc), -1, ctypes.byref(plan)))
    return plan


def export_leaf_array(plan, d: int) -> np.ndarray:
    L = _lib.lib()
    nl = ctypes.c_int64()
    _lib.check(L.htlr_tree_info(plan, None, None, ctypes.byref(nl), None, None))
    arr = np.empty((nl.value, 3 + 4 * d), dtype=np.int32)
    _lib.check(L.htlr_export_lists(plan, arr.ctypes.data, arr.size))
    return arr


def build_block_cluster_tree(tree: ClusterTree, rule: AdmissibilityRule,
                             grid: Optional[UniformGrid] = None) -> BlockClusterTree:
    """Interaction lists via the C++ builder (grids.py:268-296, bit-exact)."""
    grid = tree.grid if grid is None else grid
    L = _lib.lib()
    plan = _host_plan(grid.d, grid.n, tree.leaf_side, rule, grid)
    try:
        _lib.check(L.htlr_build_lists(plan))
        arr = export_leaf_array(plan, grid.d)
    finally:
        L.htlr_plan_destroy(plan)
    return BlockClusterTree(grid, rule, tree, arr)
