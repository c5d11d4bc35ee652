"""Chebyshev interpolation building blocks (drop-in for the hot-path part of
``htlr.chebyshev``, chebyshev.py:17-85), evaluated on the device.

The plan's construction computes the same quantities inline for every level
and core; these wrappers expose them with the reference's signatures for
users and parity tools.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _lib
from .kernels import KernelSpec, pairwise


@dataclass(frozen=True)
class ChebGrid1D:
    """First-kind nodes on [lo, hi], decreasing (chebyshev.py:17-28)."""

    lo: float
    hi: float
    nodes: np.ndarray

    @property
    def order(self) -> int:
        return len(self.nodes)


def cheb_points(lo: float, hi: float, order: int) -> ChebGrid1D:
    """chebyshev.py:31-38."""
    if not lo < hi:
        raise ValueError("interval must satisfy lo < hi")
    if order < 1:
        raise ValueError("order must be >= 1")
    out = np.empty(order)
    _lib.check(_lib.lib().htlr_cheb_nodes(float(lo), float(hi), int(order), out.ctypes.data))
    return ChebGrid1D(lo=float(lo), hi=float(hi), nodes=out)


def factor_matrix(points: Sequence[float], grid: ChebGrid1D) -> np.ndarray:
    """Lagrange basis of the grid at the points, (n, p) (chebyshev.py:52-66)."""
    pts = np.ascontiguousarray(np.asarray(points, dtype=np.float64).ravel())
    if pts.size and (pts.min() < grid.lo or pts.max() > grid.hi):
        raise ValueError("interpolation points must lie inside the interval")
    nodes = np.ascontiguousarray(grid.nodes, dtype=np.float64)
    out = np.empty((pts.size, grid.order))
    _lib.check(_lib.lib().htlr_lagrange_matrix(pts.ctypes.data, pts.size, nodes.ctypes.data, grid.order,
                                               out.ctypes.data))
    return out


def core_tensor(kernel: KernelSpec, grids_tau: Sequence[ChebGrid1D], grids_sigma: Sequence[ChebGrid1D]) -> np.ndarray:
    """Kernel at all tensor node pairs, order-2d tensor with target modes first
    (chebyshev.py:69-85)."""
    d = len(grids_tau)
    if len(grids_sigma) != d:
        raise ValueError("box dimensions differ")

    def tensor_pts(grids):
        mesh = np.meshgrid(*[g.nodes for g in grids], indexing="ij")
        return np.stack([m.ravel(order="F") for m in mesh], axis=-1)

    vals = pairwise(kernel, tensor_pts(grids_tau), tensor_pts(grids_sigma))
    shape = tuple(g.order for g in grids_tau) + tuple(g.order for g in grids_sigma)
    return vals.ravel(order="F").reshape(shape, order="F")
