"""Leaf payload types (drop-in for ``htlr.blocks`` data types,
/root/reference/pkg/src/htlr/blocks.py:33-73).

On the B200 the payloads are not stored per leaf: every unique core / near
block lives once in device memory, pre-tiled for the GEMM.  These classes
are what ``HTLRMatrix.payloads[leaf_id]`` exports, in the reference layout,
for parity checks; ``materialize`` and ``storage_count`` are the
reference's host helpers over them (blocks.py:267-299).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib, tensor
from .chebyshev import cheb_points, core_tensor, factor_matrix
from .grids import domain_of
from .kernels import diagonal_entry, pairwise


@dataclass
class TuckerBlock:
    """Order-2d core (target modes first) with per-dim orthonormal factors;
    ``None`` = identity, the square factor being folded into the core."""

    core: np.ndarray
    u_factors: list
    v_factors: list

    def _side(self, factors, off):
        return tuple(f.shape[0] if f is not None else self.core.shape[off + a]
                     for a, f in enumerate(factors))

    @property
    def row_sizes(self) -> tuple:
        return self._side(self.u_factors, 0)

    @property
    def col_sizes(self) -> tuple:
        return self._side(self.v_factors, len(self.u_factors))

    @property
    def shape(self) -> tuple:
        return int(np.prod(self.row_sizes)), int(np.prod(self.col_sizes))


@dataclass
class LowRankBlock:
    """Conventional low-rank block u g v^T of the H-matrix baseline
    (blocks.py:76-86)."""

    u: np.ndarray
    g: np.ndarray
    v: np.ndarray

    @property
    def shape(self) -> tuple:
        return self.u.shape[0], self.v.shape[0]


@dataclass
class DenseBlock:
    matrix: np.ndarray

    @property
    def shape(self) -> tuple:
        return self.matrix.shape


def materialize(block) -> np.ndarray:
    """Full matrix of a block (blocks.py:267-286), the products on the device."""
    if isinstance(block, DenseBlock):
        return block.matrix
    if isinstance(block, LowRankBlock):
        return tensor._gemm(tensor._gemm(block.u, block.g), np.ascontiguousarray(block.v.T))
    d = len(block.u_factors)
    updates = [(f, a + 1) for a, f in enumerate(block.u_factors) if f is not None]
    updates += [(f, d + a + 1) for a, f in enumerate(block.v_factors) if f is not None]
    full = tensor.multi_mode_apply(block.core, updates)
    rows, cols = block.shape
    return full.reshape(rows, cols, order="F")


# ---------------------------------------------------------------------------
# per-block builders and applies (blocks.py:89-264), device-backed: the
# Chebyshev nodes, Lagrange factors and kernel samples come from the device
# interpolation kernels (chebyshev.py), the QR, mode products and GEMMs from
# csrc/htlr_tensor.cu.  construct() does not call these (the plan builds
# deduplicated operators in bulk); they serve callers working block by block.
# ---------------------------------------------------------------------------


def _interpolation_data(k, grid, tau, sigma, rank):
    """Raw per-dimension factors and kernel core of a box pair (blocks.py:89-106)."""
    dom_tau, dom_sigma = domain_of(grid, tau), domain_of(grid, sigma)
    if dom_tau.overlap_volume(dom_sigma) > 0.0:
        raise ValueError("interpolation blocks require disjoint domains")
    g_tau = [cheb_points(lo, hi, rank) for lo, hi in dom_tau.intervals]
    g_sigma = [cheb_points(lo, hi, rank) for lo, hi in dom_sigma.intervals]
    u_raw = [factor_matrix(grid.coords1d(*tau.ranges[a]), g_tau[a]) for a in range(grid.d)]
    v_raw = [factor_matrix(grid.coords1d(*sigma.ranges[a]), g_sigma[a]) for a in range(grid.d)]
    return u_raw, v_raw, core_tensor(k, g_tau, g_sigma)


def build_tlr(k, grid, tau, sigma, rank: int, h: float, trim: bool = False) -> TuckerBlock:
    """Tucker block of a box pair: interpolate, orthogonalise every non-square
    factor by thin QR, fold h^d and the triangular (or square raw) factors into
    the core in the interleaved order u1, v1, u2, v2, ... (blocks.py:126-164)."""
    if trim:
        raise NotImplementedError("trim=True (column-pivoted, truncated QR) is not on the B200 path; "
                                  "construct() never trims (blocks.py:133)")
    u_raw, v_raw, core = _interpolation_data(k, grid, tau, sigma, rank)
    d = grid.d
    u_f, v_f, updates = [], [], []
    for a in range(d):
        for raw, facs, mode in ((u_raw[a], u_f, a + 1), (v_raw[a], v_f, d + a + 1)):
            if raw.shape[0] == raw.shape[1]:
                facs.append(None)
                updates.append((raw, mode))
            else:
                f = tensor.qr(raw)
                facs.append(f.q)
                updates.append((f.r, mode))
    core = tensor.multi_mode_apply(h ** d * core, updates)
    return TuckerBlock(core=core, u_factors=u_f, v_factors=v_f)


def build_lowrank(k, grid, tau, sigma, rank: int, h: float) -> LowRankBlock:
    """H-matrix baseline block: the same interpolant with Kronecker factors
    orthogonalised as single tall matrices (blocks.py:166-187)."""
    u_raw, v_raw, core = _interpolation_data(k, grid, tau, sigma, rank)
    d = grid.d
    u_full, v_full = u_raw[-1], v_raw[-1]
    for a in range(d - 2, -1, -1):   # last dimension outermost (first index fastest)
        u_full = tensor.kron(u_full, u_raw[a])
        v_full = tensor.kron(v_full, v_raw[a])
    g = h ** d * core.reshape(rank ** d, rank ** d, order="F")
    qu, qv = tensor.qr(u_full), tensor.qr(v_full)
    g = tensor._gemm(tensor._gemm(qu.r, g), np.ascontiguousarray(qv.r.T))
    return LowRankBlock(u=qu.q, g=g, v=qv.q)


def build_dense(k, coeff, grid, tau, sigma, h: float, cfg, diag_value=None) -> DenseBlock:
    """a(x_i) 1[i=j] + K_ij h^d over a box pair; tau == sigma takes the cell
    average on the diagonal (blocks.py:190-227, kernels.py:137-149)."""
    if tau != sigma:
        overlaps = all(max(lo1, lo2) < min(hi1, hi2) for (lo1, hi1), (lo2, hi2) in zip(tau.ranges, sigma.ranges))
        if overlaps:
            raise ValueError("dense blocks require equal or disjoint index boxes")
    x = np.ascontiguousarray(grid.points(tau))
    if tau == sigma:
        if diag_value is None:
            diag = np.asarray([diagonal_entry(k, x[i], h, cfg) for i in range(x.shape[0])])
        else:
            diag = np.full(x.shape[0], float(diag_value))
        out = np.empty((x.shape[0], x.shape[0]))
        _lib.check(_lib.lib().htlr_kernel_pairs_masked(k.device_code, float(k.sigma or 0.0), float(k.scale),
                                                       x.shape[1], x.ctypes.data, x.shape[0],
                                                       np.ascontiguousarray(diag).ctypes.data, out.ctypes.data))
        mat = out * h ** grid.d
        idx = np.arange(x.shape[0])
        mat[idx, idx] += coeff(x)
    else:
        mat = pairwise(k, x, grid.points(sigma)) * h ** grid.d
    return DenseBlock(matrix=mat)


def tlr_apply(block: TuckerBlock, u_segment) -> np.ndarray:
    """Tucker block times a source segment: V^T mode products, core
    contraction over the source modes, U mode products (blocks.py:230-259)."""
    seg = np.asarray(u_segment, dtype=np.float64).ravel(order="F")
    cols = block.col_sizes
    if seg.size != int(np.prod(cols)):
        raise ValueError("segment length does not match the block")
    d = len(cols)
    w = tensor.vec_to_tensor(seg, cols)
    w = tensor.multi_mode_apply(w, [(f.T, a + 1) for a, f in enumerate(block.v_factors) if f is not None])
    hh = tensor.contract(block.core, w, list(range(d + 1, 2 * d + 1)), list(range(1, d + 1)))
    ff = tensor.multi_mode_apply(hh, [(f, a + 1) for a, f in enumerate(block.u_factors) if f is not None])
    return tensor.tensor_to_vec(ff)


def lowrank_apply(block: LowRankBlock, u_segment) -> np.ndarray:
    """u (g (v^T seg)) (blocks.py:262-264)."""
    seg = np.asarray(u_segment, dtype=np.float64).ravel(order="F").reshape(-1, 1)
    t = tensor._gemm(np.ascontiguousarray(block.v.T), seg)
    return tensor._gemm(block.u, tensor._gemm(block.g, t)).ravel()


def storage_count(block) -> int:
    """Scalars the reference stores for this block (blocks.py:289-299)."""
    if isinstance(block, DenseBlock):
        return block.matrix.size
    if isinstance(block, LowRankBlock):
        return block.u.size + block.g.size + block.v.size
    return (sum(f.size for f in block.u_factors if f is not None)
            + sum(f.size for f in block.v_factors if f is not None) + block.core.size)
