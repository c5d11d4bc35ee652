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


def _mode(t: np.ndarray, m: np.ndarray, mode: int) -> np.ndarray:
    out = np.tensordot(m, t, axes=([1], [mode - 1]))
    return np.moveaxis(out, 0, mode - 1)


def materialize(block) -> np.ndarray:
    """Full matrix of an exported block (host helper for parity tools)."""
    if isinstance(block, DenseBlock):
        return block.matrix
    if isinstance(block, LowRankBlock):
        return block.u @ block.g @ block.v.T
    d = len(block.u_factors)
    full = block.core
    for a, f in enumerate(block.u_factors):
        if f is not None:
            full = _mode(full, f, a + 1)
    for a, f in enumerate(block.v_factors):
        if f is not None:
            full = _mode(full, f, d + a + 1)
    rows, cols = block.shape
    return full.reshape(rows, cols, order="F")


def storage_count(block) -> int:
    """Scalars the reference stores for this block (blocks.py:289-299)."""
    if isinstance(block, DenseBlock):
        return block.matrix.size
    if isinstance(block, LowRankBlock):
        return block.u.size + block.g.size + block.v.size
    return (sum(f.size for f in block.u_factors if f is not None)
            + sum(f.size for f in block.v_factors if f is not None) + block.core.size)
