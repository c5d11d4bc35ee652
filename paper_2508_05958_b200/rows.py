"""Exact-row evaluation and the sampled relative error of a fast matvec
(drop-in for ``htlr.oracles.exact_row_evaluator``, oracles.py:65-100, and
``htlr.operators.estimate_rel_error_random``, operators.py:216-239).

The exact rows are computed on the GPU (``htlr_exact_rows``): one CTA per
sampled row sums k(x_i, x_j) w_j u_j over all N points with the reference's
kernel formula, plus the diagonal (cell average x h^d, or the mapped cell
integral) and a(x_i).  For config 4 that is 1000 x 2.1M kernel evaluations,
which the reference can only do in chunks of 256 rows on the CPU.
"""

from __future__ import annotations

import ctypes
import warnings
from typing import Callable, Optional

import numpy as np

from . import _lib
from .grids import AdmissibilityRule
from .kernels import CoefficientFn, KernelSpec, QuadratureConfig
from .operators import BuildConfig, HTLRMatrix, _all_points, matvec


class DegenerateErrorEstimate(ValueError):
    """Raised when the sampled exact result has zero norm (operators.py:211-213)."""


def exact_row_evaluator(k: KernelSpec, coeff: CoefficientFn, grid, cfg: QuadratureConfig,
                        device: Optional[int] = None) -> Callable[[np.ndarray, np.ndarray], np.ndarray]:
    """Callable (rows, u) -> exact matvec values on those rows."""
    import torch
    if device is None:
        device = torch.cuda.current_device()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        bc = BuildConfig(rank=1, leaf_side=grid.n, rule=AdmissibilityRule.weak(), kernel=k, coeff=coeff,
                         quadrature=cfg)
    holder = HTLRMatrix(grid, bc, int(device))     # geometry + kernel only; no lists, no construct
    if coeff.constant_value is None:
        a = np.ascontiguousarray(coeff(_all_points(grid)), dtype=np.float64)
        _lib.check(_lib.lib().htlr_set_coeff(holder._plan, a.ctypes.data))

    def rows_apply(rows: np.ndarray, u: np.ndarray) -> np.ndarray:
        rows = np.asarray(rows, dtype=np.int64).ravel()
        uu = np.ascontiguousarray(np.asarray(u, dtype=np.float64).ravel(order="F"))
        if uu.size != grid.num_points:
            raise ValueError(f"vector length {uu.size} != {grid.num_points}")
        dev = torch.device("cuda", holder.device)
        rd = torch.from_numpy(rows).to(dev)
        ud = torch.from_numpy(uu).to(dev)
        out = torch.empty(rows.size, dtype=torch.float64, device=dev)
        with torch.cuda.device(holder.device):
            st = torch.cuda.current_stream().cuda_stream
            _lib.check(_lib.lib().htlr_exact_rows(holder._plan, ctypes.c_void_p(rd.data_ptr()), rows.size,
                                                  ctypes.c_void_p(ud.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                                  ctypes.c_void_p(st)))
        return out.cpu().numpy()

    rows_apply.holder = holder
    return rows_apply


def estimate_rel_error_random(op: HTLRMatrix, exact_rows, u: np.ndarray, sample_size: int = 1000,
                              seed: int = 0) -> float:
    """Relative l2 error on a uniformly sampled row subset (operators.py:216-239)."""
    u = np.asarray(u, dtype=np.float64).ravel(order="F")
    n_rows = op.num_points
    if sample_size > n_rows:
        raise ValueError("sample size exceeds the number of rows")
    rows = np.random.default_rng(seed).choice(n_rows, size=sample_size, replace=False)
    approx = matvec(op, u)
    exact = exact_rows(rows, u)
    denom = np.linalg.norm(exact)
    if denom == 0.0:
        raise DegenerateErrorEstimate("exact result has zero norm on the sample")
    return float(np.linalg.norm(approx[rows] - exact) / denom)
