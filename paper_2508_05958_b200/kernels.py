"""Kernel specifications, coefficients and quadrature settings (drop-in for
``htlr.kernels``, /root/reference/pkg/src/htlr/kernels.py).

``KernelSpec`` keeps the reference's fields and adds ``scale`` (a constant
factor on the reference formula) so the BASELINE.json kernels are
expressible:  -log|x-y| = ``neg_log_2d()`` = 2*pi*slp_2d,
1/|x-y| = ``inv_r_3d()`` = 4*pi*slp_3d, exp(-|x-y|^2/s^2) =
``gaussian_bw(s)`` = gaussian(s/sqrt(2)).

Kernel values are only ever evaluated on the device.  ``custom`` Python
callables are accepted for API compatibility but rejected by ``construct``:
the B200 path has no CPU fallback.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from . import _lib

GAUSSIAN = "gaussian"
SLP2D = "slp2d"
SLP3D = "slp3d"
CUSTOM = "custom"

_KIND_CODE = {GAUSSIAN: _lib.HTLR_KERNEL_GAUSSIAN, SLP2D: _lib.HTLR_KERNEL_SLP2D,
              SLP3D: _lib.HTLR_KERNEL_SLP3D}


@dataclass(frozen=True)
class KernelSpec:
    """kernels.py:33-47 plus ``scale``."""

    kind: str
    sigma: Optional[float] = None
    evaluator: Optional[Callable[[np.ndarray, np.ndarray], np.ndarray]] = None
    smooth_at_diagonal: bool = True
    translation_invariant: bool = False
    scale: float = 1.0

    def __post_init__(self):
        if self.kind == GAUSSIAN and (self.sigma is None or self.sigma <= 0):
            raise ValueError("gaussian kernel needs sigma > 0")
        if self.kind == CUSTOM and self.evaluator is None:
            raise ValueError("custom kernel needs an evaluator")

    @property
    def device_code(self) -> int:
        if self.kind not in _KIND_CODE:
            raise ValueError(
                f"kernel kind {self.kind!r} cannot run on the B200 path (custom Python "
                "evaluators are not device code); use gaussian / slp_2d / slp_3d with `scale`")
        return _KIND_CODE[self.kind]


def gaussian(sigma: float, scale: float = 1.0) -> KernelSpec:
    """exp(-|x-y|^2 / (2 sigma^2)) (kernels.py:50-52, :90-92)."""
    return KernelSpec(kind=GAUSSIAN, sigma=sigma, smooth_at_diagonal=True,
                      translation_invariant=True, scale=scale)


def slp_2d(scale: float = 1.0) -> KernelSpec:
    """-log|x-y| / (2 pi) (kernels.py:55-57, :93-97)."""
    return KernelSpec(kind=SLP2D, smooth_at_diagonal=False, translation_invariant=True, scale=scale)


def slp_3d(scale: float = 1.0) -> KernelSpec:
    """1 / (4 pi |x-y|) (kernels.py:60-62, :98-102)."""
    return KernelSpec(kind=SLP3D, smooth_at_diagonal=False, translation_invariant=True, scale=scale)


def custom(evaluator, smooth_at_diagonal: bool = True) -> KernelSpec:
    """kernels.py:65-70 (accepted, but not runnable on the device)."""
    return KernelSpec(kind=CUSTOM, evaluator=evaluator, smooth_at_diagonal=smooth_at_diagonal)


def neg_log_2d() -> KernelSpec:
    """BASELINE config 1 kernel -log|x-y|."""
    return slp_2d(scale=2.0 * math.pi)


def inv_r_3d() -> KernelSpec:
    """BASELINE configs 2, 3, 5 kernel 1/|x-y|."""
    return slp_3d(scale=4.0 * math.pi)


def gaussian_bw(s: float) -> KernelSpec:
    """BASELINE config 4 kernel exp(-|x-y|^2 / s^2)."""
    return gaussian(s / math.sqrt(2.0))


def by_name(name: str, d: int) -> KernelSpec:
    """CLI kernel names; Gaussian bandwidth sqrt(d) (kernels.py:73-85)."""
    if name == GAUSSIAN:
        return gaussian(sigma=float(np.sqrt(d)))
    if name == SLP2D:
        if d != 2:
            raise ValueError("slp2d requires dimension 2")
        return slp_2d()
    if name == SLP3D:
        if d != 3:
            raise ValueError("slp3d requires dimension 3")
        return slp_3d()
    raise ValueError(f"unknown kernel '{name}'")


@dataclass(frozen=True)
class CoefficientFn:
    """a(x) (kernels.py:162-175).  ``constant(c)`` is recognised and passed
    to the device as a scalar; any other evaluator is called once on the grid
    points at construction and uploaded."""

    evaluator: Callable[[np.ndarray], np.ndarray]
    constant_value: Optional[float] = None

    @staticmethod
    def constant(c: float) -> "CoefficientFn":
        c = float(c)
        return CoefficientFn(evaluator=lambda pts: np.full(len(pts), c), constant_value=c)

    def __call__(self, pts: np.ndarray) -> np.ndarray:
        return np.asarray(self.evaluator(np.asarray(pts, dtype=np.float64)), dtype=np.float64)


@dataclass(frozen=True)
class QuadratureConfig:
    """kernels.py:178-192."""

    q: int = 10
    corner_subdivision: bool = True

    def __post_init__(self):
        if self.q < 2:
            raise ValueError("quadrature order must be >= 2")


def pairwise(k: KernelSpec, xpts: np.ndarray, ypts: np.ndarray) -> np.ndarray:
    """Kernel values on all pairs, (m1, d) x (m2, d) -> (m1, m2), evaluated on
    the device with the reference formula (kernels.py:113-117)."""
    x = np.ascontiguousarray(np.atleast_2d(np.asarray(xpts, dtype=np.float64)))
    y = np.ascontiguousarray(np.atleast_2d(np.asarray(ypts, dtype=np.float64)))
    if x.shape[1] != y.shape[1]:
        raise ValueError("point dimensions differ")
    out = np.empty((x.shape[0], y.shape[0]))
    _lib.check(_lib.lib().htlr_kernel_pairs(k.device_code, float(k.sigma or 0.0), float(k.scale), x.shape[1],
                                            x.ctypes.data, x.shape[0], y.ctypes.data, y.shape[0], out.ctypes.data))
    return out


def evaluate(k: KernelSpec, x, y) -> float:
    """Kernel value at one point pair (kernels.py:106-110)."""
    return float(pairwise(k, np.atleast_2d(x), np.atleast_2d(y))[0, 0])


def singular_rule(k: KernelSpec, cfg: QuadratureConfig) -> int:
    """1 when the Duffy corner rule applies (kernels.py:263-265)."""
    return int((not k.smooth_at_diagonal) and bool(cfg.corner_subdivision))


def diagonal_entry(k: KernelSpec, cell_center, h: float, cfg: QuadratureConfig,
                   device: Optional[int] = None) -> float:
    """Cell average of k(x_i, .) over the width-h cell at x_i, computed by
    the device quadrature kernel (kernels.py:252-265).  Only translation
    invariant kernels are supported (the centre is irrelevant, as in the
    reference, which integrates them around the origin)."""
    if h <= 0:
        raise ValueError("cell width must be positive")
    if not k.translation_invariant:
        raise ValueError("the B200 path supports translation-invariant kernels only")
    d = len(np.atleast_1d(cell_center))
    if device is None:
        import torch
        device = torch.cuda.current_device()
    out = ctypes.c_double()
    _lib.check(_lib.lib().htlr_cell_average(k.device_code, float(k.sigma or 0.0), float(k.scale), d,
                                            float(h), int(cfg.q), singular_rule(k, cfg),
                                            int(device), ctypes.byref(out)))
    return out.value
