"""The BASELINE.json workloads as (grid, BuildConfig, input) recipes.

configs[0..4] of /root/repo/BASELINE.json; inputs follow its seeds in the
reference's F-order grid linearisation.  Config 5 uses the mapped
quasi-uniform grid (not representable by the reference's UniformGrid) with
the reference's leaf semantics: leaf_side 8 at n = 96 gives side-6 leaves
(grids.py:196-207).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np

from .grids import AdmissibilityRule, MappedGrid, UniformGrid
from .kernels import CoefficientFn, KernelSpec, gaussian_bw, inv_r_3d, neg_log_2d
from .operators import BuildConfig


@dataclass(frozen=True)
class Workload:
    name: str
    d: int
    n: int
    leaf: int
    rank: int
    kernel: Callable[[], KernelSpec]
    a: float
    nrhs: int
    matvecs: int
    description: str
    amplitude: float = -1.0   # >= 0: MappedGrid with this amplitude

    @property
    def grid(self):
        if self.amplitude >= 0:
            return MappedGrid(self.d, self.n, self.amplitude)
        return UniformGrid(self.d, self.n)

    def build_config(self) -> BuildConfig:
        return BuildConfig(rank=self.rank, leaf_side=self.leaf, rule=AdmissibilityRule.strong(1.0),
                           kernel=self.kernel(), coeff=CoefficientFn.constant(self.a))

    def input(self) -> np.ndarray:
        N = self.n ** self.d
        seed = int(self.name[-1]) - 1
        rng = np.random.default_rng(seed)
        if self.nrhs > 1:
            return rng.standard_normal((N, self.nrhs))
        return rng.uniform(-1, 1, N)


WORKLOADS = {
    "cfg1": Workload("cfg1", 2, 64, 8, 8, neg_log_2d, 1.0, 1, 1,
                     "2D n=64 -log|x-y| a=1 leaf 8 eta=1 p=8, 1 matvec"),
    "cfg2": Workload("cfg2", 3, 32, 8, 6, inv_r_3d, 0.0, 1, 10,
                     "3D n=32 1/|x-y| leaf 8 eta=1 p=6, construct + 10 matvecs"),
    "cfg3": Workload("cfg3", 3, 64, 8, 6, inv_r_3d, 0.0, 16, 1,
                     "3D n=64 1/|x-y| leaf 8 eta=1 p=6, 16 RHS batched matvec"),
    "cfg4": Workload("cfg4", 3, 128, 8, 8, lambda: gaussian_bw(0.1), 0.0, 1, 1,
                     "3D n=128 exp(-|x-y|^2/0.01) leaf 8 eta=1 p=8, matvec"),
    "cfg5": Workload("cfg5", 3, 96, 8, 6, inv_r_3d, 0.0, 1, 1,
                     "3D mapped quasi-uniform n=96 (x=t+0.05 sin(2 pi t)/(2 pi)) 1/|x-y| leaf 8 (side 6) "
                     "eta=1 p=6, construct + matvec", amplitude=0.05),
}
