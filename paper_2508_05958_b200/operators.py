"""Hierarchical Tucker operator: construct and matvec on the B200 (drop-in for
``htlr.operators``, /root/reference/pkg/src/htlr/operators.py).

``construct`` builds the interaction lists (C++, bit-exact with the
reference) and runs every numeric construction step on the device;
``matvec`` / ``matmat`` apply the operator with the sm_100a kernels.  Host
numpy vectors are accepted (copied to and from the device, as a drop-in for
the reference's numpy API); CUDA torch tensors stay on the device.
"""

from __future__ import annotations

import ctypes
import warnings
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from .blocks import DenseBlock, LowRankBlock, TuckerBlock
from .grids import (AdmissibilityRule, BlockClusterTree, UniformGrid,
                    build_cluster_tree, export_leaf_array, grid_kind)
from .kernels import CoefficientFn, KernelSpec, QuadratureConfig, singular_rule


@dataclass(frozen=True)
class BuildConfig:
    """operators.py:38-59."""

    rank: int
    leaf_side: int
    rule: AdmissibilityRule
    kernel: KernelSpec
    coeff: CoefficientFn
    quadrature: QuadratureConfig = field(default_factory=QuadratureConfig)

    def __post_init__(self):
        if self.rank < 1:
            raise ValueError("rank must be positive")
        if not self.rank <= self.leaf_side <= 2 * self.rank:
            warnings.warn(
                f"leaf side {self.leaf_side} outside the recommended range "
                f"[rank, 2*rank] = [{self.rank}, {2 * self.rank}]; the linear "
                "storage bound assumes it",
                stacklevel=2,
            )


@dataclass(frozen=True)
class StorageReport:
    dense_scalars: int
    factor_scalars: int
    core_scalars: int
    total_scalars: int
    theoretical_bound: float
    device_scalars: int = 0   # what the B200 plan actually stores (deduplicated)


def _desc(cfg: BuildConfig, grid: UniformGrid) -> _lib.HtlrDesc:
    k = cfg.kernel
    coeff = cfg.coeff.constant_value if cfg.coeff.constant_value is not None else 0.0
    return _lib.HtlrDesc(
        d=grid.d, n=grid.n, leaf_side_max=cfg.leaf_side, rank=cfg.rank,
        rule=_lib.HTLR_RULE_WEAK if cfg.rule.kind == "weak" else _lib.HTLR_RULE_STRONG,
        eta=float(cfg.rule.eta or 0.0), kernel=k.device_code, sigma=float(k.sigma or 0.0),
        scale=float(k.scale), quad_q=int(cfg.quadrature.q),
        corner_subdivision=singular_rule(k, cfg.quadrature), coeff_const=float(coeff),
        grid_kind=grid_kind(grid)[0], amplitude=grid_kind(grid)[1])


class _Payloads:
    """Lazy leaf_id -> TuckerBlock | DenseBlock view (exports from the device)."""

    def __init__(self, op: "HTLRMatrix"):
        self._op = op

    def __len__(self):
        return self._op.num_leaves

    def __getitem__(self, leaf_id: int):
        if leaf_id < 0:
            leaf_id += len(self)
        return self._op.export_block(leaf_id)

    def __iter__(self):
        for i in range(len(self)):
            yield self[i]


class HTLRMatrix:
    """Device-resident HTLR operator (operators.py:62-71 attribute names)."""

    def __init__(self, grid: UniformGrid, config: BuildConfig, device: int):
        self.grid = grid
        self.config = config
        self.device = device
        self._plan = ctypes.c_void_p()
        _lib.check(_lib.lib().htlr_plan_create(ctypes.byref(_desc(config, grid)), device,
                                               ctypes.byref(self._plan)))
        self._block_tree: Optional[BlockClusterTree] = None
        self.payloads = _Payloads(self)

    def __del__(self):
        plan = getattr(self, "_plan", None)
        if plan:
            try:
                _lib.lib().htlr_plan_destroy(plan)
            except Exception:
                pass
            self._plan = None

    @property
    def num_points(self) -> int:
        return self.grid.num_points

    def _info(self):
        depth, side = ctypes.c_int32(), ctypes.c_int32()
        nl, na, nn = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _lib.check(_lib.lib().htlr_tree_info(self._plan, ctypes.byref(depth), ctypes.byref(side),
                                             ctypes.byref(nl), ctypes.byref(na), ctypes.byref(nn)))
        return depth.value, side.value, nl.value, na.value, nn.value

    @property
    def num_leaves(self) -> int:
        return self._info()[2]

    @property
    def block_tree(self) -> BlockClusterTree:
        if self._block_tree is None:
            arr = export_leaf_array(self._plan, self.grid.d)
            tree = build_cluster_tree(self.grid, self.config.leaf_side)
            self._block_tree = BlockClusterTree(self.grid, self.config.rule, tree, arr)
        return self._block_tree

    def diag_value(self) -> float:
        out = ctypes.c_double()
        _lib.check(_lib.lib().htlr_diag_value(self._plan, ctypes.byref(out)))
        return out.value

    def export_block(self, leaf_id: int):
        """Reference-layout payload of one leaf (blocks.py:33-73)."""
        depth, side, nl, _, _ = self._info()
        d, p = self.grid.d, self.config.rank
        cap = max(p ** (2 * d), side ** (2 * d))
        buf = np.zeros(cap)
        nfac_max = 2 * d * self.grid.n * p
        if isinstance(self, HMatrix):   # dense factors: 2 x side^d x p^d at the coarsest level
            nfac_max = max(nfac_max, 2 * max(self.grid.n // 2, 1) ** d * p ** d)
        fac = np.zeros(nfac_max)
        shapes = np.zeros(4, dtype=np.int32)
        _lib.check(_lib.lib().htlr_export_block(self._plan, int(leaf_id), buf.ctypes.data, buf.size,
                                                fac.ctypes.data, fac.size, shapes.ctypes.data))
        kind, rows, cols, nfac = (int(v) for v in shapes)
        if kind == 1:
            return DenseBlock(matrix=buf[: rows * cols].reshape(rows, cols).copy())
        if kind == 2:
            P = p ** d
            g = buf[: P * P].reshape(P, P).copy()
            u = fac[: rows * P].reshape(rows, P).copy()
            v = fac[rows * P: 2 * rows * P].reshape(rows, P).copy()
            return LowRankBlock(u=u, g=g, v=v)
        core = buf[: p ** (2 * d)].reshape((p,) * (2 * d), order="F").copy()
        if nfac == 0:
            return TuckerBlock(core=core, u_factors=[None] * d, v_factors=[None] * d)
        # (mapped grids export raw factors: target Lagrange factor, source
        # cell-width-weighted factor; square factors included)
        s = nfac // (2 * d * p)
        mats = [fac[i * s * p:(i + 1) * s * p].reshape(s, p).copy() for i in range(2 * d)]
        return TuckerBlock(core=core, u_factors=mats[:d], v_factors=mats[d:])

    FORMULATIONS = ("dense", "separable", "regenerated")

    def formulation(self) -> str:
        """How the device applies the blocks (same operator in every case):
        "dense" deduplicated cores, "separable" Kronecker per-axis factors
        (Gaussian kernel, p = leaf side = 8, 3-D), or "regenerated" (mapped grid)."""
        rc = _lib.lib().htlr_formulation(self._plan)
        if rc < 0:
            _lib.check(rc)
        return self.FORMULATIONS[rc]

    LEAF_PASSES = ("gemm", "items", "cooperative", "banded")

    def leaf_pass(self) -> str:
        """How a separable plan runs its leaf level: "items" (per-warp pair
        runs), "cooperative" (per-parent CTAs) or "banded" (three line sweeps
        over the leaf grid, eta = 1); "gemm" for the other formulations."""
        rc = _lib.lib().htlr_leaf_pass(self._plan)
        if rc < 0:
            _lib.check(rc)
        return self.LEAF_PASSES[rc]

    def last_launch_count(self) -> int:
        return int(_lib.lib().htlr_last_launch_count(self._plan))

    PHASES = ("permute", "upward", "gemm_level", "gemm_leaf", "downward", "regen_level", "regen_near", "sep_level",
              "sep_leaf", "band_z", "band_yx")

    def profile(self, on: bool = True) -> None:
        """Bracket every kernel launch of later matvecs with CUDA events."""
        _lib.check(_lib.lib().htlr_profile_enable(self._plan, int(bool(on))))

    def profile_read(self) -> list:
        """Per-launch records of the last matvec: phase, level, device ms,
        algorithmic flops and bytes (synchronises)."""
        cnt = ctypes.c_int64()
        _lib.check(_lib.lib().htlr_profile_read(self._plan, None, None, None, None, None, 0, ctypes.byref(cnt)))
        n = cnt.value
        if n == 0:
            return []
        kinds = np.zeros(n, dtype=np.int32)
        levels = np.zeros(n, dtype=np.int32)
        ms = np.zeros(n)
        fl = np.zeros(n)
        by = np.zeros(n)
        _lib.check(_lib.lib().htlr_profile_read(self._plan, kinds.ctypes.data, levels.ctypes.data, ms.ctypes.data,
                                                fl.ctypes.data, by.ctypes.data, n, ctypes.byref(cnt)))
        return [{"phase": self.PHASES[k], "level": int(lv), "ms": float(t), "flops": float(f), "bytes": float(b)}
                for k, lv, t, f, b in zip(kinds, levels, ms, fl, by)]


def _current_stream_ptr(device: int) -> int:
    import torch
    return torch.cuda.current_stream(device).cuda_stream


def construct(cfg: BuildConfig, grid: UniformGrid, threads: int = 1,
              device: Optional[int] = None) -> HTLRMatrix:
    """Build the hierarchical Tucker operator (operators.py:121-126).
    `threads` is accepted for API compatibility; construction runs on the
    GPU."""
    import torch
    if cfg.kernel.kind not in ("gaussian", "slp2d", "slp3d"):
        cfg.kernel.device_code  # raises ValueError with the explanation
    if grid_kind(grid)[0] == 1 and not cfg.kernel.translation_invariant:
        raise ValueError("mapped grids need a translation-invariant kernel formula")
    if device is None:
        device = torch.cuda.current_device() if torch.cuda.is_available() else 0
    op = HTLRMatrix(grid, cfg, int(device))
    L = _lib.lib()
    _lib.check(L.htlr_build_lists(op._plan))
    if cfg.coeff.constant_value is None:
        a = np.ascontiguousarray(cfg.coeff(_all_points(grid)), dtype=np.float64)
        if a.shape != (grid.num_points,):
            raise ValueError("coefficient evaluator must return one value per point")
        _lib.check(L.htlr_set_coeff(op._plan, a.ctypes.data))
    with torch.cuda.device(device):
        _lib.check(L.htlr_construct(op._plan, ctypes.c_void_p(_current_stream_ptr(device))))
    return op


class HMatrix(HTLRMatrix):
    """H-matrix baseline handle (operators.py:74-83)."""


def construct_hmatrix(cfg: BuildConfig, grid: UniformGrid, threads: int = 1,
                      device: Optional[int] = None) -> HMatrix:
    """Baseline with conventional low-rank leaves (operators.py:129-135): same
    interpolant and cores, factors applied as dense kron(Q,..,Q) matrices."""
    import torch
    cfg.kernel.device_code
    if grid_kind(grid)[0] != 0:
        raise ValueError("the H-matrix baseline is built for uniform grids only")
    if device is None:
        device = torch.cuda.current_device() if torch.cuda.is_available() else 0
    op = HMatrix(grid, cfg, int(device))
    L = _lib.lib()
    _lib.check(L.htlr_set_lowrank(op._plan, 1))
    _lib.check(L.htlr_build_lists(op._plan))
    if cfg.coeff.constant_value is None:
        a = np.ascontiguousarray(cfg.coeff(_all_points(grid)), dtype=np.float64)
        _lib.check(L.htlr_set_coeff(op._plan, a.ctypes.data))
    with torch.cuda.device(device):
        _lib.check(L.htlr_construct(op._plan, ctypes.c_void_p(_current_stream_ptr(device))))
    return op


def hmatrix_matvec(op: HMatrix, u):
    """operators.py:164-165."""
    return _apply(op, u, 1)


def _all_points(grid: UniformGrid) -> np.ndarray:
    axes = [grid.coords1d()] * grid.d
    mesh = np.meshgrid(*axes, indexing="ij")
    return np.stack([m.ravel(order="F") for m in mesh], axis=-1)


def _apply_device_fast(op: HTLRMatrix, u, nrhs_expected: Optional[int], out):
    """Contiguous float64 CUDA input on the plan's device (and a matching
    contiguous CUDA `out`, if given): straight to htlr_matvec with the
    caller's buffers -- no reshapes, copies or extra checks (a few us of host
    time per call, which the small configs' steps are made of).  None when
    the input needs the general path."""
    import torch
    if not (u.is_cuda and u.dtype == torch.float64 and u.is_contiguous() and u.device.index == op.device):
        return None
    n_pts = op.num_points
    if nrhs_expected == 1:
        if u.dim() != 1 or u.shape[0] != n_pts:
            return None
        R = 1
    else:
        if u.dim() != 2 or u.shape[0] != n_pts:
            return None
        R = u.shape[1]
    if out is None:
        f = torch.empty_like(u)
    elif (isinstance(out, torch.Tensor) and out.is_cuda and out.dtype == torch.float64 and out.is_contiguous()
          and out.shape == u.shape and out.device == u.device and out.data_ptr() != u.data_ptr()):
        f = out
    else:
        return None
    _lib.check(_lib.lib().htlr_matvec(op._plan, u.data_ptr(), f.data_ptr(), R,
                                      torch.cuda.current_stream(op.device).cuda_stream))
    return f


def _apply(op: HTLRMatrix, u, nrhs_expected: Optional[int], out=None):
    import torch
    is_torch = isinstance(u, torch.Tensor)
    if is_torch and u.is_cuda:
        f = _apply_device_fast(op, u, nrhs_expected, out)
        if f is not None:
            return f
    if is_torch:
        x = u.to(dtype=torch.float64)
        host = x.device.type != "cuda"
    else:
        x = torch.from_numpy(np.ascontiguousarray(np.asarray(u, dtype=np.float64)))
        host = True
    n_pts = op.num_points
    if nrhs_expected == 1:
        # the reference flattens in F order (operators.py:139 u.ravel(order="F")):
        # an (n,)*d field's first index runs fastest
        flat = x.permute(*reversed(range(x.dim()))).reshape(-1) if x.dim() > 1 else x.reshape(-1)
        if flat.numel() != n_pts:
            raise ValueError(f"vector length {flat.numel()} != {n_pts}")
        x2 = flat.reshape(n_pts, 1)
    else:
        if x.dim() != 2 or x.shape[0] != n_pts:
            raise ValueError(f"expected an ({n_pts}, R) block, got shape {tuple(x.shape)}")
        x2 = x
    R = int(x2.shape[1])
    dev = torch.device("cuda", op.device)
    if host and is_torch and x2.is_pinned() and x2.is_contiguous():
        # page-locked host vectors: the plan copies them itself, overlapped
        # with the device work where the formulation allows (htlr_matvec_host)
        shape = (n_pts,) if nrhs_expected == 1 else (n_pts, R)
        if out is not None:
            if not isinstance(out, torch.Tensor) or tuple(out.shape) != shape or out.dtype != torch.float64:
                raise ValueError(f"out must be a float64 tensor of shape {shape}")
        if out is not None and out.device.type == "cpu" and out.is_pinned() and out.is_contiguous():
            res = out
        else:
            res = torch.empty(shape, dtype=torch.float64, pin_memory=True)
        with torch.cuda.device(op.device):
            stream = torch.cuda.current_stream(op.device)
            _lib.check(_lib.lib().htlr_matvec_host(op._plan, ctypes.c_void_p(x2.data_ptr()),
                                                   ctypes.c_void_p(res.data_ptr()), R,
                                                   ctypes.c_void_p(stream.cuda_stream)))
            stream.synchronize()
        if out is not None and res is not out:
            out.copy_(res)
            return out
        return res
    ud = x2.to(dev, non_blocking=True).contiguous()
    fd = torch.empty_like(ud)
    with torch.cuda.device(op.device):
        stream = torch.cuda.current_stream(op.device).cuda_stream
        _lib.check(_lib.lib().htlr_matvec(op._plan, ctypes.c_void_p(ud.data_ptr()),
                                          ctypes.c_void_p(fd.data_ptr()), R, ctypes.c_void_p(stream)))
    res_d = fd.reshape(-1) if nrhs_expected == 1 else fd
    if out is not None:
        # caller-provided result buffer (host or device), e.g. a reused pinned
        # tensor: one async copy on the same stream, no allocation
        if not isinstance(out, torch.Tensor) or tuple(out.shape) != tuple(res_d.shape) or \
                out.dtype != torch.float64:
            raise ValueError(f"out must be a float64 tensor of shape {tuple(res_d.shape)}")
        out.copy_(res_d, non_blocking=True)
        if out.device.type != "cuda":
            torch.cuda.current_stream(op.device).synchronize()
        return out
    if host:
        if is_torch and x.is_pinned():
            # pinned in -> pinned out (torch's caching host allocator), one
            # async D2H copy on the same stream
            res = torch.empty(res_d.shape, dtype=res_d.dtype, pin_memory=True)
            res.copy_(res_d, non_blocking=True)
            torch.cuda.current_stream(op.device).synchronize()
            return res
        res = res_d.cpu()
        return res.numpy() if not is_torch else res
    return res_d


def matvec(op: HTLRMatrix, u, out=None):
    """f = A u (operators.py:159-161).  numpy in -> numpy out; CUDA tensor in
    -> CUDA tensor out (no host copies).  `out`: optional float64 torch tensor
    (host, e.g. pinned, or device) that receives f and is returned."""
    return _apply(op, u, 1, out)


def matmat(op: HTLRMatrix, U, out=None):
    """F = A U for a block of right-hand sides U of shape (N, R); `out` as in
    matvec."""
    return _apply(op, U, None, out)


def weak_storage_bound(d: int, rank: int, num_points: int) -> float:
    """operators.py:164-172."""
    p = float(rank)
    return (16.0 * d * p ** (2 - d) + p ** d + 2 ** d * p ** d) * num_points


def storage_report(op: HTLRMatrix) -> StorageReport:
    """Scalars the reference would store per leaf (operators.py:175-197), plus
    the deduplicated device storage of this plan."""
    out = np.zeros(5, dtype=np.int64)
    _lib.check(_lib.lib().htlr_storage(op._plan, out.ctypes.data))
    return StorageReport(
        dense_scalars=int(out[0]), factor_scalars=int(out[1]), core_scalars=int(out[2]),
        total_scalars=int(out[3]),
        theoretical_bound=weak_storage_bound(op.grid.d, op.config.rank, op.num_points),
        device_scalars=int(out[4]))


def operation_counts(op: HTLRMatrix) -> dict:
    """operators.py:200-209."""
    _, _, nl, na, nn = op._info()
    return {"dense_leaves": nn, "compressed_leaves": na, "total_leaves": nl}


# the reference defines the row-sampling error estimate in operators.py
# (operators.py:212-260); here it lives in rows.py (device exact rows)
from .rows import DegenerateErrorEstimate, estimate_rel_error_random, exact_row_evaluator  # noqa: E402,F401
