"""Multi-GPU HTLR matvec: target boxes sharded by cluster subtrees.

One process per GPU (torchrun).  Shard r owns the contiguous Morton range
[r, r+1) * M_l / world of the clusters of every level l (a union of whole
subtrees; in 3-D with world <= 8 these are octants, which are reflections of
each other, so the work per shard is identical).  Per matvec each shard

  1. local  : permutes its own leaf boxes and runs the upward pass of its own
              source clusters into the exchange buffers (ub, W_l);
  2. exchange: all-gathers those buffers over NCCL / NVLink (each shard's part
              is a contiguous 1/world chunk of each buffer);
  3. remote : runs the gathered GEMMs of its own targets and the fused
              downward pass, writing the f rows of its own leaf boxes.  On a
              mapped grid with the symmetric regeneration every unordered
              block pair is evaluated by one shard, whose column sums land in
              other shards' rows: the full-size accumulators are
              sum-reduce-scattered between the contract and the expand half.

The reference has no parallel matvec; the exchange volume is
|u| + sum_l |W_l| (19 MB for config 4), against milliseconds of fp64 GEMM.
"""

from __future__ import annotations

import ctypes
from typing import Optional

import numpy as np

from . import _lib
from .grids import UniformGrid
from .operators import BuildConfig, HTLRMatrix, _all_points


def allgather_chunks(bufs, rank: int, world: int, group=None) -> None:
    """In-place all-gather of equal contiguous chunks of each 1-D tensor:
    chunk r of every buffer comes from rank r.  NCCL uses the in-place
    all_gather_into_tensor; other backends (gloo, CPU tests) the list form."""
    import torch.distributed as dist
    for b in bufs:
        n = b.numel()
        if n % world:
            raise ValueError("exchange buffer not divisible by the world size")
        c = n // world
        mine = b[rank * c:(rank + 1) * c]
        if b.is_cuda and dist.get_backend(group) == "nccl":
            dist.all_gather_into_tensor(b, mine, group=group)
        elif b.is_cuda:   # gloo harness runs: staged through host memory
            h = b.cpu()
            outs = [h[r * c:(r + 1) * c] for r in range(world)]
            dist.all_gather(outs, h[rank * c:(rank + 1) * c].clone(), group=group)
            b.copy_(h)
        else:
            outs = [b[r * c:(r + 1) * c] for r in range(world)]
            dist.all_gather(outs, mine.clone(), group=group)


def allgather_chunks_async(bufs, rank: int, world: int, group=None):
    """NCCL all-gather of the exchange buffers issued asynchronously (one
    work handle per buffer); the caller enqueues device work that reads only
    its own chunks, then waits (the current stream waits on the collective)."""
    import torch.distributed as dist
    works = []
    for b in bufs:
        n = b.numel()
        if n % world:
            raise ValueError("exchange buffer not divisible by the world size")
        c = n // world
        works.append(dist.all_gather_into_tensor(b, b[rank * c:(rank + 1) * c], group=group, async_op=True))
    return works


def reduce_scatter_chunks(bufs, rank: int, world: int, group=None) -> None:
    """In-place sum-reduce-scatter of each 1-D tensor: afterwards chunk
    `rank` holds the sum over all ranks' buffers (other chunks are scratch).
    NCCL uses reduce_scatter_tensor; other backends an all-reduce."""
    import torch.distributed as dist
    for b in bufs:
        n = b.numel()
        if n % world:
            raise ValueError("reduce buffer not divisible by the world size")
        c = n // world
        if b.is_cuda and dist.get_backend(group) == "nccl":
            out = b.new_empty(c)
            dist.reduce_scatter_tensor(out, b, op=dist.ReduceOp.SUM, group=group)
            b[rank * c:(rank + 1) * c].copy_(out)
        elif b.is_cuda:   # gloo harness runs: staged through host memory
            h = b.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
            b.copy_(h)
        else:
            dist.all_reduce(b, op=dist.ReduceOp.SUM, group=group)


def shard_ranges(M: int, rank: int, world: int):
    """Owned cluster id range of a level with M clusters."""
    if M % world:
        raise ValueError("level cannot be split evenly across shards")
    return M // world * rank, M // world * (rank + 1)


def allreduce_sum(bufs, group=None) -> None:
    """In-place sum of each buffer over all ranks (z-slab shards' W_l)."""
    import torch.distributed as dist
    for b in bufs:
        if b.is_cuda and dist.get_backend(group) != "nccl":   # gloo harness runs
            h = b.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
            b.copy_(h)
        else:
            dist.all_reduce(b, op=dist.ReduceOp.SUM, group=group)


class ShardedOperator:
    """HTLR operator whose targets are split across `world` GPUs.

    mode "subtree": Morton subtrees of every level (the general scheme, module
    docstring).  mode "zslab" (banded separable plans, BASELINE config 4): the
    leaf boxes with z in the rank's 1/world slab -- every rank holds the whole
    u, the only exchange is a sum of the upward coefficients W_l (2.4 MB for
    config 4), and every banded sweep, the upward and the downward pass run
    over the own slab (htlr_set_zslab).  mode "auto" picks zslab when the plan
    is banded."""

    def __init__(self, cfg: BuildConfig, grid: UniformGrid, rank: int, world: int,
                 device: Optional[int] = None, group=None, mode: str = "auto"):
        import torch
        if mode not in ("auto", "subtree", "zslab"):
            raise ValueError(f"unknown shard mode {mode!r}")
        self.grid, self.config = grid, cfg
        self.rank, self.world, self.group = rank, world, group
        if device is None:
            device = torch.cuda.current_device()
        self.device = int(device)
        L = _lib.lib()
        op = None
        # the banded formulation: 3-D Gaussian on a uniform grid, p = leaf side = 8, strong eta = 1
        maybe_banded = (isinstance(grid, UniformGrid) and grid.d == 3 and cfg.kernel.kind == "gaussian"
                        and cfg.rank == 8 and cfg.leaf_side == 8 and cfg.rule.kind == "strong"
                        and float(cfg.rule.eta) == 1.0)
        if mode == "zslab" or (mode == "auto" and maybe_banded):
            from .operators import construct
            op = construct(cfg, grid, device=self.device)
            if op.leaf_pass() == "banded":
                _lib.check(L.htlr_set_zslab(op._plan, int(rank), int(world)))
                self.mode = "zslab"
            elif mode == "zslab":
                raise ValueError("zslab shards need the banded separable formulation")
            else:
                op = None
        if op is None:
            op = HTLRMatrix(grid, cfg, self.device)
            _lib.check(L.htlr_set_shard(op._plan, int(rank), int(world)))
            _lib.check(L.htlr_build_lists(op._plan))
            if cfg.coeff.constant_value is None:
                a = np.ascontiguousarray(cfg.coeff(_all_points(grid)), dtype=np.float64)
                _lib.check(L.htlr_set_coeff(op._plan, a.ctypes.data))
            with torch.cuda.device(self.device):
                _lib.check(L.htlr_construct(op._plan, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
            self.mode = "subtree"
        self.local = op
        self._xbufs = {}
        self._rbufs = {}

    graphs = True   # NCCL z-slab matvecs replay one CUDA graph (local, all-reduce, remote)

    def _zslab_graph(self, ud, R: int):
        """One CUDA graph per RHS count of [local phase, NCCL all-reduce of the
        W_l, remote phase] over plan-owned staging vectors (the caller's u is
        copied in, the result returned as a copy): one host call per matvec
        instead of ~15 launches, so a small shard's device work is not starved
        by the host."""
        import torch
        if not hasattr(self, "_graphs"):
            self._graphs = {}
        if R not in self._graphs:
            # captured over the first caller's u itself (kept alive here): a
            # caller that reuses its input vector pays no staging copy
            u_st = ud
            f_st = torch.zeros_like(ud)
            bufs = self.exchange_buffers(R)
            side = torch.cuda.Stream(device=self.device)
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):   # warm-up outside the capture (lazy allocations)
                self.local_phase(u_st, R)
                if self.world > 1:
                    allreduce_sum(bufs, self.group)
                self.remote_phase(u_st, f_st, R)
            torch.cuda.current_stream().wait_stream(side)
            # the warm-up collective has completed before the capture starts,
            # and the capture is thread-local: the process group's watchdog
            # thread may query its events meanwhile
            torch.cuda.synchronize(self.device)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, capture_error_mode="thread_local"):
                self.local_phase(u_st, R)
                if self.world > 1:
                    allreduce_sum(bufs, self.group)
                self.remote_phase(u_st, f_st, R)
            self._graphs[R] = (g, u_st, f_st)
        g, u_st, f_st = self._graphs[R]
        if ud.data_ptr() != u_st.data_ptr():
            u_st.copy_(ud)
        g.replay()
        return f_st.clone()

    @property
    def exchange_sums(self) -> bool:
        """True when the exchange buffers are summed (all-reduce), not gathered."""
        return _lib.lib().htlr_exchange_kind(self.local._plan) == 1

    # exchange buffers are torch tensors so torch.distributed can move them
    def exchange_buffers(self, R: int):
        import torch
        if R not in self._xbufs:
            L = _lib.lib()
            cnt = ctypes.c_int64()
            _lib.check(L.htlr_exchange_info(self.local._plan, R, ctypes.byref(cnt), None, 0))
            sizes = np.zeros(cnt.value, dtype=np.int64)
            _lib.check(L.htlr_exchange_info(self.local._plan, R, ctypes.byref(cnt), sizes.ctypes.data, cnt.value))
            bufs = [torch.zeros(int(b) // 8, dtype=torch.float64, device=f"cuda:{self.device}") for b in sizes]
            self._xbufs[R] = bufs
        bufs = self._xbufs[R]
        ptrs = (ctypes.c_void_p * len(bufs))(*[b.data_ptr() for b in bufs])
        _lib.check(_lib.lib().htlr_bind_exchange(self.local._plan, R, ptrs, len(bufs)))
        return bufs

    def reduce_buffers(self, R: int):
        """Full-size accumulators the shards sum between the contract and the
        expand half of the remote phase (mapped grid, symmetric
        regeneration); empty for every other plan."""
        import torch
        if R not in self._rbufs:
            L = _lib.lib()
            cnt = ctypes.c_int64()
            _lib.check(L.htlr_reduce_info(self.local._plan, R, ctypes.byref(cnt), None, 0))
            sizes = np.zeros(max(1, cnt.value), dtype=np.int64)
            _lib.check(L.htlr_reduce_info(self.local._plan, R, ctypes.byref(cnt), sizes.ctypes.data, cnt.value))
            bufs = [torch.zeros(int(b) // 8, dtype=torch.float64, device=f"cuda:{self.device}")
                    for b in sizes[:cnt.value]]
            self._rbufs[R] = bufs
        bufs = self._rbufs[R]
        if bufs:
            ptrs = (ctypes.c_void_p * len(bufs))(*[b.data_ptr() for b in bufs])
            _lib.check(_lib.lib().htlr_bind_reduce(self.local._plan, R, ptrs, len(bufs)))
        return bufs

    def shard_info(self) -> dict:
        lo, hi, pairs, fl = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_double()
        _lib.check(_lib.lib().htlr_shard_info(self.local._plan, ctypes.byref(lo), ctypes.byref(hi),
                                              ctypes.byref(pairs), ctypes.byref(fl)))
        return {"leaf_lo": lo.value, "leaf_hi": hi.value, "pairs": pairs.value, "flops_per_rhs": fl.value}

    def local_phase(self, ud, R: int):
        """Permute + upward of the own clusters into the exchange buffers."""
        import torch
        bufs = self.exchange_buffers(R)
        with torch.cuda.device(self.device):
            st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
            _lib.check(_lib.lib().htlr_matvec_local(self.local._plan, ctypes.c_void_p(ud.data_ptr()), R, st))
        return bufs

    def contract_phase(self, ud, R: int):
        """GEMMs / regenerated blocks of the own targets into the
        accumulators; returns the buffers to sum over the shards (maybe [])."""
        import torch
        self.exchange_buffers(R)
        rbufs = self.reduce_buffers(R)
        with torch.cuda.device(self.device):
            st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
            _lib.check(_lib.lib().htlr_matvec_contract(self.local._plan, ctypes.c_void_p(ud.data_ptr()), R, st))
        return rbufs

    def expand_phase(self, ud, fd, R: int):
        """Downward pass of the own leaf boxes into fd."""
        import torch
        self.exchange_buffers(R)
        self.reduce_buffers(R)
        with torch.cuda.device(self.device):
            st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
            _lib.check(_lib.lib().htlr_matvec_expand(self.local._plan, ctypes.c_void_p(ud.data_ptr()),
                                                     ctypes.c_void_p(fd.data_ptr()), R, st))

    def remote_begin(self, ud, R: int):
        """Zero the accumulators and apply the blocks whose sources this shard
        owns (separable plans): reads only the own chunks of the exchange
        buffers, so it runs while the all-gather is in flight."""
        import torch
        self.exchange_buffers(R)
        with torch.cuda.device(self.device):
            st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
            _lib.check(_lib.lib().htlr_matvec_remote_begin(self.local._plan, ctypes.c_void_p(ud.data_ptr()), R, st))

    def remote_finish(self, ud, fd, R: int):
        """After the exchange: the remaining blocks and the downward pass."""
        import torch
        self.exchange_buffers(R)
        with torch.cuda.device(self.device):
            st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
            _lib.check(_lib.lib().htlr_matvec_remote_finish(self.local._plan, ctypes.c_void_p(ud.data_ptr()),
                                                            ctypes.c_void_p(fd.data_ptr()), R, st))

    def remote_phase(self, ud, fd, R: int, reduce=None):
        """GEMMs of the own targets + downward of the own leaf boxes.  A
        sharded symmetric plan sums its accumulators over the shards in
        between: NCCL reduce-scatter, or `reduce(self, bufs)` (tests)."""
        rbufs = self.contract_phase(ud, R)
        if rbufs:
            if reduce is not None:
                reduce(self, rbufs)
            else:
                reduce_scatter_chunks(rbufs, self.rank, self.world, self.group)
        self.expand_phase(ud, fd, R)

    def matmat(self, U, exchange=None):
        """F rows of this shard's leaf boxes (other rows 0).  `exchange`
        replaces the NCCL all-gather (used by single-GPU tests)."""
        import torch
        host = not (isinstance(U, torch.Tensor) and U.is_cuda)
        x = U if isinstance(U, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(U, dtype=np.float64))
        vec = x.dim() == 1
        x2 = x.reshape(-1, 1) if vec else x
        if x2.shape[0] != self.grid.num_points:
            raise ValueError(f"vector length {x2.shape[0]} != {self.grid.num_points}")
        R = int(x2.shape[1])
        ud = x2.to(f"cuda:{self.device}", dtype=torch.float64, non_blocking=True).contiguous()
        fd = torch.zeros_like(ud)
        bufs = self.exchange_buffers(R)
        L = _lib.lib()
        import torch.distributed as dist
        if self.mode == "zslab":
            # own slab's upward contributions, summed over the ranks, then the
            # banded passes and the downward pass of the own slab
            nccl = self.world > 1 and dist.get_backend(self.group) == "nccl"
            out = None
            if exchange is None and self.graphs and (nccl or self.world == 1):
                try:
                    out = self._zslab_graph(ud, R)
                except RuntimeError:   # a collective that cannot be captured: direct launches from now on
                    self.graphs = False
                    self._graphs = {}
                    torch.cuda.synchronize(self.device)
            if out is None:
                self.local_phase(ud, R)
                if exchange is not None:
                    exchange(self, bufs)
                elif self.world > 1:
                    allreduce_sum(bufs, self.group)
                self.remote_phase(ud, fd, R)
                out = fd
            out = out.reshape(-1) if vec else out
            return out.cpu() if host else out
        overlap = exchange is None and self.world > 1 and not self.reduce_buffers(R)
        with torch.cuda.device(self.device):
            st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
            _lib.check(L.htlr_matvec_local(self.local._plan, ctypes.c_void_p(ud.data_ptr()), R, st))
            if overlap:
                # the all-gather overlaps the blocks over own sources (NCCL:
                # asynchronous collective; other backends: the same order,
                # exchange in between -- the gloo harness runs this flow)
                if dist.get_backend(self.group) == "nccl":
                    works = allgather_chunks_async(bufs, self.rank, self.world, self.group)
                    self.remote_begin(ud, R)
                    for w in works:
                        w.wait()
                else:
                    self.remote_begin(ud, R)
                    torch.cuda.current_stream().synchronize()
                    allgather_chunks(bufs, self.rank, self.world, self.group)
                self.remote_finish(ud, fd, R)
            else:
                if exchange is not None:
                    exchange(self, bufs)
                elif self.world > 1:
                    allgather_chunks(bufs, self.rank, self.world, self.group)
        if not overlap:
            self.remote_phase(ud, fd, R)
        out = fd.reshape(-1) if vec else fd
        return out.cpu() if host else out

    def matvec(self, u, exchange=None):
        return self.matmat(u, exchange)
