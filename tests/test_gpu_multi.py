"""Sharded (multi-GPU) matvec, emulated on one GPU: every shard's plan runs
its local phase, the all-gather is replayed as device copies of each shard's
contiguous chunk, then every shard runs its remote phase.  The union of the
shards' f rows must equal the single-GPU matvec.  (The NCCL plumbing itself
is covered by tests/test_multi_gloo.py on CPU.)"""

import numpy as np
import pytest
import torch

import paper_2508_05958_b200 as H
from paper_2508_05958_b200.configs import WORKLOADS
from paper_2508_05958_b200.multi import ShardedOperator

pytestmark = pytest.mark.gpu


def emulate(cfg, grid, U, world, mode="subtree"):
    ops = [ShardedOperator(cfg, grid, r, world, device=0, mode=mode) for r in range(world)]
    ud = torch.from_numpy(np.ascontiguousarray(U)).cuda()
    ud2 = ud.reshape(grid.num_points, -1)
    R = ud2.shape[1]
    bufs = [op.local_phase(ud2, R) for op in ops]
    for i in range(len(bufs[0])):
        if ops[0].exchange_sums:   # z-slab shards: the NCCL all-reduce (sum)
            tot = sum(b[i] for b in bufs)
            for r in range(world):
                bufs[r][i].copy_(tot)
            continue
        n = bufs[0][i].numel()
        c = n // world
        for r in range(world):
            for q in range(world):
                if q != r:
                    bufs[q][i][r * c:(r + 1) * c].copy_(bufs[r][i][r * c:(r + 1) * c])
    total = torch.zeros_like(ud2)
    infos = []
    for op in ops:
        fd = torch.zeros_like(ud2)
        op.remote_phase(ud2, fd, R)
        total += fd
        infos.append(op.shard_info())
    torch.cuda.synchronize()
    return total.cpu().numpy().reshape(U.shape), infos


def emulate_split(cfg, grid, U, world):
    """The overlapped remote phase: remote_begin runs before the exchange
    with every non-own chunk of the exchange buffers poisoned with NaN (so it
    provably reads own sources only), then the chunks are exchanged and
    remote_finish completes the matvec."""
    ops = [ShardedOperator(cfg, grid, r, world, device=0, mode="subtree") for r in range(world)]
    ud = torch.from_numpy(np.ascontiguousarray(U)).cuda()
    ud2 = ud.reshape(grid.num_points, -1)
    R = ud2.shape[1]
    bufs = [op.local_phase(ud2, R) for op in ops]
    for r, op in enumerate(ops):
        for b in bufs[r]:
            c = b.numel() // world
            keep = b[r * c:(r + 1) * c].clone()
            b.fill_(float("nan"))
            b[r * c:(r + 1) * c].copy_(keep)
        op.remote_begin(ud2, R)
    for i in range(len(bufs[0])):
        c = bufs[0][i].numel() // world
        for r in range(world):
            for q in range(world):
                if q != r:
                    bufs[q][i][r * c:(r + 1) * c].copy_(bufs[r][i][r * c:(r + 1) * c])
    total = torch.zeros_like(ud2)
    for op in ops:
        fd = torch.zeros_like(ud2)
        op.remote_finish(ud2, fd, R)
        total += fd
    torch.cuda.synchronize()
    return total.cpu().numpy().reshape(U.shape)


@pytest.mark.parametrize("name,world", [("cfg4", 8), ("cfg4", 2), ("cfg2", 4)])
def test_sharded_overlapped_exchange(name, world):
    """remote_begin (own sources, before the exchange) + remote_finish equals
    the single-GPU matvec; config 4 is separable (own / remote parts), config
    2 dense (begin only zeroes)."""
    w = WORKLOADS[name]
    cfg, grid = w.build_config(), w.grid
    U = w.input()
    single = H.construct(cfg, grid)
    ref = H.matmat(single, U) if U.ndim == 2 else H.matvec(single, U)
    got = emulate_split(cfg, grid, U, world)
    assert np.isfinite(got).all()
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert err <= 1e-13, err


@pytest.mark.parametrize("name,world", [("cfg2", 2), ("cfg2", 8), ("cfg3", 4), ("cfg4", 8), ("cfg4", 2), ("cfg4", 4)])
def test_sharded_equals_single(name, world):
    w = WORKLOADS[name]
    cfg, grid = w.build_config(), w.grid
    U = w.input()
    single = H.construct(cfg, grid)
    ref = H.matmat(single, U) if U.ndim == 2 else H.matvec(single, U)
    got, infos = emulate(cfg, grid, U, world)
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert err <= 1e-13
    # octants are reflections of each other: identical work per shard
    assert len({i["pairs"] for i in infos}) == 1
    leaves = sorted((i["leaf_lo"], i["leaf_hi"]) for i in infos)
    assert leaves[0][0] == 0 and all(a[1] == b[0] for a, b in zip(leaves, leaves[1:]))


@pytest.mark.parametrize("world", [2, 4, 8])
def test_zslab_shards_equal_single(world):
    """z-slab shards of the banded config-4 plan (htlr_set_zslab): each shard
    sums its slab's upward contributions into W_l, the W_l are summed over
    the shards (NCCL all-reduce, replayed here), then each shard runs the
    banded passes, the downward pass and writes the f rows of its z slab
    (a contiguous block of the F-order f) -- together the single-GPU matvec."""
    w = WORKLOADS["cfg4"]
    cfg, grid = w.build_config(), w.grid
    U = w.input()
    single = H.construct(cfg, grid)
    ref = H.matvec(single, U)
    ops = [ShardedOperator(cfg, grid, r, world, device=0, mode="zslab") for r in range(world)]
    assert all(op.mode == "zslab" and op.exchange_sums for op in ops)
    ud = torch.from_numpy(np.ascontiguousarray(U)).cuda().reshape(-1, 1)
    bufs = [op.local_phase(ud, 1) for op in ops]
    for i in range(len(bufs[0])):
        tot = sum(b[i] for b in bufs)
        for b in bufs:
            b[i].copy_(tot)
    n = grid.n
    rows = n * n * n // world
    total = torch.zeros_like(ud)
    for r, op in enumerate(ops):
        fd = torch.zeros_like(ud)
        op.remote_phase(ud, fd, 1)
        f = fd.reshape(-1)
        # only the own z slab is written
        assert float(f[:r * rows].abs().sum()) == 0.0 and float(f[(r + 1) * rows:].abs().sum()) == 0.0
        total += fd
    err = np.linalg.norm(total.cpu().numpy().ravel() - ref) / np.linalg.norm(ref)
    assert err <= 1e-13, err


def test_sharded_2d_weak_rejects_uneven_levels():
    grid = H.UniformGrid(2, 32)
    cfg = H.BuildConfig(rank=8, leaf_side=8, rule=H.AdmissibilityRule.weak(),
                        kernel=H.gaussian(1.0), coeff=H.CoefficientFn.constant(0.0))
    with pytest.raises(ValueError):
        ShardedOperator(cfg, grid, 0, 8, device=0)


def test_profiling_on_direct_launches():
    """Per-launch profiling works where the matvec is launched directly (a
    sharded plan's local / remote phases, or graphs switched off), not only
    inside graph capture: the harness of `bench.py --gpus N` profiles that
    way."""
    w = WORKLOADS["cfg2"]
    cfg, grid = w.build_config(), w.grid
    op = ShardedOperator(cfg, grid, 0, 2, device=0, mode="subtree")
    ud = torch.from_numpy(np.ascontiguousarray(w.input())).cuda().reshape(grid.num_points, 1)
    op.local.profile(True)
    op.local_phase(ud, 1)
    fd = torch.zeros_like(ud)
    op.remote_phase(ud, fd, 1)
    recs = op.local.profile_read()
    op.local.profile(False)
    assert recs and all(r["ms"] >= 0 for r in recs)
    single = H.construct(cfg, grid)
    H._lib.check(H._lib.lib().htlr_set_graphs(single._plan, 0))
    single.profile(True)
    H.matvec(single, w.input())
    assert single.profile_read()


def test_zslab_graph_replay():
    """The NCCL z-slab path replays one CUDA graph per RHS count of [local
    phase, all-reduce, remote phase]; at world 1 (no collective: this run has
    one GPU) the captured phases equal the plain matvec on capture and on
    replay, and a new input reaches the graph through its staging copy."""
    w = WORKLOADS["cfg4"]
    cfg, grid = w.build_config(), w.grid
    single = H.construct(cfg, grid)
    op = ShardedOperator(cfg, grid, 0, 1, device=0, mode="zslab")
    for seed in (0, 0, 1):
        u = np.random.default_rng(seed).uniform(-1, 1, grid.num_points)
        ref = H.matvec(single, u)
        got = op.matvec(torch.from_numpy(u).cuda()).cpu().numpy()
        assert np.linalg.norm(got - ref) <= 1e-13 * np.linalg.norm(ref)
    assert op.graphs and 1 in op._graphs
