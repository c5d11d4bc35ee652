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


def emulate(cfg, grid, U, world):
    ops = [ShardedOperator(cfg, grid, r, world, device=0) for r in range(world)]
    ud = torch.from_numpy(np.ascontiguousarray(U)).cuda()
    ud2 = ud.reshape(grid.num_points, -1)
    R = ud2.shape[1]
    bufs = [op.local_phase(ud2, R) for op in ops]
    for i in range(len(bufs[0])):
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
    ops = [ShardedOperator(cfg, grid, r, world, device=0) for r in range(world)]
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
    op = ShardedOperator(cfg, grid, 0, 2, device=0)
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
