"""Multi-process (world_size 2, gloo, CPU) tests of the sharded path's host
logic: shard ownership from the C++ plan (host-only, no device), balance and
coverage of the target lists, the all-gather exchange of Morton-contiguous
chunks used between the local and remote phases, and the sum-reduce-scatter
of the symmetric mapped path."""

import ctypes
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def host_shard(rank, world, d=3, n=64, leaf=8, rank_p=6):
    from paper_2508_05958_b200 import _lib
    L = _lib.lib()
    desc = _lib.HtlrDesc(d=d, n=n, leaf_side_max=leaf, rank=rank_p, rule=1, eta=1.0, kernel=2, sigma=0.0,
                         scale=1.0, quad_q=10, corner_subdivision=1, coeff_const=0.0)
    plan = ctypes.c_void_p()
    _lib.check(L.htlr_plan_create(ctypes.byref(desc), -1, ctypes.byref(plan)))
    try:
        _lib.check(L.htlr_set_shard(plan, rank, world))
        _lib.check(L.htlr_build_lists(plan))
        lo, hi, pairs, fl = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_double()
        _lib.check(L.htlr_shard_info(plan, ctypes.byref(lo), ctypes.byref(hi), ctypes.byref(pairs), ctypes.byref(fl)))
        cnt = ctypes.c_int64()
        _lib.check(L.htlr_exchange_info(plan, 1, ctypes.byref(cnt), None, 0))
        sizes = np.zeros(cnt.value, dtype=np.int64)
        _lib.check(L.htlr_exchange_info(plan, 1, ctypes.byref(cnt), sizes.ctypes.data, cnt.value))
        return lo.value, hi.value, pairs.value, fl.value, sizes
    finally:
        L.htlr_plan_destroy(plan)


def worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import sys
    sys.path.insert(0, ROOT)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2508_05958_b200.multi import allgather_chunks, reduce_scatter_chunks
    lo, hi, pairs, fl, sizes = host_shard(rank, world)
    # exchange: every rank fills its own chunk, the all-gather completes the rest
    bufs = [torch.full((int(b) // 8,), -1.0, dtype=torch.float64) for b in sizes]
    for b in bufs:
        c = b.numel() // world
        b[rank * c:(rank + 1) * c] = torch.arange(c, dtype=torch.float64) + 1000.0 * rank
    allgather_chunks(bufs, rank, world)
    ok = True
    for b in bufs:
        c = b.numel() // world
        for r in range(world):
            ok &= bool(torch.equal(b[r * c:(r + 1) * c], torch.arange(c, dtype=torch.float64) + 1000.0 * r))
    # reduction of the symmetric mapped path: every rank adds into all rows,
    # afterwards its own chunk holds the sum over the ranks
    red = [torch.arange(12 * world, dtype=torch.float64) * (rank + 1) for _ in range(2)]
    reduce_scatter_chunks(red, rank, world)
    tot = sum(r + 1 for r in range(world))
    for b in red:
        c = b.numel() // world
        ok &= bool(torch.equal(b[rank * c:(rank + 1) * c],
                               torch.arange(rank * c, (rank + 1) * c, dtype=torch.float64) * tot))
    t = torch.tensor([lo, hi, pairs, fl, float(ok)], dtype=torch.float64)
    gathered = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(gathered, t)
    if rank == 0:
        out.put([g.tolist() for g in gathered])
    dist.destroy_process_group()


def test_gloo_two_shards():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (lo0, hi0, pr0, fl0, ok0), (lo1, hi1, pr1, fl1, ok1) = res
    assert ok0 == 1.0 and ok1 == 1.0
    assert lo0 == 0 and hi0 == lo1 and hi1 == 512          # 8^3 leaf boxes, contiguous halves
    assert pr0 == pr1 and fl0 == fl1                        # mirror-symmetric halves
    # union of the shards' target lists is the whole interaction list
    full = host_shard(0, 1)
    assert pr0 + pr1 == full[2]


@pytest.mark.parametrize("world", [2, 4, 8])
def test_shard_lists_partition_all_pairs(world):
    full = host_shard(0, 1, n=32, leaf=4, rank_p=4)
    parts = [host_shard(r, world, n=32, leaf=4, rank_p=4) for r in range(world)]
    assert sum(p[2] for p in parts) == full[2]
    assert len({p[2] for p in parts}) == 1
    edges = [(p[0], p[1]) for p in parts]
    assert edges[0][0] == 0 and edges[-1][1] == 8 ** 3
    assert all(a[1] == b[0] for a, b in zip(edges, edges[1:]))
