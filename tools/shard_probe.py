"""Sharded matvec, emulated on one GPU (dev tool): per shard, the local phase
and the remote phase timed alone with CUDA events (the exchange between them
replayed as device copies / sums), and the union of the shards' f against
the single-GPU matvec.  Reports per-shard time against unsharded / world.

    python tools/shard_probe.py [cfg4] [mode: auto|subtree|zslab]
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2508_05958_b200 as H  # noqa: E402
from paper_2508_05958_b200.configs import WORKLOADS  # noqa: E402
from paper_2508_05958_b200.multi import ShardedOperator  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
mode = sys.argv[2] if len(sys.argv) > 2 else "auto"
w = WORKLOADS[name]
cfg, grid = w.build_config(), w.grid
U = torch.from_numpy(np.ascontiguousarray(w.input())).cuda().reshape(grid.num_points, -1)
R = U.shape[1]
single = H.construct(cfg, grid)
ref = H.matmat(single, U).cpu().numpy()


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


unsharded = timed(lambda: H.matmat(single, U))
print(json.dumps({"workload": name, "unsharded_ms": unsharded}), flush=True)
for world in (2, 4, 8):
    ops = [ShardedOperator(cfg, grid, r, world, device=0, mode=mode) for r in range(world)]
    bufs = [op.local_phase(U, R) for op in ops]
    for i in range(len(bufs[0])):
        if ops[0].exchange_sums:
            tot = sum(b[i] for b in bufs)
            for b in bufs:
                b[i].copy_(tot)
        else:
            c = bufs[0][i].numel() // world
            for r in range(world):
                for q in range(world):
                    if q != r:
                        bufs[q][i][r * c:(r + 1) * c].copy_(bufs[r][i][r * c:(r + 1) * c])
    total = torch.zeros_like(U)
    loc, rem = [], []
    for op in ops:
        fd = torch.zeros_like(U)
        op.remote_phase(U, fd, R)
        total += fd
        saved = [b.clone() for b in op.exchange_buffers(R)]
        loc.append(timed(lambda: op.local_phase(U, R)))
        for b, sv in zip(op.exchange_buffers(R), saved):   # the exchanged values back
            b.copy_(sv)
        rem.append(timed(lambda: op.remote_phase(U, fd, R)))
    err = np.linalg.norm(total.cpu().numpy() - ref) / np.linalg.norm(ref)
    per = max(a + b for a, b in zip(loc, rem))
    xbytes = sum(b.numel() * 8 for b in bufs[0])
    print(json.dumps({"world": world, "mode": ops[0].mode, "leaf_pass": ops[0].local.leaf_pass(),
                      "local_ms_max": max(loc), "remote_ms_max": max(rem), "per_shard_ms": per,
                      "ideal_ms": unsharded / world, "ratio_to_ideal": per / (unsharded / world),
                      "exchange_bytes": xbytes, "exchange": "sum" if ops[0].exchange_sums else "gather",
                      "rel_err_vs_single": float(err)}), flush=True)

# per-launch breakdown of one shard's phases (world 8, rank 0)
ops = [ShardedOperator(cfg, grid, r, 8, device=0, mode=mode) for r in range(8)]
op = ops[0]
fd = torch.zeros_like(U)
op.local_phase(U, R)
op.remote_phase(U, fd, R)
op.local.profile(True)
op.local_phase(U, R)
op.remote_phase(U, fd, R)
torch.cuda.synchronize()
recs = op.local.profile_read()
op.local.profile(False)
print(json.dumps({"world": 8, "rank": 0, "launches": [(r["phase"], r["level"], round(r["ms"], 4)) for r in recs]}))
