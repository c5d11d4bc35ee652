"""Sharded banded passes, emulated on one GPU: each shard's remote phase timed
alone (after the exchange), and the union of the shards' f against the
single-GPU matvec.  Usage: python tools/shard_probe.py [cfg4]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2508_05958_b200 as H  # noqa: E402
from paper_2508_05958_b200.configs import WORKLOADS  # noqa: E402
from paper_2508_05958_b200.multi import ShardedOperator  # noqa: E402

w = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cfg4"]
cfg, grid = w.build_config(), w.grid
U = torch.from_numpy(np.ascontiguousarray(w.input())).cuda().reshape(grid.num_points, -1)
R = U.shape[1]
single = H.construct(cfg, grid)
ref = H.matmat(single, U).cpu().numpy()
for world in (2, 4, 8):
    ops = [ShardedOperator(cfg, grid, r, world, device=0) for r in range(world)]
    bufs = [op.local_phase(U, R) for op in ops]
    for i in range(len(bufs[0])):
        c = bufs[0][i].numel() // world
        for r in range(world):
            for q in range(world):
                if q != r:
                    bufs[q][i][r * c:(r + 1) * c].copy_(bufs[r][i][r * c:(r + 1) * c])
    total = torch.zeros_like(U)
    ms = []
    for op in ops:
        fd = torch.zeros_like(U)
        for _ in range(3):
            op.remote_phase(U, fd, R)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            op.remote_phase(U, fd, R)
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b) / 10)
        total += fd
    err = np.linalg.norm(total.cpu().numpy() - ref) / np.linalg.norm(ref)
    print(f"world {world}: leaf pass {ops[0].local.leaf_pass()}, remote phase ms per shard "
          f"{min(ms):.4f}..{max(ms):.4f}, rel err vs single {err:.2e}")
