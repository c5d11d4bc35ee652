"""z-slab shard phases replayed from a CUDA graph (dev tool): separates the
GPU time of one shard's matvec from the host launch overhead of the direct
(uncaptured) local / remote calls.  python tools/shard_graph_probe.py"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2508_05958_b200.configs import WORKLOADS  # noqa: E402
from paper_2508_05958_b200.multi import ShardedOperator  # noqa: E402

w = WORKLOADS["cfg4"]
cfg, grid = w.build_config(), w.grid
U = torch.from_numpy(np.ascontiguousarray(w.input())).cuda().reshape(-1, 1)
for world in (1, 2, 4, 8):
    op = ShardedOperator(cfg, grid, 0, world, device=0, mode="zslab")
    fd = torch.zeros_like(U)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            op.local_phase(U, 1)
            op.remote_phase(U, fd, 1)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        op.local_phase(U, 1)
        op.remote_phase(U, fd, 1)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    print(json.dumps({"world": world, "graph_ms_per_shard_matvec": a.elapsed_time(b) / 20}), flush=True)
