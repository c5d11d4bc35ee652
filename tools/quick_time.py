"""Quick timing of construct + matvec per BASELINE config (dev tool)."""
import sys
import time

import numpy as np
import torch

import paper_2508_05958_b200 as H
from paper_2508_05958_b200.configs import WORKLOADS

names = sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "cfg4"]
for name in names:
    w = WORKLOADS[name]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    op = H.construct(w.build_config(), w.grid)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    u = torch.from_numpy(w.input()).cuda()
    f = H.matmat(op, u) if w.nrhs > 1 else H.matvec(op, u)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    ev0.record()
    for _ in range(reps):
        f = H.matmat(op, u) if w.nrhs > 1 else H.matvec(op, u)
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / reps
    rep = H.storage_report(op)
    print(f"{name}: construct {t1 - t0:.3f}s matvec {ms:.3f} ms  points/s {w.grid.num_points * w.nrhs / ms * 1e3:.3e}"
          f"  device GB {rep.device_scalars * 8 / 1e9:.2f}  launches {op.last_launch_count()}", flush=True)
