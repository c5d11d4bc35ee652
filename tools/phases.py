"""Per-phase device times of one workload's matvec (dev tool for A/B runs):
    python tools/phases.py cfg4 [reps]
prints the formulation, the graph-replayed matvec time (CUDA events, L2 not
flushed) and the per-launch profile of the last profiled matvec."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2508_05958_b200 as H  # noqa: E402
from paper_2508_05958_b200.configs import WORKLOADS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
w = WORKLOADS[name]
op = H.construct(w.build_config(), w.grid)
u = torch.from_numpy(np.ascontiguousarray(w.input())).cuda()


def run():
    return H.matmat(op, u) if w.nrhs > 1 else H.matvec(op, u)


for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    run()
e1.record()
torch.cuda.synchronize()
print(f"{name} [{op.formulation()}] matvec {e0.elapsed_time(e1) / reps:.4f} ms")
op.profile(True)
acc = {}
for _ in range(reps):
    run()
    for rec in op.profile_read():
        key = f"{rec['phase']}_L{rec['level']}"
        acc[key] = acc.get(key, 0.0) + rec["ms"] / reps
op.profile(False)
for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    print(f"  {k:16s} {v:.4f} ms")
