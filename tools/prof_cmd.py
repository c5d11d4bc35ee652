"""Short command for ncu captures: construct a workload, warm up, run N matvecs."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2508_05958_b200 as H  # noqa: E402
from paper_2508_05958_b200.configs import WORKLOADS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
w = WORKLOADS[name]
op = H.construct(w.build_config(), w.grid)
u = torch.from_numpy(np.ascontiguousarray(w.input())).cuda()
for _ in range(2 + reps):
    f = H.matmat(op, u) if w.nrhs > 1 else H.matvec(op, u)
torch.cuda.synchronize()
print("ok", float(f.abs().sum()))
