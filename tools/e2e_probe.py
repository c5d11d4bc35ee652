"""Where does the e2e time go? (dev tool)"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2508_05958_b200 as H  # noqa: E402
from paper_2508_05958_b200.configs import WORKLOADS  # noqa: E402

w = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cfg4"]
op = H.construct(w.build_config(), w.grid)
u = np.ascontiguousarray(w.input())
up = torch.from_numpy(u).pin_memory()
ud = up.cuda()


def timeit(label, fn, reps=10, pre=None):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if pre is not None:
            pre()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append((e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3))
    print(label, "device ms %.3f  wall ms %.3f" % tuple(np.median(np.array(ts), axis=0)), flush=True)


timeit("device in/out      ", lambda: H.matvec(op, ud))
timeit("h2d only           ", lambda: up.to("cuda", non_blocking=True))
out = torch.empty_like(ud)
timeit("d2h pinned only    ", lambda: torch.empty(out.shape, dtype=out.dtype, pin_memory=True).copy_(out, non_blocking=True))
timeit("pinned in/out      ", lambda: H.matvec(op, up))
timeit("numpy in/out       ", lambda: H.matvec(op, u))
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
keep = [None]


def kept():
    keep[0] = H.matvec(op, up)


timeit("pinned, result kept ", kept)
timeit("pinned, L2 flushed  ", lambda: H.matvec(op, up), pre=flush.zero_)
timeit("kept + flushed      ", kept, pre=flush.zero_)
