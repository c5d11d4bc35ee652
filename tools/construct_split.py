"""Per-call timing of construct's C-ABI sequence (dev tool)."""
import ctypes
import sys
import time

import torch

from paper_2508_05958_b200 import _lib
from paper_2508_05958_b200.configs import WORKLOADS
from paper_2508_05958_b200.operators import HTLRMatrix

for name in sys.argv[1:] or ["cfg5"]:
    w = WORKLOADS[name]
    cfg = w.build_config()
    for rep in range(2):
        torch.cuda.synchronize()
        t = [time.perf_counter()]
        op = HTLRMatrix(w.grid, cfg, 0)
        t.append(time.perf_counter())
        _lib.check(_lib.lib().htlr_build_lists(op._plan))
        t.append(time.perf_counter())
        _lib.check(_lib.lib().htlr_construct(op._plan, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        del op
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        print(name, "create %.3f lists %.3f construct %.3f destroy %.3f" % tuple(b - a for a, b in zip(t, t[1:])))
