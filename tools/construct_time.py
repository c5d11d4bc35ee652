"""Construction time split (dev tool): host list build vs the whole construct."""
import ctypes
import sys
import time

import torch

import paper_2508_05958_b200 as H
from paper_2508_05958_b200 import _lib
from paper_2508_05958_b200.configs import WORKLOADS
from paper_2508_05958_b200.operators import _desc

for name in sys.argv[1:] or ["cfg4"]:
    w = WORKLOADS[name]
    cfg = w.build_config()
    torch.cuda.synchronize()
    op = None
    for rep in range(2):
        del op   # the previous plan's teardown stays outside the timed region
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        op = H.construct(cfg, w.grid)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
    L = _lib.lib()
    plan = ctypes.c_void_p()
    _lib.check(L.htlr_plan_create(ctypes.byref(_desc(cfg, w.grid)), -1, ctypes.byref(plan)))
    t2 = time.perf_counter()
    _lib.check(L.htlr_build_lists(plan))
    t3 = time.perf_counter()
    L.htlr_plan_destroy(plan)
    print(f"{name}: construct {t1 - t0:.3f} s ({w.grid.num_points / (t1 - t0):.3e} points/s), "
          f"of which host lists {t3 - t2:.3f} s", flush=True)
