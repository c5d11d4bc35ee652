"""Device time of the overlapped host-vector schedule with DEVICE vectors
(HTLR_HOST_DEVICE_OK=1): the cost of the split launches without the PCIe
copies, against the one-graph device matvec (dev tool)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2508_05958_b200 as H  # noqa: E402
from paper_2508_05958_b200 import _lib  # noqa: E402
from paper_2508_05958_b200.configs import WORKLOADS  # noqa: E402

w = WORKLOADS["cfg4"]
op = H.construct(w.build_config(), w.grid)
u = torch.from_numpy(w.input()).cuda()
f = torch.empty_like(u)


def split():
    _lib.check(_lib.lib().htlr_matvec_host(op._plan, ctypes.c_void_p(u.data_ptr()), ctypes.c_void_p(f.data_ptr()), 1,
                                           ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))


def whole():
    H.matvec(op, u)


for name, fn in (("one graph", whole), ("split schedule", split)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) / 20:.4f} ms")
ref = H.matvec(op, u)
split()
torch.cuda.synchronize()
print("max rel diff", float((f - ref).norm() / ref.norm()))
