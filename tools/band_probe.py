"""Banded vs cooperative leaf pass: equality and matvec time (one process per
mode; HTLR_SEP_BAND decides).  Usage: python tools/band_probe.py N [R]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_05958_b200 as H  # noqa: E402

n = int(sys.argv[1])
R = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = H.BuildConfig(rank=8, leaf_side=8, rule=H.AdmissibilityRule.strong(1.0), kernel=H.gaussian(0.1),
                    coeff=H.CoefficientFn.constant(0.0))
op = H.construct(cfg, H.UniformGrid(3, n))
U = torch.from_numpy(np.random.default_rng(7).standard_normal((n ** 3, R))).cuda()
F = H.matmat(op, U)
torch.cuda.synchronize()
t = []
for _ in range(20):
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    H.matmat(op, U, out=F)
    b.record()
    torch.cuda.synchronize()
    t.append(a.elapsed_time(b))
out = sys.argv[3] if len(sys.argv) > 3 else None
if out:
    np.save(out, F.cpu().numpy())
print(f"n={n} R={R} leaf_pass={op.leaf_pass()} matvec ms median {np.median(t):.4f} min {min(t):.4f}")
