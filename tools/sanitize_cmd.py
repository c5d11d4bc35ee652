"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
config 2 (dense cores, gathered GEMMs, generated near blocks), a banded
separable n = 64 plan (upward8, band line/plane kernels with the TMEM
accumulator, downward8), its z-slab shards (pair units, y/x line kernels),
and a small mapped plan (regeneration kernels).  One matvec each.
    compute-sanitizer --tool memcheck python tools/sanitize_cmd.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2508_05958_b200 as H  # noqa: E402
from paper_2508_05958_b200.configs import WORKLOADS  # noqa: E402
from paper_2508_05958_b200.multi import ShardedOperator  # noqa: E402

w = WORKLOADS["cfg2"]
op = H.construct(w.build_config(), w.grid)
f2 = H.matvec(op, torch.from_numpy(w.input()).cuda())
cfg = H.BuildConfig(rank=8, leaf_side=8, rule=H.AdmissibilityRule.strong(1.0), kernel=H.gaussian_bw(0.1),
                    coeff=H.CoefficientFn.constant(0.0))
grid = H.UniformGrid(3, 64)
band = H.construct(cfg, grid)
assert band.leaf_pass() == "banded"
u = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, 64 ** 3)).cuda()
fb = H.matvec(band, u)
shards = [ShardedOperator(cfg, grid, r, 4, device=0, mode="zslab") for r in range(4)]
ud = u.reshape(-1, 1)
bufs = [s.local_phase(ud, 1) for s in shards]
for i in range(len(bufs[0])):
    tot = sum(b[i] for b in bufs)
    for b in bufs:
        b[i].copy_(tot)
total = torch.zeros_like(ud)
for s in shards:
    fd = torch.zeros_like(ud)
    s.remote_phase(ud, fd, 1)
    total += fd
err = float((total.reshape(-1) - fb).norm() / fb.norm())
mcfg = H.BuildConfig(rank=6, leaf_side=6, rule=H.AdmissibilityRule.strong(1.0), kernel=H.inv_r_3d(),
                     coeff=H.CoefficientFn.constant(0.0))
mop = H.construct(mcfg, H.MappedGrid(3, 24, 0.05))
fm = H.matvec(mop, torch.from_numpy(np.random.default_rng(1).standard_normal(24 ** 3)).cuda())
torch.cuda.synchronize()
print("sanitize workload ok", float(f2.norm()), float(fb.norm()), err, float(fm.norm()))
