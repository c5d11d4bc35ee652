"""A/B of the direct-f matvec (HTLR_FDIRECT, htlr_plan.cu mv_remote) on one GPU:
the same plan applied with the downward pass after the leaf pass (0) and beside
it (1); prints the difference of the results and the time per matvec."""
import os
import subprocess
import sys

import numpy as np

if len(sys.argv) > 1 and sys.argv[1] == "child":
    import torch
    import paper_2508_05958_b200 as H
    from paper_2508_05958_b200.configs import WORKLOADS
    name = sys.argv[2]
    w = WORKLOADS[name]
    op = H.construct(w.build_config(), w.grid)
    u = torch.from_numpy(np.ascontiguousarray(w.input())).cuda()
    f = H.matvec(op, u)
    torch.cuda.synchronize()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
    best = []
    for cold in (0, 1):
        ts = []
        for _ in range(30):
            if cold:
                flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            f = H.matvec(op, u)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        best.append((ts[0], ts[len(ts) // 2]))
    np.save(sys.argv[3], f.cpu().numpy())
    print(f"{name} HTLR_FDIRECT={os.environ.get('HTLR_FDIRECT', '1')}: warm min/median {best[0][0]:.4f}/{best[0][1]:.4f} ms, "
          f"L2-flushed min/median {best[1][0]:.4f}/{best[1][1]:.4f} ms, launches {op.last_launch_count()}", flush=True)
    sys.exit(0)

for name in sys.argv[1:] or ["cfg4"]:
    outs = []
    for mode in os.environ.get("AB_MODES", "0,1").split(","):
        env = dict(os.environ, HTLR_FDIRECT=mode[0], PYTHONPATH=os.getcwd())
        out = f"/tmp/fdirect_{name}_{mode}.npy"
        subprocess.run([sys.executable, __file__, "child", name, out], env=env, check=True)
        outs.append(np.load(out))
    d = np.linalg.norm(outs[0] - outs[1]) / np.linalg.norm(outs[0])
    print(f"{name}: rel diff between the two formulations {d:.3e}", flush=True)
