"""Randomised parity sweep (dev tool): random small problems -- dimension,
grid, leaf side, rank, admissibility, kernel, coefficient, RHS count,
uniform or mapped grid -- against the oracle's full matvec.  Prints one line
per case and the worst relative error; exits 1 above 1e-12."""
import sys
import warnings

import numpy as np

sys.path.insert(0, ".")
import paper_2508_05958_b200 as H  # noqa: E402
from oracle import htlr_oracle as O  # noqa: E402

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
ncases = int(sys.argv[2]) if len(sys.argv) > 2 else 40
worst = 0.0
for case in range(ncases):
    d = int(rng.choice([2, 3]))
    leaf = int(rng.choice([4, 5, 6, 8]) if d == 3 else rng.choice([4, 6, 8, 16]))
    levels = int(rng.integers(1, 3 if d == 3 else 5))
    n = leaf * 2 ** levels
    rank = int(rng.integers(2, min(leaf, 8) + 1))
    rule = str(rng.choice(["weak", "strong"]))
    eta = float(rng.choice([0.7, 1.0, 1.5])) if rule == "strong" else None
    kind = str(rng.choice(["gaussian", "slp"]))
    a = float(rng.choice([0.0, 0.5]))
    R = int(rng.choice([1, 1, 2, 3, 17]))
    mapped = bool(rng.random() < 0.3) and kind == "slp"
    if kind == "gaussian":
        sig = float(rng.choice([0.1, 0.3]))
        ko, kd = O.Kernel("gaussian", sigma=sig), H.gaussian(sig)
    elif d == 2:
        ko, kd = O.Kernel("slp2d", scale=2 * np.pi), H.neg_log_2d()
    else:
        ko, kd = O.Kernel("slp3d", scale=4 * np.pi), H.inv_r_3d()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        arule = H.AdmissibilityRule.weak() if rule == "weak" else H.AdmissibilityRule.strong(eta)
        cfg = H.BuildConfig(rank=rank, leaf_side=leaf, rule=arule, kernel=kd, coeff=H.CoefficientFn.constant(a))
        try:
            if mapped:
                grid = H.MappedGrid(d, n, 0.05)
                pb = O.MappedProblem(d=d, geo=O.MappedGeometry(n, 0.05), rank=rank, leaf_side_max=leaf, kernel=ko,
                                     coeff=O.constant_coeff(a), rule=rule, eta=eta)
            else:
                grid = H.UniformGrid(d, n)
                pb = O.Problem(d=d, n=n, rank=rank, leaf_side_max=leaf, kernel=ko, coeff=O.constant_coeff(a),
                               rule=rule, eta=eta)
            op = H.construct(cfg, grid)
        except ValueError as exc:   # e.g. rank above a box side: the reference raises too
            print(f"case {case}: skipped ({exc})")
            continue
    U = rng.standard_normal((grid.num_points, R))
    F = H.matmat(op, U)
    ref = O.mapped_matvec(pb, U) if mapped else O.matvec(pb, U)
    err = float(np.linalg.norm(F - ref) / np.linalg.norm(ref))
    worst = max(worst, err)
    print(f"case {case}: d={d} n={n} leaf={leaf} p={rank} {rule} eta={eta} {kind} a={a} R={R} "
          f"{'mapped' if mapped else 'uniform'} rel={err:.2e}", flush=True)
print(f"worst {worst:.2e}")
sys.exit(0 if worst <= 1e-12 else 1)
