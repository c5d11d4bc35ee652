"""Benchmark rows in the reference's output contract.

    python -m paper_2508_05958_b200.cli bench-uniform --dim 3 --kernel slp3d --n 32 --p 6 --leaf 8 \\
        --adm strong --eta 1 [--format json] [--out FILE]

Same flags, header and exit codes (0 ok, 1 runtime error, 2 usage error) as
``htlr-bench bench-uniform`` (cli.py:47-51, 121-172, 336-410 of the
reference), with the construction and the matvec on the B200: timings are
best-of-3 wall clock around a synchronised device call, the error is the
sampled relative error against 1000 exact rows computed on the device.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import sys
import time

import numpy as np

UNIFORM_HEADER = [
    "id", "variant", "d", "n", "kernel", "adm", "p", "leaf",
    "t_construct", "t_apply", "dense_scalars", "factor_scalars",
    "core_scalars", "total_scalars", "bound", "e_apply_rand", "seed",
]
TIMING_REPEATS = 3


class UsageError(Exception):
    pass


def _best_of(fn, repeats=TIMING_REPEATS):
    import torch
    best, result = float("inf"), None
    for _ in range(repeats):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        result = fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return result, best


def validate_uniform_side(n: int, leaf: int) -> None:
    """The reference's CLI check (cli.py:76-91): n must halve evenly to a leaf
    side of at most `leaf`."""
    side = n
    while side > leaf:
        if side % 2:
            raise UsageError(f"--n {n} cannot be halved evenly down to --leaf {leaf}")
        side //= 2


def cmd_bench_uniform(args) -> list:
    import paper_2508_05958_b200 as H
    validate_uniform_side(args.n, args.leaf)
    kernel = H.by_name(args.kernel, args.dim)
    if args.adm == "weak":
        rule = H.AdmissibilityRule.weak()
    else:
        rule = H.AdmissibilityRule.strong(args.eta if args.eta is not None else float(np.sqrt(args.dim)))
    grid = H.UniformGrid(args.dim, args.n)
    cfg = H.BuildConfig(rank=args.p, leaf_side=args.leaf, rule=rule, kernel=kernel,
                        coeff=H.CoefficientFn.constant(0.0), quadrature=H.QuadratureConfig())
    u = np.random.default_rng((args.seed, 0)).standard_normal(grid.num_points)
    op, t_con = _best_of(lambda: H.construct(cfg, grid))
    import torch
    ud = torch.from_numpy(u).cuda()
    _, t_apply = _best_of(lambda: H.matvec(op, ud))
    exact = H.exact_row_evaluator(kernel, cfg.coeff, grid, cfg.quadrature)
    err = H.estimate_rel_error_random(op, exact, u, sample_size=min(1000, grid.num_points),
                                      seed=(args.seed, 1))
    rep = H.storage_report(op)
    run_id = f"u-d{args.dim}-{args.kernel}-n{args.n}-{args.adm}-p{args.p}-l{args.leaf}-s{args.seed}"
    base = {"id": run_id, "d": args.dim, "n": args.n, "kernel": args.kernel, "adm": args.adm, "p": args.p,
            "leaf": args.leaf, "seed": args.seed}
    rows = [{
        **base, "variant": "htlr-b200", "t_construct": t_con, "t_apply": t_apply,
        "dense_scalars": rep.dense_scalars, "factor_scalars": rep.factor_scalars,
        "core_scalars": rep.core_scalars, "total_scalars": rep.total_scalars,
        "bound": rep.theoretical_bound, "e_apply_rand": err,
    }]
    if args.baseline:
        hop, t_con_h = _best_of(lambda: H.construct_hmatrix(cfg, grid))
        _, t_apply_h = _best_of(lambda: H.hmatrix_matvec(hop, ud))
        err_h = _sampled_error(H, hop, H.hmatrix_matvec, exact, u, (args.seed, 1), grid.num_points)
        rep_h = H.storage_report(hop)
        rows.append({
            **base, "variant": "hmatrix-b200", "t_construct": t_con_h, "t_apply": t_apply_h,
            "dense_scalars": rep_h.dense_scalars, "factor_scalars": rep_h.factor_scalars,
            "core_scalars": rep_h.core_scalars, "total_scalars": rep_h.total_scalars,
            "bound": rep_h.theoretical_bound, "e_apply_rand": err_h,
        })
    return rows


def _sampled_error(H, op, apply_fn, exact, u, seed, n_rows):
    rows = np.random.default_rng(seed).choice(n_rows, size=min(1000, n_rows), replace=False)
    approx = np.asarray(apply_fn(op, u))
    ex = exact(rows, u)
    return float(np.linalg.norm(approx[rows] - ex) / np.linalg.norm(ex))


QUASI_HEADER = [
    "id", "variant", "d", "n_quasi", "rho", "m_side", "kernel", "adm", "p",
    "leaf", "t_construct", "t_apply", "dense_scalars", "factor_scalars",
    "core_scalars", "total_scalars", "bound", "e_apply_rand", "seed",
]


def quasi_test_field(points: np.ndarray) -> np.ndarray:
    """The reference's smooth benchmark field (cli.py:66-73)."""
    x1, x2 = points[:, 0], points[:, 1]
    return 1.0 + 0.5 * np.exp(-((x1 - 0.3) ** 2) - (x2 - 0.6) ** 2) + np.sin(5.0 * x1 * x2)


def cmd_bench_quasi(args) -> list:
    """Triangle-mesh pipeline rows (cli.py:263-316).  e_apply_rand is left NaN:
    the reference computes it with a triangle-average row oracle
    (oracles.py:186-209) that is not part of the B200 path."""
    import paper_2508_05958_b200 as H
    if args.dim != 2:
        raise UsageError("the quasi-uniform pipeline is two-dimensional")
    if args.mesh is not None:
        mesh = H.load_mesh(args.mesh)
    else:
        if args.n is None:
            raise UsageError("bench-quasi needs --n (number of triangles) or --mesh")
        k = int(round(np.sqrt(args.n / 2.0)))
        if 2 * k * k != args.n:
            raise UsageError(f"--n {args.n} is not of the form 2*k^2 for a structured mesh")
        mesh = H.structured_trimesh(k)
    kernel = H.by_name(args.kernel, 2)
    rule = (H.AdmissibilityRule.weak() if args.adm == "weak"
            else H.AdmissibilityRule.strong(args.eta if args.eta is not None else float(np.sqrt(2))))
    cfg = H.BuildConfig(rank=args.p, leaf_side=args.leaf, rule=rule, kernel=kernel,
                        coeff=H.CoefficientFn.constant(0.0), quadrature=H.QuadratureConfig())
    u = quasi_test_field(mesh.centroids)
    rows = []
    for rho in (args.rho or [2.0]):
        pipe, t_con = _best_of(lambda: H.build_pipeline(mesh, cfg, rho))
        out, t_apply = _best_of(lambda: H.apply_pipeline(pipe, u))
        rep = H.storage_report(pipe.op)
        rows.append({
            "id": f"q-{args.kernel}-N{mesh.num_triangles}-rho{rho:g}-{args.adm}-p{args.p}-l{args.leaf}-s{args.seed}",
            "variant": "htlr-quasi-b200", "d": 2, "n_quasi": mesh.num_triangles, "rho": pipe.rho,
            "m_side": pipe.m_side, "kernel": args.kernel, "adm": args.adm, "p": args.p, "leaf": args.leaf,
            "t_construct": t_con, "t_apply": t_apply, "dense_scalars": rep.dense_scalars,
            "factor_scalars": rep.factor_scalars, "core_scalars": rep.core_scalars,
            "total_scalars": rep.total_scalars, "bound": rep.theoretical_bound,
            "e_apply_rand": float("nan"), "seed": args.seed,
        })
    return rows


def _write_rows(rows, header, args) -> None:
    if args.format == "json":
        text = json.dumps(rows, indent=2, default=float) + "\n"
    else:
        buf = io.StringIO()
        w = csv.DictWriter(buf, fieldnames=header)
        w.writeheader()
        for row in rows:
            w.writerow(row)
        text = buf.getvalue()
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="htlr-bench-b200",
                                     description="B200 benchmarks in the htlr-bench row format.")
    sub = parser.add_subparsers(dest="command", required=True)
    pu = sub.add_parser("bench-uniform", help="uniform-grid benchmark")
    pu.add_argument("--dim", type=int, choices=(2, 3), default=2)
    pu.add_argument("--kernel", choices=("gaussian", "slp2d", "slp3d"), default="gaussian")
    pu.add_argument("--seed", type=int, default=0)
    pu.add_argument("--out", default=None)
    pu.add_argument("--format", choices=("csv", "json"), default="csv")
    pu.add_argument("--threads", type=int, default=1)
    pu.add_argument("--n", type=int, required=True)
    pu.add_argument("--p", type=int, default=8)
    pu.add_argument("--leaf", type=int, default=16)
    pu.add_argument("--adm", choices=("weak", "strong"), default="weak")
    pu.add_argument("--eta", type=float, default=None)
    pu.add_argument("--baseline", action="store_true", help="also run the H-matrix baseline")
    pq = sub.add_parser("bench-quasi", help="triangulated-grid pipeline benchmark")
    pq.add_argument("--dim", type=int, choices=(2, 3), default=2)
    pq.add_argument("--kernel", choices=("gaussian", "slp2d", "slp3d"), default="gaussian")
    pq.add_argument("--seed", type=int, default=0)
    pq.add_argument("--out", default=None)
    pq.add_argument("--format", choices=("csv", "json"), default="csv")
    pq.add_argument("--threads", type=int, default=1)
    pq.add_argument("--n", type=int, default=None)
    pq.add_argument("--mesh", default=None)
    pq.add_argument("--rho", type=float, action="append", default=None)
    pq.add_argument("--p", type=int, default=8)
    pq.add_argument("--leaf", type=int, default=16)
    pq.add_argument("--adm", choices=("weak", "strong"), default="weak")
    pq.add_argument("--eta", type=float, default=None)
    return parser


def main(argv=None) -> int:
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
    except SystemExit as exc:
        return int(exc.code) if exc.code is not None else 0
    try:
        if args.kernel == "slp3d" and args.dim != 3:
            raise UsageError("slp3d requires --dim 3")
        if args.kernel == "slp2d" and args.dim != 2:
            raise UsageError("slp2d requires --dim 2")
        if args.command == "bench-uniform":
            _write_rows(cmd_bench_uniform(args), UNIFORM_HEADER, args)
        else:
            _write_rows(cmd_bench_quasi(args), QUASI_HEADER, args)
    except UsageError as exc:
        print(f"usage error: {exc}", file=sys.stderr)
        return 2
    except Exception as exc:   # runtime failure
        print(f"error: {exc}", file=sys.stderr)
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
