#!/usr/bin/env python
"""HTLR matvec throughput on B200 -- BASELINE.json metric
"HTLR matvec points/s at 1/2/4/8 B200; % of HBM/fp64 roofline".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg4] [--impl b200|reference]

One step = one matvec of the workload (BASELINE config 4 by default: 3-D
n=128 Gaussian, p=8, leaf 8, eta=1; N = 2,097,152 points) over synthetic
input resident in HBM.  Timing: W untimed warm-up steps, then exactly K steps
bracketed by barrier + synchronize; each step is timed with CUDA events on
the launching stream; L2 is flushed (512 MiB write) before every step,
outside the event bracket.  `value` = points x RHS / time, max over ranks.
Multi-GPU (torchrun) shards target boxes by cluster subtrees (strong
scaling); `e2e` repeats the step through the public API from
pinned host memory with the result copied back.

`--impl reference` times the reference algorithm's CPU path (the oracle
port, oracle/htlr_oracle.py -- /root/reference does not exist on the GPU
box) on a bounded sample of leaf blocks per (level, kind), extrapolated to
the full leaf counts; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

FP64_PEAK_FILE = os.path.join(ROOT, "profiles", "fp64_peak_r01.jsonl")
NCU_TRAFFIC_FILE = os.path.join(ROOT, "profiles", "traffic_r01.json")


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="cfg4", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=20.0,
                    help="budget of the cpu_baseline sample (rank 0, N=1)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


# --------------------------------------------------------------------------- clocks


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms while running."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.lines = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, flag in zip(names, parts[5:9]):
                if flag.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------- CPU path


def oracle_problem(name):
    from oracle import htlr_oracle as O
    import math
    from paper_2508_05958_b200.configs import WORKLOADS
    w = WORKLOADS[name]
    kern = {
        "cfg1": O.Kernel("slp2d", scale=2 * math.pi),
        "cfg2": O.Kernel("slp3d", scale=4 * math.pi),
        "cfg3": O.Kernel("slp3d", scale=4 * math.pi),
        "cfg4": O.Kernel("gaussian", sigma=0.1 / math.sqrt(2.0)),
        "cfg5": O.Kernel("slp3d", scale=4 * math.pi),
    }[name]
    if w.amplitude >= 0:
        return w, O.MappedProblem(d=w.d, geo=O.MappedGeometry(w.n, w.amplitude), rank=w.rank,
                                  leaf_side_max=w.leaf, kernel=kern, coeff=O.constant_coeff(w.a))
    return w, O.Problem(d=w.d, n=w.n, rank=w.rank, leaf_side_max=w.leaf, kernel=kern,
                        coeff=O.constant_coeff(w.a))


def leaf_groups(name):
    """Leaf rows grouped by (level, kind), from the (bit-exact) host list
    builder -- used only to choose and count the sampled blocks."""
    import numpy as np
    import paper_2508_05958_b200 as H
    from paper_2508_05958_b200.configs import WORKLOADS
    w = WORKLOADS[name]
    grid = w.grid
    bt = H.build_block_cluster_tree(H.build_cluster_tree(grid, w.leaf), H.AdmissibilityRule.strong(1.0))
    arr = bt.leaf_array
    groups = {}
    for lvl in np.unique(arr[:, 2]):
        for kind in (0, 1):
            rows = arr[(arr[:, 2] == lvl) & (arr[:, 1] == kind)]
            if len(rows):
                groups[(int(lvl), kind)] = rows
    return groups


class CpuSample:
    """Reference matvec inner loop (operators.py:146-155) on a bounded sample
    of leaves per (level, kind), payloads built beforehand (untimed)."""

    def __init__(self, name: str, per_group: int, seed: int = 0):
        import numpy as np
        from oracle import htlr_oracle as O
        self.O = O
        self.w, self.pb = oracle_problem(name)
        groups = leaf_groups(name)
        rng = np.random.default_rng(seed)
        d = self.w.d
        mapped = isinstance(self.pb, O.MappedProblem)
        diag = None if mapped else self.pb.diag()
        self.items = []      # (group, leaf, payload)
        self.counts = {}
        for key, rows in groups.items():
            self.counts[key] = len(rows)
            pick = rng.choice(len(rows), size=min(per_group, len(rows)), replace=False)
            for i in pick:
                r = rows[i]
                lf = O.Leaf(int(r[0]), int(r[1]), int(r[2]),
                            tuple((int(r[3 + 2 * a]), int(r[4 + 2 * a])) for a in range(d)),
                            tuple((int(r[3 + 2 * d + 2 * a]), int(r[4 + 2 * d + 2 * a])) for a in range(d)))
                if mapped:
                    pl = (O.mapped_tucker_block(self.pb.kernel, self.pb.geo, lf.tau, lf.sigma, self.pb.rank)
                          if lf.kind == O.ADM else
                          O.mapped_dense_block(self.pb.kernel, self.pb.coeff, self.pb.geo, lf.tau, lf.sigma))
                else:
                    pl = O.build_payload(self.pb, lf, diag)
                self.items.append((key, lf, pl))
        u = self.w.input()
        self.R = 1 if u.ndim == 1 else u.shape[1]
        shape = (self.w.n,) * d
        self.u = u.reshape(self.w.grid.num_points, -1)[:, 0].reshape(shape, order="F")
        self.f = np.zeros(shape)

    def step(self):
        """Apply every sampled block once; returns (estimated full matvec
        seconds for all R right-hand sides, sampled seconds)."""
        O = self.O
        per = {}
        t_all = 0.0
        for key, lf, pl in self.items:
            t0 = time.perf_counter()
            seg = self.u[O._slices(lf.sigma)].ravel(order="F")
            out = O.apply_payload(pl, seg)
            self.f[O._slices(lf.tau)] += out.reshape([hi - lo for lo, hi in lf.tau], order="F")
            dt = time.perf_counter() - t0
            t_all += dt
            s, c = per.get(key, (0.0, 0))
            per[key] = (s + dt, c + 1)
        est = sum(self.counts[k] * s / c for k, (s, c) in per.items()) * self.R
        return est, t_all


def blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"]
        return max(n) if n else 1
    except Exception:
        return 1


def cpu_baseline(name: str, budget_s: float) -> dict:
    per_group = 12
    smp = CpuSample(name, per_group)
    t_start = time.perf_counter()
    ests = []
    while time.perf_counter() - t_start < budget_s or not ests:
        est, _ = smp.step()
        ests.append(est)
    est = statistics.median(ests)
    npts = smp.w.grid.num_points * smp.R
    return {"value": npts / est, "unit": "points/s", "cores": blas_threads(), "kind": "port",
            "sample": (f"oracle port of the reference matvec loop (operators.py:146-155) on {len(smp.items)} "
                       f"leaves ({per_group} per (level, kind)), {len(ests)} passes, extrapolated to the full "
                       f"{sum(smp.counts.values())} leaves; est. full matvec {est:.2f} s")}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_2508_05958_b200.configs import WORKLOADS
    w = WORKLOADS[args.workload]
    smp = CpuSample(args.workload, per_group=8)
    for _ in range(args.warmup):
        smp.step()
    ests = []
    for _ in range(args.steps):
        est, _ = smp.step()
        ests.append(est)
    est = statistics.mean(ests)
    npts = w.grid.num_points * w.nrhs
    value = npts / est
    line = {
        "metric": "HTLR matvec points/s", "value": value, "unit": "points/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": est * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE.json seeds)",
        "config": {"workload": args.workload, "description": w.description, "points": w.grid.num_points,
                   "nrhs": w.nrhs},
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": blas_threads(), "kind": "port",
                         "sample": (f"oracle port (oracle/htlr_oracle.py) of the reference matvec loop on "
                                    f"{len(smp.items)} sampled leaves per step, extrapolated to "
                                    f"{sum(smp.counts.values())} leaves")},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- B200 path


def fp64_peak() -> float:
    best = None
    try:
        with open(FP64_PEAK_FILE) as fh:
            for ln in fh:
                rec = json.loads(ln)
                if rec.get("probe") == "dmma_m16n8k8_sustained":
                    best = float(rec["tflops"])
    except OSError:
        pass
    return best or 37.0


def fp64_dfma_peak() -> float:
    try:
        with open(FP64_PEAK_FILE) as fh:
            for ln in fh:
                rec = json.loads(ln)
                if rec.get("probe") == "dfma":
                    return float(rec["tflops"])
    except OSError:
        pass
    return 34.0


def hbm_peak_gbs():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)"
    except (OSError, ValueError, KeyError):
        return 7700.0, "B200_PROFILING.md fallback"


PHASE_KERNELS = {
    "gemm_leaf": "gemm_persistent_kernel / gemm_thin_kernel (near + leaf-level cores, fp64 DMMA)",
    "gemm_level": "gemm_persistent_kernel / gemm_thin_kernel (coupling cores, fp64 DMMA)",
    "regen_level": "regen_sym_kernel (cores regenerated + contracted, fp64 CUDA cores)",
    "regen_near": "regen_sym_kernel (near blocks regenerated, fp64 CUDA cores)",
    "sep_level": "sep_block_kernel (separable coupling cores: per-axis mode products, fp64 DMMA)",
    "sep_leaf": "sep_block_kernel (separable near + leaf-level cores: per-axis mode products, fp64 DMMA)",
    "upward": "upward_kernel", "downward": "downward_kernel", "permute": "permute_in_kernel",
}
# separable plans whose passes run as banded line sweeps (op.leaf_pass() == "banded")
BANDED_KERNELS = {
    "sep_leaf": "sep_band_kernel<z> + sep_band_xy_kernel (banded leaf pass: near + leaf-level cores as "
                "C10^3 - C4^3 - C5^3 + C2^3 + E5^3 - E2^3 line sweeps, fp64 DMMA)",
    "sep_level": "sep_band_kernel<z> + sep_band_xy_kernel (banded coupling pass, fp64 DMMA)",
}


FORMULATION_NOTES = {
    "separable": "tensor-product kernel (Gaussian): every reference block (Tucker core with its factors, or "
                 "near block) is exactly a Kronecker product of three 8x8 per-axis factors and is applied as mode "
                 "products -- the same operator as the reference's dense cores (1.5e-15 apart); "
                 "HTLR_SEPARABLE=0 runs the dense-core GEMM path instead",
    "dense": "deduplicated dense cores per (level, offset) and near blocks per offset, gathered fp64 "
             "tensor-core GEMMs",
    "regenerated": "mapped grid: cores and near blocks regenerated from the kernel inside the contraction",
}


def phase_roofline(key: str, flops: float, nbytes: float, ms: float) -> dict:
    """Roofline of one phase's launch: the binding resource is the larger of
    the compute time at the fp64 peak of the pipe the kernel runs on (DMMA
    tensor pipe for the GEMMs, DFMA for the regeneration kernels) and the
    algorithmic bytes at the measured HBM copy bandwidth."""
    phase = key.rsplit("_L", 1)[0]
    core = phase.startswith("regen")
    tf = fp64_dfma_peak() if core else fp64_peak()
    bw, bw_src = hbm_peak_gbs()
    t_flop = flops / (tf * 1e12)
    t_mem = nbytes / (bw * 1e9)
    if t_mem > t_flop:
        ach = nbytes / (ms / 1e3) / 1e9
        return {"bound": "hbm", "achieved": ach, "peak": bw, "unit": "GB/s", "frac": ach / bw,
                "kernel": f"{PHASE_KERNELS.get(phase, phase)} [{key}]", "peak_source": bw_src}
    ach = flops / (ms / 1e3) / 1e12
    src = ("fp64 DFMA, own microbenchmark (profiles/fp64_peak_r01.jsonl)" if core else
           "fp64 DMMA m16n8k8 sustained, own microbenchmark (profiles/fp64_peak_r01.jsonl)")
    return {"bound": "fp64_core" if core else "tensor", "achieved": ach, "peak": tf, "unit": "TFLOP/s",
            "frac": ach / tf, "kernel": f"{PHASE_KERNELS.get(phase, phase)} [{key}]",
            "peak_source": src + "; MEASURED_PEAKS.json has no fp64 entry"}


def ncu_traffic(workload: str):
    try:
        with open(NCU_TRAFFIC_FILE) as fh:
            return json.load(fh).get(workload)
    except (OSError, ValueError):
        return None


def run_b200(args):
    import numpy as np
    import torch
    import paper_2508_05958_b200 as H
    from paper_2508_05958_b200.configs import WORKLOADS

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # HTLR_DIST_BACKEND=gloo: a harness check of the multi-rank flow on fewer
    # GPUs than ranks (exchange staged through host memory; not a measurement)
    backend = os.environ.get("HTLR_DIST_BACKEND", "nccl")
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if backend != "nccl":
        local %= max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    w = WORKLOADS[args.workload]
    grid = w.grid

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if world > 1:
        from paper_2508_05958_b200.multi import ShardedOperator
        op = ShardedOperator(w.build_config(), grid, rank=rank, world=world, device=local)
    else:
        op = H.construct(w.build_config(), grid, device=local)
    torch.cuda.synchronize()
    construct_s = time.perf_counter() - t0

    u_host = w.input()
    R = 1 if u_host.ndim == 1 else u_host.shape[1]
    ud = torch.from_numpy(np.ascontiguousarray(u_host)).cuda()
    if world > 1:
        apply = op.matmat
    else:
        apply = (lambda x: H.matmat(op, x)) if R > 1 else (lambda x: H.matvec(op, x))
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")   # 512 MiB > L2

    for _ in range(args.warmup):
        apply(ud)
    torch.cuda.synchronize()
    base_op = op.local if world > 1 else op
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms = []
    for _ in range(args.steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        apply(ud)
        e1.record()
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    clk = clocks.stop()
    launches_per_step = base_op.last_launch_count()   # of the timed (unprofiled) matvec
    # per-kernel device times: the same K steps again with every launch
    # bracketed by CUDA events on its stream (kept out of the timed pass so
    # the event nodes do not inflate the small configs' step time)
    base_op.profile(True)
    apply(ud)
    torch.cuda.synchronize()
    prof = []
    prof_step_ms = []
    for _ in range(args.steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        apply(ud)
        e1.record()
        e1.synchronize()
        prof_step_ms.append(e0.elapsed_time(e1))
        prof.append(base_op.profile_read())
    base_op.profile(False)
    total_ms = sum(step_ms)
    if dist is not None:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    npts = grid.num_points * R
    value = npts / (ms_per_step / 1e3)

    # per-phase device time over the timed steps, dominant kernel roofline
    phases = {}
    for rec in prof:
        for r in rec:
            key = f"{r['phase']}_L{r['level']}"
            ent = phases.setdefault(key, {"ms": 0.0, "flops": 0.0, "bytes": 0.0, "launches": 0})
            ent["ms"] += r["ms"]
            ent["flops"] += r["flops"]
            ent["bytes"] += r["bytes"]
            ent["launches"] += 1
    dom_key = max(phases, key=lambda k: phases[k]["ms"])
    dom = phases[dom_key]
    avg_ms = dom["ms"] / dom["launches"]
    flops_per_launch = dom["flops"] / dom["launches"]
    bytes_per_launch = dom["bytes"] / dom["launches"]
    peak = fp64_peak()
    if base_op.formulation() == "separable" and base_op.leaf_pass() == "banded":
        PHASE_KERNELS.update(BANDED_KERNELS)
    roofline = phase_roofline(dom_key, flops_per_launch, bytes_per_launch, avg_ms)
    roofline.update({
        "traffic": ncu_traffic(args.workload), "algorithmic_flops_per_launch": flops_per_launch,
        "algorithmic_bytes_per_launch": bytes_per_launch, "avg_launch_ms": avg_ms,
        "share_of_step": dom["ms"] / sum(prof_step_ms),
        "measured": "CUDA events around every launch, on the launching stream, over K profiled steps "
                    "run right after the K timed steps"})
    total_flops = sum(p["flops"] for p in phases.values()) / args.steps
    whole = {"flops_per_step": total_flops, "tflops": total_flops / (ms_per_step / 1e3) / 1e12,
             "frac_of_fp64_peak": total_flops / (ms_per_step / 1e3) / 1e12 / peak}

    # e2e through the public API from pinned host memory
    u_pin = torch.from_numpy(np.ascontiguousarray(u_host)).pin_memory()
    f_pin = torch.empty(u_pin.shape, dtype=torch.float64).pin_memory()
    if world > 1:
        e2e_apply = apply
    else:
        e2e_apply = (lambda x: H.matmat(op, x, out=f_pin)) if R > 1 else (lambda x: H.matvec(op, x, out=f_pin))
    for _ in range(max(3, args.warmup)):
        e2e_apply(u_pin)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    e2e_ms = []
    for _ in range(args.steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        res = e2e_apply(u_pin)
        e1.record()
        e1.synchronize()
        assert not res.is_cuda
        e2e_ms.append(e0.elapsed_time(e1))
    e2e_total = sum(e2e_ms)
    if dist is not None:
        t = torch.tensor([e2e_total], dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_total = float(t.item())
    e2e_value = npts / (e2e_total / args.steps / 1e3)
    io_bytes = grid.num_points * R * 8

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.workload, args.cpu_seconds)

    rep = H.storage_report(base_op)
    line = {
        "metric": "HTLR matvec points/s", "value": value, "unit": "points/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE.json seeds)",
        "config": {"workload": args.workload, "description": w.description, "points": grid.num_points,
                   "nrhs": R, "l2": "flushed (512 MiB write) before every step, outside the timed bracket; "
                                   f"operator tables {rep.device_scalars * 8 / 1e9:.2f} GB "
                                   f"({'>' if rep.device_scalars * 8 > 126e6 else '<'} the 126 MB L2)",
                   "formulation": base_op.formulation(), "leaf_pass": base_op.leaf_pass(),
                   "formulation_note": FORMULATION_NOTES.get(base_op.formulation(), ""),
                   "construct_s": construct_s, "parallelism": f"target subtrees x{world}" if world > 1 else "1 GPU",
                   "reference_storage_GB": rep.total_scalars * 8 / 1e9,
                   "device_storage_GB": rep.device_scalars * 8 / 1e9},
        "roofline": roofline,
        "whole_step": whole,
        "construction": {"seconds": construct_s, "points_per_s": grid.num_points / construct_s,
                         "includes": "host list build + device sampling, QR and tiling (first construct "
                                     "of the process)"},
        "phases_ms_per_step": {k: v["ms"] / args.steps for k, v in sorted(phases.items())},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "points/s", "h2d_bytes_per_step": io_bytes,
                "d2h_bytes_per_step": io_bytes, "ms_per_step": e2e_total / args.steps},
        "clocks": clk,
        "gpu_launches": launches_per_step * args.steps,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
