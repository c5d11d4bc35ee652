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

`--impl reference` times the reference's CPU matvec on the host cores (the
reference is pure Python and absent on the GPU box: its leaf loop restated
call for call, oracle/htlr_oracle.py rl_*): the whole loop per step for
configs 1-2, a stratified leaf sample extrapolated to all leaves (stated in
the line) for configs 3-5; rank 0 only, no product code imported.  `--gpus N`
without torchrun starts N ranks itself.
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
NCU_TRAFFIC_FILE = os.path.join(ROOT, "profiles", "traffic_r02.json")


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


# --------------------------------------------------------------------------- workloads

# BASELINE.json configs[0..4] as plain data, shared by both arms so their
# `config` objects are identical.  The reference arm must not import the
# product package (its __init__ loads _htlr_b200.so); tests/test_bench_contract.py
# checks this table against paper_2508_05958_b200/configs.py.
#   name: (d, n, leaf_side_max, rank, (oracle kernel, sigma, scale), a, nrhs, seed, amplitude, description)
TWO_PI, FOUR_PI = 2.0 * 3.141592653589793, 4.0 * 3.141592653589793
WORKLOADS_PLAIN = {
    "cfg1": (2, 64, 8, 8, ("slp2d", None, TWO_PI), 1.0, 1, 0, None,
             "2D n=64 -log|x-y| a=1 leaf 8 eta=1 p=8, 1 matvec"),
    "cfg2": (3, 32, 8, 6, ("slp3d", None, FOUR_PI), 0.0, 1, 1, None,
             "3D n=32 1/|x-y| leaf 8 eta=1 p=6, construct + 10 matvecs"),
    "cfg3": (3, 64, 8, 6, ("slp3d", None, FOUR_PI), 0.0, 16, 2, None,
             "3D n=64 1/|x-y| leaf 8 eta=1 p=6, 16 RHS batched matvec"),
    "cfg4": (3, 128, 8, 8, ("gaussian", 0.1 / 2.0 ** 0.5, 1.0), 0.0, 1, 3, None,
             "3D n=128 exp(-|x-y|^2/0.01) leaf 8 eta=1 p=8, matvec"),
    "cfg5": (3, 96, 8, 6, ("slp3d", None, FOUR_PI), 0.0, 1, 4, 0.05,
             "3D mapped quasi-uniform n=96 (x=t+0.05 sin(2 pi t)/(2 pi)) 1/|x-y| leaf 8 (side 6) "
             "eta=1 p=6, construct + matvec"),
}
L2_NOTE = ("inputs re-read from HBM every step: the GPU arm writes a 512 MiB buffer (> the 126 MB L2) before "
           "every step, outside the timed bracket; the reference arm runs on the host CPU")


def workload_config(name: str) -> dict:
    """The `config` object of both arms' JSON lines (identical by construction)."""
    d, n, _, _, _, _, nrhs, _, _, desc = WORKLOADS_PLAIN[name]
    return {"workload": name, "description": desc, "points": n ** d, "nrhs": nrhs, "l2": L2_NOTE}


def workload_input(name: str):
    """BASELINE.json's seeded input in the reference's F-order linearisation
    (same recipe as paper_2508_05958_b200/configs.py Workload.input)."""
    import numpy as np
    d, n, _, _, _, _, nrhs, seed, _, _ = WORKLOADS_PLAIN[name]
    rng = np.random.default_rng(seed)
    return rng.standard_normal((n ** d, nrhs)) if nrhs > 1 else rng.uniform(-1, 1, n ** d)


# --------------------------------------------------------------------------- CPU path (reference algorithm)


def oracle_problem(name):
    from oracle import htlr_oracle as O
    d, n, leaf, rank, (kind, sigma, scale), a, _, _, amp, _ = WORKLOADS_PLAIN[name]
    kern = O.Kernel(kind, sigma=sigma, scale=scale) if sigma is not None else O.Kernel(kind, scale=scale)
    if amp is not None:
        return O.MappedProblem(d=d, geo=O.MappedGeometry(n, amp), rank=rank, leaf_side_max=leaf, kernel=kern,
                               coeff=O.constant_coeff(a))
    return O.Problem(d=d, n=n, rank=rank, leaf_side_max=leaf, kernel=kern, coeff=O.constant_coeff(a))


FULL_REFERENCE = ("cfg1", "cfg2")   # the whole leaf loop per step; larger configs: stratified samples
SAMPLES_FILE = os.path.join(ROOT, "tests", "golden", "bench_samples.npz")


class ReferenceLoop:
    """The reference's matvec (operators.py:138-156 with blocks.py:230-259,
    restated call for call in oracle/htlr_oracle.py `rl_*`) on the host CPU.

    Configs 1-2: one step is the whole DFS leaf loop over every leaf (payloads
    built beforehand, untimed, one block object per distinct (kind, level,
    offset): equal values).  Configs 3-5 (0.17-2.7 M leaves, 0.1-5 TB of
    payloads): one step applies a stratified sample -- the leaves of
    tests/golden/bench_samples.npz, 32 per (level, kind) stratum -- and the full
    matvec time is extrapolated as sum over strata of count / sampled x the
    stratum's measured time, x the RHS count."""

    def __init__(self, name: str):
        import numpy as np
        from oracle import htlr_oracle as O
        self.O, self.name = O, name
        self.pb = oracle_problem(name)
        d, n, leaf, rank = WORKLOADS_PLAIN[name][:4]
        self.d, self.n, self.nrhs = d, n, WORKLOADS_PLAIN[name][6]
        self.full = name in FULL_REFERENCE
        mapped = isinstance(self.pb, O.MappedProblem)
        if self.full:
            self.leaves = O.block_leaves(n, d, leaf)
            self.payloads = O.shared_payloads(self.pb, self.leaves)
            self.strata = None
        else:
            smp = np.load(SAMPLES_FILE)
            counts, rows = smp[f"{name}_counts"], smp[f"{name}_rows"]
            self.counts = {(int(l), int(k)): int(c) for l, k, c in counts}
            self.leaves, self.payloads, self.strata = [], [], []
            diag = None if mapped else self.pb.diag()
            cache = {}
            for r in rows:
                lf = O.Leaf(int(r[0]), int(r[1]), int(r[2]),
                            tuple((int(r[3 + 2 * a]), int(r[4 + 2 * a])) for a in range(d)),
                            tuple((int(r[3 + 2 * d + 2 * a]), int(r[4 + 2 * d + 2 * a])) for a in range(d)))
                if mapped:
                    pl = (O.mapped_tucker_block(self.pb.kernel, self.pb.geo, lf.tau, lf.sigma, self.pb.rank)
                          if lf.kind == O.ADM else
                          O.mapped_dense_block(self.pb.kernel, self.pb.coeff, self.pb.geo, lf.tau, lf.sigma))
                else:
                    key = O.leaf_key(lf)
                    if key not in cache:
                        cache[key] = O.build_payload(self.pb, lf, diag)
                    pl = cache[key]
                self.leaves.append(lf)
                self.payloads.append(pl)
                self.strata.append((lf.level, lf.kind))
        u = workload_input(name)
        self.u = u.reshape(n ** d, -1)[:, 0].reshape((n,) * d, order="F")
        self.f = np.zeros((n,) * d)

    @property
    def sample(self) -> str:
        if self.full:
            return (f"the whole reference leaf loop (operators.py:146-155, {len(self.leaves)} leaves, "
                    f"rl_* restatement in oracle/htlr_oracle.py) per step")
        return (f"{len(self.leaves)} leaves per step ({len(self.leaves) // max(1, len(self.counts))} per (level, kind) "
                f"stratum, tests/golden/bench_samples.npz) through the reference leaf loop (rl_* restatement), "
                f"extrapolated to all {sum(self.counts.values())} leaves x {self.nrhs} RHS")

    def step(self):
        """One step; returns (elapsed seconds, seconds of one full matvec of
        all RHS: measured for the full loop, else extrapolated)."""
        O = self.O
        t_start = time.perf_counter()
        if self.full:
            self.f[...] = 0.0
            for lf, pl in zip(self.leaves, self.payloads):
                O.rl_leaf(self.u, self.f, lf, pl)
            el = time.perf_counter() - t_start
            return el, el * self.nrhs
        per = {}
        for lf, pl, key in zip(self.leaves, self.payloads, self.strata):
            t0 = time.perf_counter()
            O.rl_leaf(self.u, self.f, lf, pl)
            s, c = per.get(key, (0.0, 0))
            per[key] = (s + time.perf_counter() - t0, c + 1)
        el = time.perf_counter() - t_start
        est = sum(self.counts[k] * s / c for k, (s, c) in per.items()) * self.nrhs
        return el, est


def host_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"]
        return max(n) if n else 1
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(name: str, budget_s: float) -> dict:
    """The reference arm's loop, bounded to about `budget_s` seconds."""
    loop = ReferenceLoop(name)
    t_start = time.perf_counter()
    ests = []
    while time.perf_counter() - t_start < budget_s or not ests:
        ests.append(loop.step()[1])
    est = statistics.median(ests)
    npts = loop.n ** loop.d * loop.nrhs
    return {"value": npts / est, "unit": "points/s", "cores": host_threads(), "kind": "port",
            "sample": f"{loop.sample}; {len(ests)} steps in {time.perf_counter() - t_start:.1f} s; "
                      f"full matvec {est:.3f} s"}


def run_reference(args):
    """`--impl reference`: the reference's CPU matvec (oracle port; the
    reference is pure Python, not installable on the GPU box), rank 0 only,
    with the BLAS threads of every host core, on the B200 arm's config."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    loop = ReferenceLoop(args.workload)
    for _ in range(args.warmup):
        loop.step()
    els, ests = [], []
    for _ in range(args.steps):
        el, est = loop.step()
        els.append(el)
        ests.append(est)
    ms_per_step = statistics.mean(els) * 1e3
    est = statistics.mean(ests)
    npts = loop.n ** loop.d * loop.nrhs
    value = npts / est
    line = {
        "metric": "HTLR matvec points/s", "value": value, "unit": "points/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE.json seeds)",
        "config": workload_config(args.workload),
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": host_threads(), "kind": "port",
                         "sample": loop.sample},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not loop.full:
        line["extrapolated"] = {"ms_per_step_is": "the measured time of the sampled leaves",
                                "full_matvec_s_est": est, "sampled_leaves": len(loop.leaves),
                                "leaves": sum(loop.counts.values())}
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
    "band_z": "band_line_kernel (z sweep of a banded pass -- near + admissible blocks as C10^3 - C4^3 - C5^3 + "
              "C2^3 (+ E5^3 - E2^3 at the leaf level) line sweeps: reads the sources, writes the terms' z-swept "
              "lines; fp64 DMMA, bound by its stores)",
    "band_yx": "band_plane_kernel (fused y and x sweeps of a banded pass, one z-point plane per CTA, accumulator "
               "in tensor memory; fp64 DMMA)",
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
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} (launch N ranks with torchrun, or "
                         f"run without WORLD_SIZE and bench.py starts them)")
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

    u_host = workload_input(args.workload)
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
    rank_ms = [total_ms / args.steps]
    if dist is not None:
        t = torch.zeros(world, dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
        t[rank] = total_ms
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        rank_ms = [float(v) / args.steps for v in t.tolist()]
        total_ms = max(float(v) for v in t.tolist())
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
    # the other kernels that take a tenth of the step or more, each with its own roofline
    also = []
    for k, ent in sorted(phases.items(), key=lambda kv: -kv[1]["ms"]):
        if k == dom_key or ent["ms"] < 0.1 * sum(prof_step_ms):
            continue
        r2 = phase_roofline(k, ent["flops"] / ent["launches"], ent["bytes"] / ent["launches"],
                            ent["ms"] / ent["launches"])
        r2.pop("peak_source", None)
        r2["avg_launch_ms"] = ent["ms"] / ent["launches"]
        also.append(r2)
    roofline.update({
        "also": also,
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
    xbytes = 0
    if world > 1:
        xbytes = sum(b.numel() * 8 for b in op.exchange_buffers(R)) * (world - 1) // world
    line = {
        "metric": "HTLR matvec points/s", "value": value, "unit": "points/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE.json seeds)",
        "config": workload_config(args.workload),
        "plan": {"formulation": base_op.formulation(), "leaf_pass": base_op.leaf_pass(),
                 "formulation_note": FORMULATION_NOTES.get(base_op.formulation(), ""),
                 "construct_s": construct_s, "parallelism": f"target subtrees x{world}" if world > 1 else "1 GPU",
                 "operator_tables_GB": rep.device_scalars * 8 / 1e9,
                 "reference_storage_GB": rep.total_scalars * 8 / 1e9,
                 "rank_ms_per_step": rank_ms, "exchange_bytes_per_rank_per_step": xbytes},
        "roofline": roofline,
        "whole_step": whole,
        "construction": {"seconds": construct_s, "points_per_s": grid.num_points / construct_s,
                         "includes": "host list build + device sampling, QR and tiling (first construct "
                                     "of the process)"},
        "phases_ms_per_step": {k: v["ms"] / args.steps for k, v in sorted(phases.items())},
        "phases_note": "per-kernel times of a profiled pass: the same kernels with their launches serialised on one "
                       "stream; the timed step replays a graph with the level passes on side streams and, for "
                       "unsharded banded plans, the downward pass beside the leaf y-x sweep (both add into a zeroed f "
                       "with fp64 REDs; HTLR_FDIRECT=0 stores Y and runs the downward pass after it)",
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "points/s", "h2d_bytes_per_step": io_bytes,
                "d2h_bytes_per_step": io_bytes, "ms_per_step": e2e_total / args.steps,
                "ms_min": min(e2e_ms), "ms_median": sorted(e2e_ms)[len(e2e_ms) // 2], "ms_max": max(e2e_ms)},
        "clocks": clk,
        "gpu_launches": launches_per_step * args.steps,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def self_launch(args) -> int:
    """`--gpus N` without a torchrun environment: start N ranks of this
    script (torch.distributed.run, one process per GPU, 127.0.0.1)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd, env=env).returncode


def main():
    args = parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
