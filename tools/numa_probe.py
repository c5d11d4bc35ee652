"""Which host CPUs / NUMA node are local to GPU 0, and does binding the
process there change the pinned H2D / D2H rate? (dev tool)"""
import glob
import os
import time

import pynvml
import torch

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
allowed = sorted(os.sched_getaffinity(0))
print("allowed cpus", allowed)
try:
    words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
    local = [64 * i + b for i, w in enumerate(words) for b in range(64) if (w >> b) & 1]
    print("gpu-local cpus", local[:8], "...", len(local))
except Exception as e:   # noqa: BLE001
    local = []
    print("nvml affinity failed", e)
for nd in sorted(glob.glob("/sys/devices/system/node/node[0-9]*")):
    print(os.path.basename(nd), open(nd + "/cpulist").read().strip())
try:
    print("gpu numa node", open(f"/sys/bus/pci/devices/{pynvml.nvmlDeviceGetPciInfo(h).busId.lower()[4:]}/numa_node").read().strip())
except Exception as e:   # noqa: BLE001
    print("numa_node read failed", e)


def rate(tag):
    x = torch.empty(2 * 1024 * 1024, dtype=torch.float64).pin_memory()
    d = torch.empty_like(x, device="cuda")
    for _ in range(3):
        d.copy_(x, non_blocking=True)
    torch.cuda.synchronize()
    ts = []
    for fn in (lambda: d.copy_(x, non_blocking=True), lambda: x.copy_(d, non_blocking=True)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 20)
    print(tag, "h2d ms %.3f d2h ms %.3f" % tuple(ts), flush=True)


torch.zeros(1, device="cuda")
rate("unbound          ")
cands = [("gpu-local", [c for c in local if c in allowed])]
half = len(allowed) // 2
cands += [("first half", allowed[:half]), ("second half", allowed[half:])]
for name, cpus in cands:
    if not cpus:
        continue
    os.sched_setaffinity(0, cpus)
    time.sleep(0.05)
    rate(f"bound {name:11s}")
os.sched_setaffinity(0, allowed)
