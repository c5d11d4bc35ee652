"""bench.py's JSON contract on CPU: the reference arm (the oracle port of the
reference's matvec loop, timed on the host) prints one line with the keys the
driver reads, and the roofline helper picks the binding resource."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "cfg1", "--steps", "1",
                          "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=600, check=True)
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference"
    assert line["config"]["workload"] == "cfg1"
    assert line["steps"] == 1 and line["warmup"] == 3
    assert line["value"] > 0 and line["higher_is_better"] is True
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert line["e2e"]["value"] == line["value"] and line["e2e"]["h2d_bytes_per_step"] == 0


def test_phase_roofline_picks_binding_resource():
    sys.path.insert(0, ROOT)
    import bench
    # GEMM phase, compute-bound: 1e12 flop, 1e9 bytes in 30 ms
    r = bench.phase_roofline("gemm_leaf_L4", 1e12, 1e9, 30.0)
    assert r["bound"] == "tensor" and r["unit"] == "TFLOP/s"
    assert abs(r["achieved"] - 1e12 / 0.030 / 1e12) < 1e-9 and 0 < r["frac"] < 1
    # same phase, memory-bound: few flops, many bytes
    r = bench.phase_roofline("gemm_leaf_L2", 1e6, 3e8, 0.1)
    assert r["bound"] == "hbm" and r["unit"] == "GB/s"
    # regeneration runs on the fp64 CUDA cores
    r = bench.phase_roofline("regen_level_L4", 5e11, 1e6, 30.0)
    assert r["bound"] == "fp64_core" and r["peak"] < bench.fp64_peak()
