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


def test_reference_arm_loads_no_product_code():
    """The reference arm must time the reference algorithm only: run it and
    check that neither the product package nor its .so was imported."""
    code = ("import sys, runpy; sys.argv = ['bench.py', '--impl', 'reference', '--workload', 'cfg1', '--steps', '1',"
            " '--warmup', '0']\n"
            "try:\n    runpy.run_path('bench.py', run_name='__main__')\nexcept SystemExit:\n    pass\n"
            "bad = [m for m in sys.modules if m.startswith('paper_2508_05958_b200')]\n"
            "maps = open('/proc/self/maps').read()\n"
            "print('BAD', bad, '_htlr_b200' in maps)\n")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600,
                         check=True)
    assert "BAD [] False" in out.stdout, out.stdout[-2000:]


def test_workload_table_matches_package_configs():
    """bench.py's plain workload table (both arms' `config`) is the product's
    configs.py: same sizes, RHS counts, descriptions and seeded inputs."""
    import numpy as np
    sys.path.insert(0, ROOT)
    import bench
    from paper_2508_05958_b200.configs import WORKLOADS
    for name, w in WORKLOADS.items():
        d, n, leaf, rank, _, a, nrhs, _, amp, desc = bench.WORKLOADS_PLAIN[name]
        assert (d, n, leaf, rank, a, nrhs, desc) == (w.d, w.n, w.leaf, w.rank, w.a, w.nrhs, w.description)
        assert (amp if amp is not None else -1.0) == w.amplitude
        cfg = bench.workload_config(name)
        assert cfg["points"] == w.grid.num_points and cfg["nrhs"] == w.nrhs
        if name in ("cfg1", "cfg2"):
            assert np.array_equal(bench.workload_input(name), w.input())


def test_reference_loop_matches_golden_cfg1():
    """The timed reference loop (rl_* restatement, shared payloads) computes
    the reference's cfg1 matvec (fixture from the reference itself)."""
    import numpy as np
    sys.path.insert(0, ROOT)
    import bench
    loop = bench.ReferenceLoop("cfg1")
    loop.step()
    ref = np.load(os.path.join(ROOT, "tests", "golden", "cfg1_matvec.npz"))
    f = loop.f.ravel(order="F")
    assert np.linalg.norm(f - ref["f"]) / np.linalg.norm(ref["f"]) < 1e-12
