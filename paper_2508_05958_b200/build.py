"""Build the in-tree C-ABI library ``_htlr_b200.so`` for sm_100a.

    python -m paper_2508_05958_b200.build      (or __graft_entry__.build())

nvcc cross-compiles without a GPU.  The host list builder is compiled with
``-ffp-contract=off`` so the admissibility predicate rounds exactly like the
reference's Python floats (grids.py:153-165).
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "_htlr_b200.so")
BUILD = os.path.join(HERE, "..", "build", "htlr")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SOURCES = ["htlr_build.cu", "htlr_apply.cu", "htlr_gemm.cu", "htlr_mapped.cu", "htlr_regen_sym.cu", "htlr_rows.cu",
              "htlr_quasi.cu", "htlr_lowrank.cu", "htlr_sep.cu", "htlr_band.cu", "htlr_cube.cu", "htlr_tensor.cu", "htlr_interp.cu", "htlr_plan.cu", "htlr_matvec.cu", "htlr_capi.cu"]
CPP_SOURCES = ["htlr_lists.cpp"]


def _run(cmd):
    print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def _stale(out: str, deps) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(p) > t for p in deps)


def build(verbose_ptxas: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    headers.append(os.path.join(HERE, "..", "include", "htlr_b200.h"))
    objs, jobs = [], []
    for src in CPP_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or _stale(o, [s] + headers):
            jobs.append(["g++", "-O2", "-std=c++17", "-fPIC", "-pthread", "-ffp-contract=off", "-c", s, "-o", o])
        objs.append(o)
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or _stale(o, [s] + headers):
            cmd = [NVCC, "-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC,-ffp-contract=off",
                   "-c", s, "-o", o]
            if verbose_ptxas:
                cmd.insert(1, "-Xptxas=-v")
            jobs.append(cmd)
        objs.append(o)
    # independent translation units compile in parallel
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        for fut in [ex.submit(_run, j) for j in jobs]:
            fut.result()
    if force or _stale(OUT, objs):
        _run([NVCC, "-shared", *ARCH, "-o", OUT, *objs, "-lcudart", "-Xcompiler", "-pthread"])
    return OUT


if __name__ == "__main__":
    build(verbose_ptxas="-v" in sys.argv, force="--force" in sys.argv)
