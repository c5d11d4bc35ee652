"""The ctypes binding stub of INTEGRATION.md, executed as written (import
paths adapted): a maintainer's `htlr._b200` module must build a plan and
reproduce the package's matvec."""

import os
import re

import numpy as np
import pytest

import paper_2508_05958_b200 as H
from paper_2508_05958_b200 import _lib

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_integration_stub_runs():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    code = re.search(r"```python\n(# pkg/src/htlr/_b200.py.*?)```", text, re.S).group(1)
    code = code.replace("from .grids import IndexBox", "from paper_2508_05958_b200.grids import IndexBox")
    code = code.replace('"/path/to/paper_2508_05958_b200/_htlr_b200.so"', repr(_lib.LIB_PATH))
    ns = {}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    grid = H.UniformGrid(3, 32)
    cfg = H.BuildConfig(rank=6, leaf_side=8, rule=H.AdmissibilityRule.strong(1.0), kernel=H.slp_3d(),
                        coeff=H.CoefficientFn.constant(0.5))
    plan = ns["construct"](cfg, grid)
    u = np.random.default_rng(8).standard_normal(grid.num_points)
    f = ns["matvec"](plan, u)
    ref = H.matvec(H.construct(cfg, grid), u)
    assert np.linalg.norm(f - ref) <= 1e-13 * np.linalg.norm(ref)
    _lib.lib().htlr_plan_destroy(plan)
