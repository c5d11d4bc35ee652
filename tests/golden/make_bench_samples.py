"""Stratified leaf samples for the reference arm of bench.py (configs 3-5).

    python tests/golden/make_bench_samples.py

The reference arm times the reference's leaf loop (operators.py:146-155,
restated in oracle/htlr_oracle.py `rl_*`) on the GPU box's host cores.
Configs 3-5 have 0.17-2.5 M leaves and 0.13-5.3 TB of payloads, so one step
applies a bounded sample: PER_STRATUM leaves of every (level, kind) stratum
of the DFS leaf list, drawn with a fixed seed.  The full DFS walk of the
larger trees takes minutes in Python, so the strata counts and the sampled
rows are computed once here, with the oracle's list builder (bit-exact with
the reference's, tests/test_oracle_golden.py), and committed as
bench_samples.npz.  Row format: oracle.leaves_to_array.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import htlr_oracle as O  # noqa: E402

PER_STRATUM = 32
# (d, n, leaf_side_max, amplitude or None)
TREES = {"cfg3": (3, 64, 8, None), "cfg4": (3, 128, 8, None), "cfg5": (3, 96, 8, 0.05)}


def main(names):
    out = {}
    path = os.path.join(HERE, "bench_samples.npz")
    if os.path.exists(path):
        out.update(dict(np.load(path)))
    for name in names:
        d, n, leaf, amp = TREES[name]
        if amp is None:
            leaves = O.block_leaves(n, d, leaf)
        else:
            leaves = O.mapped_block_leaves(O.MappedGeometry(n, amp), d, leaf)
        arr = O.leaves_to_array(leaves, d)
        rng = np.random.default_rng(2508)
        counts, rows = [], []
        for lvl in np.unique(arr[:, 2]):
            for kind in (O.ADM, O.NEAR):
                sel = np.nonzero((arr[:, 2] == lvl) & (arr[:, 1] == kind))[0]
                if len(sel) == 0:
                    continue
                counts.append((int(lvl), kind, len(sel)))
                pick = np.sort(rng.choice(sel, size=min(PER_STRATUM, len(sel)), replace=False))
                rows.append(arr[pick])
        out[f"{name}_counts"] = np.asarray(counts, dtype=np.int64)
        out[f"{name}_rows"] = np.concatenate(rows)
        print(name, len(leaves), "leaves;", out[f"{name}_counts"].tolist(), flush=True)
    np.savez_compressed(path, **out)


if __name__ == "__main__":
    main(sys.argv[1:] or list(TREES))
