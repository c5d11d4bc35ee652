"""Fixtures that pin BASELINE config 5 (mapped quasi-uniform grid) at its own
size, from the oracle's mapped restatement (the reference has no mapped grid;
the restatement is self-checked in tests/test_mapped_cpu.py and reproduces
the reference's uniform fixtures at amplitude 0).

    python tests/golden/make_mapped_fixtures.py

mapped.npz:
  cfg5_sha / cfg5_hist / cfg5_spotidx / cfg5_spot: the n = 96 (leaf_side 8 ->
      side-6 leaves) DFS leaf list of oracle.mapped_block_leaves (sha256 of the
      int32 leaf array, per-(level, kind) histogram, strided rows);
  cfg5_boxes / cfg5_rows: rows of the n = 96 matvec (1/r, p = 6, u of seed 4)
      on corner, face, interior and octant-boundary leaf boxes, by
      oracle.mapped_sampled_matvec (the restriction of operators.py:146-155);
  m48_boxes / m48_rows: the same for n = 48, leaf 6 (levels with 24 x 6 and
      12 x 6 non-square factors), u = default_rng(48).standard_normal.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import htlr_oracle as O  # noqa: E402

K_INVR = O.Kernel("slp3d", scale=4 * np.pi)
# side-6 leaf boxes at n = 96: corner, face, interior, and one touching the
# octant planes (48) along all three axes
CFG5_BOXES = [((0, 6), (0, 6), (0, 6)), ((90, 96), (42, 48), (24, 30)), ((30, 36), (60, 66), (54, 60)),
              ((42, 48), (48, 54), (42, 48))]
M48_BOXES = [((0, 6), (42, 48), (18, 24)), ((24, 30), (18, 24), (30, 36))]


def problem(n):
    return O.MappedProblem(d=3, geo=O.MappedGeometry(n, 0.05), rank=6, leaf_side_max=8 if n == 96 else 6,
                           kernel=K_INVR, coeff=O.constant_coeff(0.0))


def main():
    out = {}
    t0 = time.time()
    pb = problem(96)
    leaves = O.mapped_block_leaves(pb.geo, 3, 8, "strong", 1.0)
    arr = O.leaves_to_array(leaves, 3)
    out["cfg5_sha"] = np.frombuffer(hashlib.sha256(np.ascontiguousarray(arr, dtype=np.int32).tobytes()).digest(),
                                    dtype=np.uint8)
    hist = np.zeros((16, 2), dtype=np.int64)
    np.add.at(hist, (arr[:, 2], arr[:, 1]), 1)
    out["cfg5_hist"] = hist
    idx = np.arange(0, len(arr), 997)
    out["cfg5_spotidx"] = idx
    out["cfg5_spot"] = arr[idx]
    print("cfg5 lists", len(arr), f"{time.time() - t0:.0f}s", flush=True)
    u = np.random.default_rng(4).uniform(-1, 1, 96 ** 3)
    out["cfg5_boxes"] = np.asarray(CFG5_BOXES, dtype=np.int64)
    out["cfg5_rows"] = O.mapped_sampled_matvec(pb, u, CFG5_BOXES, leaves)
    print("cfg5 rows", f"{time.time() - t0:.0f}s", flush=True)
    pb48 = problem(48)
    u48 = np.random.default_rng(48).standard_normal(48 ** 3)
    out["m48_boxes"] = np.asarray(M48_BOXES, dtype=np.int64)
    out["m48_rows"] = O.mapped_sampled_matvec(pb48, u48, M48_BOXES)
    print("m48 rows", f"{time.time() - t0:.0f}s", flush=True)
    np.savez_compressed(os.path.join(HERE, "mapped.npz"), **out)


if __name__ == "__main__":
    main()
