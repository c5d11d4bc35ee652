"""CPU check of the product-set structure the banded passes rely on
(htlr_sep.cu, sep_band_kernel / sep_band_xy_kernel; DESIGN.md "Banded
passes"): with strong admissibility at eta = 1 on a uniform 3-D grid, the
(kind, offset) set a target box meets at a level L >= 2 is, per axis with c =
the box coordinate parity,

    leaf level:  adm = (R10^3 minus A4^3) minus near,  near = R5^3 minus {+-2}^3
    coupling:    adm = (R10^3 minus A4^3) minus near   (near pairs are refined)

R10 = {-4-c..5-c}, A4 = {-4-c, -3-c, 4-c, 5-c}, R5 = {-2..2}, clipped to the
domain.  The multiset of signed Kronecker terms C10^3 - C4^3 - C5^3 + C2^3
(+ E5^3 - E2^3) then covers every listed block exactly once.  Checked here
against the oracle's restatement of the reference's block cluster tree
(grids.py:268-296, pinned to the reference fixtures in test_oracle_golden.py);
the device plan runs the same check on its own lists before enabling the
banded passes."""

from collections import Counter, defaultdict
from itertools import product

import pytest

from oracle import htlr_oracle as O


def expected(tc, nb, leaf):
    want = {}
    for o in product(range(-5, 6), repeat=3):
        s = [tc[a] + o[a] for a in range(3)]
        if min(s) < 0 or max(s) >= nb:
            continue
        c = [t & 1 for t in tc]
        in10 = all(-4 - c[a] <= o[a] <= 5 - c[a] for a in range(3))
        in_a4 = all(o[a] <= -3 - c[a] or o[a] >= 4 - c[a] for a in range(3))
        in5 = all(-2 <= v <= 2 for v in o)
        corner = all(abs(v) == 2 for v in o)
        if not in10 or in_a4:
            continue
        near = in5 and not corner
        if near and not leaf:
            continue
        want[o] = O.NEAR if near else O.ADM
    return want


def signed_cover(tc, nb, leaf):
    """Multiplicity of every (kind, offset) under the signed term expansion."""
    c = [t & 1 for t in tc]
    sets = {
        "R10": lambda a: range(-4 - c[a], 6 - c[a]),
        "A4": lambda a: (-4 - c[a], -3 - c[a], 4 - c[a], 5 - c[a]),
        "R5": lambda a: range(-2, 3),
        "C2": lambda a: (-2, 2),
    }
    terms = [(+1, O.ADM, "R10"), (-1, O.ADM, "A4"), (-1, O.ADM, "R5"), (+1, O.ADM, "C2")]
    if leaf:
        terms += [(+1, O.NEAR, "R5"), (-1, O.NEAR, "C2")]
    cover = Counter()
    for sign, kind, name in terms:
        for o in product(*(sets[name](a) for a in range(3))):
            s = [tc[a] + o[a] for a in range(3)]
            if min(s) < 0 or max(s) >= nb:
                continue
            cover[(kind, o)] += sign
    return {k: v for k, v in cover.items() if v != 0}


@pytest.mark.parametrize("n", [32, 64])
def test_leaf_lists_are_product_sets(n):
    leaves = O.block_leaves(n, 3, 8)
    L = max(lf.level for lf in leaves)
    got = defaultdict(dict)   # (level, target coords) -> {offset: kind}
    for lf in leaves:
        side = lf.tau[0][1] - lf.tau[0][0]
        tc = tuple(r[0] // side for r in lf.tau)
        o = tuple((lf.sigma[a][0] - lf.tau[a][0]) // side for a in range(3))
        assert o not in got[(lf.level, tc)]
        got[(lf.level, tc)][o] = lf.kind
    checked = 0
    for (level, tc), have in got.items():
        if level < 2:
            continue
        nb = 1 << level
        leaf = level == L
        want = expected(tc, nb, leaf)
        assert have == want, (level, tc)
        # the signed terms cover each listed block exactly once and nothing else
        cover = signed_cover(tc, nb, leaf)
        assert cover == {(k, o): 1 for o, k in want.items()}, (level, tc)
        checked += 1
    assert checked > 0
