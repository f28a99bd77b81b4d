"""CPU: host-side planning of the persistent step kernel (engine.py) — the
work split and counter weights the kernel's dependency counters rely on.

* participants(): never more CTAs than 32-row groups; tile-aligned counts
  keep every range inside one tile;
* max_contributors(): bound on the split-K slots of the LM-head workspace;
* weighted_ranges() (gate/up split): contiguous cover of every 32-row group,
  at most two tiles per CTA, and the counter weights of each tile's
  contributors sum to CONTRIB exactly (the consumers' wait target).
"""

from __future__ import annotations

import pytest

from paper_2408_14690_b200 import engine as E


@pytest.mark.parametrize("ntiles,m,grid", [(112, 4096, 296), (112, 4096, 264), (224, 8192, 296), (56, 2048, 148)])
@pytest.mark.parametrize("penalty", [1, 6, 10])
def test_weighted_ranges_cover_and_weights(ntiles, m, grid, penalty):
    rs = E.weighted_ranges(ntiles, m, grid, penalty)
    gpt = -(-m // 32)
    F = ntiles * gpt
    assert rs is not None and 1 <= len(rs) <= grid
    assert rs[0][0] == 0 and rs[-1][1] == F
    tot = {}
    for i, (a, b, w0, w1) in enumerate(rs):
        assert a < b
        if i:
            assert rs[i - 1][1] == a
        tiles = list(range(a // gpt, (b - 1) // gpt + 1))
        assert 1 <= len(tiles) <= 2
        if len(tiles) == 1:
            assert w1 == 0
        for t, w in zip(tiles, (w0, w1)):
            assert w >= 1
            tot[t] = tot.get(t, 0) + w
    assert sorted(tot) == list(range(ntiles))
    assert all(v == E.CONTRIB for v in tot.values())


def test_weighted_ranges_balance():
    # two-tile CTAs carry `penalty` fewer groups than one-tile CTAs (+-1)
    pen = 10
    rs = E.weighted_ranges(112, 4096, 296, pen)
    gpt = 128
    cost = [(b - a) + pen * ((b - 1) // gpt - a // gpt) for a, b, _, _ in rs]
    assert max(cost) - min(cost[:-1]) <= pen


@pytest.mark.parametrize("ntiles,m,grid", [(24, 4096, 296), (16, 4096, 296), (16, 14336, 296)])
def test_weighted_ranges_not_needed_when_aligned(ntiles, m, grid):
    # participants() already aligns these to the tile count: one tile per range
    assert E.weighted_ranges(ntiles, m, grid, 10) is None
    F = ntiles * (m // 32)
    G = E.participants(ntiles, F, grid)
    assert G % ntiles == 0 and G <= grid


def test_participants_and_contributors():
    assert E.participants(8, 5, 296) == 5           # fewer groups than CTAs
    assert E.participants(16, 2048, 296) == 288     # aligned to 16 tiles (>= 90 % busy)
    assert E.participants(112, 14336, 296) == 296   # 224 would idle 24 % of the grid
    assert E.max_contributors(16, 4096, 296) == 18
    assert E.max_contributors(501, 4096, 296) >= 1
