"""Pins of oracle.grid and oracle.ring."""
import json
import os
from math import comb
from itertools import product

import numpy as np
import pytest

from oracle import grid, ring

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_paper_group_example():
    g = json.load(open(os.path.join(GOLD, "paper_group_example.json")))
    cfg = tuple(g["cfg"])
    xs = [tuple(x) for x in grid.groups(cfg, "x") if max(x) < 8]
    ys = [tuple(y) for y in grid.groups(cfg, "y") if max(y) < 8]
    assert xs == [tuple(p) for p in g["x_groups_among_first_8"]]
    assert ys == [tuple(p) for p in g["y_groups_among_first_8"]]


def test_z_groups_of_2x2x2():
    # SPEC.md:63 example, derived from the bijection by hand
    assert grid.groups((2, 2, 2, 1), "z") == [(0, 4), (1, 5), (2, 6), (3, 7)]
    assert grid.groups((2, 2, 2, 2), "d") == [(r, r + 8) for r in range(8)]


@pytest.mark.parametrize("cfg", [(1, 1, 1, 1), (2, 3, 1, 2), (4, 1, 2, 2), (1, 2, 2, 4), (3, 2, 2, 1)])
def test_bijection_and_partition(cfg):
    G = cfg[0] * cfg[1] * cfg[2] * cfg[3]
    seen = set()
    for r in range(G):
        c = grid.rank_to_coords(r, cfg)
        assert grid.coords_to_rank(c, cfg) == r
        seen.add(c)
    assert len(seen) == G
    for a, axis in enumerate(grid.AXES):
        gs = grid.groups(cfg, axis)
        assert sorted(r for g_ in gs for r in g_) == list(range(G))
        assert all(len(g_) == cfg[a] for g_ in gs)
        for g_ in gs:     # members differ only in the axis coordinate, ordered by it
            cs = [grid.rank_to_coords(r, cfg) for r in g_]
            assert [c[a] for c in cs] == list(range(cfg[a]))
            others = {tuple(c[:a] + c[a + 1:]) for c in cs}
            assert len(others) == 1
    # X innermost: X groups are runs of consecutive ranks
    for g_ in grid.groups(cfg, "x"):
        assert list(g_) == list(range(g_[0], g_[0] + cfg[0]))


def _count_closed_form(G, fixed_gd=0):
    # ordered factorisations into 4 slots: Π_p C(a_p + 3, 3) for G = Π p^a_p
    n, out, p = G, 1, 2
    exps = []
    while n > 1:
        a = 0
        while n % p == 0:
            n //= p
            a += 1
        if a:
            exps.append(a)
        p += 1
    if fixed_gd == 1:
        for a in exps:
            out *= comb(a + 2, 2)
        return out
    for a in exps:
        out *= comb(a + 3, 3)
    return out


@pytest.mark.parametrize("G,gd,count", [(1, 0, 1), (2, 0, 4), (4, 0, 10), (8, 0, 20), (16, 0, 35),
                                        (32, 1, 21), (12, 0, 40), (8, 1, 10)])
def test_enumeration_counts(G, gd, count):
    cf = grid.enumerate_configs(G, gd)
    assert len(cf) == count == _count_closed_form(G, gd)
    assert len(set(cf)) == len(cf)
    assert cf == sorted(cf)
    assert all(c[0] * c[1] * c[2] * c[3] == G for c in cf)


def test_config_errors():
    with pytest.raises(ValueError, match="configuration error"):
        grid.check_config(8, (2, 2, 2, 2))
    with pytest.raises(ValueError, match="configuration error"):
        grid.check_config(0, (0, 1, 1, 1))


# ---------------------------------------------------------------- ring

def test_ring_small_examples():
    out, sent = ring.all_gather([np.array([1, 2]), np.array([3, 4])])
    assert [list(o) for o in out] == [[1, 2, 3, 4]] * 2 and sent == [2, 2]
    out, sent = ring.reduce_scatter([np.array([1, 2, 3, 4]), np.array([5, 6, 7, 8])])
    assert [list(o) for o in out] == [[6, 8], [10, 12]] and sent == [2, 2]
    out, sent = ring.all_reduce([np.array([1, 2]), np.array([3, 4])])
    assert [list(o) for o in out] == [[4, 6], [4, 6]] and sent == [2, 2]
    out, sent = ring.all_gather([np.array([5.0, 6.0])])
    assert list(out[0]) == [5.0, 6.0] and sent == [0]


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 8])
def test_ring_against_naive_and_volumes(p):
    rng = np.random.default_rng(p)
    n = 12 * p
    vecs = [rng.integers(-9, 10, n).astype(float) for _ in range(p)]
    total = np.sum(vecs, axis=0)
    rs, sent = ring.reduce_scatter(vecs)
    for r in range(p):
        np.testing.assert_array_equal(rs[r], total[r * 12:(r + 1) * 12])
    assert sent == [(p - 1) * n // p] * p
    ar, sent = ring.all_reduce(vecs)
    for r in range(p):
        np.testing.assert_array_equal(ar[r], total)
    assert sent == [2 * (p - 1) * n // p] * p
    ag, sent = ring.all_gather([v[:7] for v in vecs])
    for r in range(p):
        np.testing.assert_array_equal(ag[r], np.concatenate([v[:7] for v in vecs]))
    assert sent == [(p - 1) * 7] * p


def test_ring_protocol_errors():
    with pytest.raises(ValueError, match="protocol"):
        ring.all_gather([np.zeros(2), np.zeros(3)])
    with pytest.raises(ValueError, match="protocol"):
        ring.reduce_scatter([np.zeros(3), np.zeros(3)])
