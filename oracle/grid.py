"""The 4D virtual grid: rank <-> coordinates, process groups, enumeration.

PAPER.md:307-317 (§IV-A "Data Parallelism"): G GPUs form a
G_data × G_tensor grid; G_tensor = G_x × G_y × G_z.
PAPER.md:505-510 (§IV-B): hierarchy "X-tensor parallelism (innermost),
followed by Y-tensor parallelism, Z-tensor parallelism, and data parallelism
(outermost)"; worked example "X ... GPU pairs (0,1), (2,3), (4,5), and (6,7)
... Y ... (0,2), (1,3), (4,6), and (5,7)".

Reading (R3): the example says "eight GPUs" with all four extents 2,
which is 16 GPUs; the listed pairs are the first 8 ranks of the bijection
below, which is what the hierarchy sentence fixes.
"""
from __future__ import annotations

from itertools import product

AXES = ("x", "y", "z", "d")


def check_config(G: int, cfg) -> None:
    """Configuration errors: zero factor or product != G."""
    if len(cfg) != 4:
        raise ValueError("config must be (gx, gy, gz, gd)")
    if any(int(c) < 1 for c in cfg):
        raise ValueError(f"configuration error: zero or negative factor in {tuple(cfg)}")
    p = cfg[0] * cfg[1] * cfg[2] * cfg[3]
    if p != G:
        raise ValueError(f"configuration error: gx*gy*gz*gd = {p} != G = {G}")


def rank_to_coords(r: int, cfg):
    """r -> (i, j, k, d) with X innermost."""
    gx, gy, gz, gd = cfg
    i = r % gx
    r //= gx
    j = r % gy
    r //= gy
    k = r % gz
    d = r // gz
    if d >= gd:
        raise ValueError("rank out of range")
    return i, j, k, d


def coords_to_rank(c, cfg) -> int:
    """(i, j, k, d) -> r = i + Gx·(j + Gy·(k + Gz·d))."""
    gx, gy, gz, _ = cfg
    i, j, k, d = c
    return i + gx * (j + gy * (k + gz * d))


def groups(cfg, axis: str):
    """All process groups along ``axis``; members ordered by that coordinate.

    A group is the set of ranks whose other three coordinates agree
    (PAPER.md:505-510).  Returns a list of tuples, sorted by first member.
    """
    a = AXES.index(axis)
    G = cfg[0] * cfg[1] * cfg[2] * cfg[3]
    seen = {}
    for r in range(G):
        c = list(rank_to_coords(r, cfg))
        key = tuple(c[:a] + c[a + 1:])
        seen.setdefault(key, []).append((c[a], r))
    out = [tuple(r for _, r in sorted(v)) for v in seen.values()]
    return sorted(out, key=lambda g: g[0])


def group_of(r: int, cfg, axis: str):
    """The group along ``axis`` that contains rank r."""
    for g in groups(cfg, axis):
        if r in g:
            return g
    raise ValueError("rank not in grid")


def enumerate_configs(G: int, fixed_gd: int = 0):
    """All ordered (gx, gy, gz, gd) with product G, lexicographic order.

    The candidate set the performance model ranks.
    Brute force over divisors; ``fixed_gd`` > 0 pins G_data.
    """
    divs = [d for d in range(1, G + 1) if G % d == 0]
    out = []
    for gx, gy, gz in product(divs, repeat=3):
        if G % (gx * gy * gz):
            continue
        gd = G // (gx * gy * gz)
        if fixed_gd and gd != fixed_gd:
            continue
        out.append((gx, gy, gz, gd))
    return sorted(out)
