"""Ring collectives, step by step, with per-rank byte accounting.

PAPER.md:443-445 (Assumption-1): "The ring algorithm is used for implementing
the all-reduce, reduce-scatter, and all-gather collectives" (Thakur et al.;
all-reduce = reduce-scatter + all-gather, Rabenseifner — the factor 2 of
Eqs. 3-5).

Each function takes one vector per member (member order = ring order = the
coordinate along the axis) and returns one vector per member plus the number
of ELEMENTS each member sent.  Sums are fp64 in the fixed ring order, so the
simulation is deterministic.
"""
from __future__ import annotations

import numpy as np


def all_gather(shards):
    """Ring all-gather: every member ends with concat(shards) in member order.

    p-1 steps; at step s member r forwards chunk (r - s) mod p to r+1.
    Each member sends (p-1)·s elements.
    """
    p = len(shards)
    s = len(shards[0])
    if any(len(x) != s for x in shards):
        raise ValueError("protocol error: all-gather shard lengths differ")
    have = [{r: np.array(shards[r], dtype=np.float64)} for r in range(p)]
    sent = [0] * p
    for step in range(p - 1):
        msgs = []
        for r in range(p):
            c = (r - step) % p
            msgs.append(((r + 1) % p, c, have[r][c]))
            sent[r] += s
        for dst, c, v in msgs:
            have[dst][c] = v
    out = [np.concatenate([have[r][c] for c in range(p)]) if p > 1 else have[r][0]
           for r in range(p)]
    return out, sent


def reduce_scatter(vecs):
    """Ring reduce-scatter: member r ends with segment r of the element-wise sum.

    The vector is cut into p equal segments.  At step s (0..p-2) member r sends
    its running partial of segment (r - s - 1) mod p to r+1, which adds its
    own contribution.  After p-1 steps member r holds segment r, summed in the
    ring order r+1, r+2, ..., r.  Each member sends (p-1)/p·n elements
    (SPEC.md:140).
    """
    p = len(vecs)
    n = len(vecs[0])
    if any(len(v) != n for v in vecs):
        raise ValueError("protocol error: reduce-scatter lengths differ")
    if n % p:
        raise ValueError("protocol error: length not divisible by group size")
    seg = n // p
    part = [[np.array(v[c * seg:(c + 1) * seg], dtype=np.float64) for c in range(p)]
            for v in vecs]
    sent = [0] * p
    for step in range(p - 1):
        msgs = []
        for r in range(p):
            c = (r - step - 1) % p
            msgs.append(((r + 1) % p, c, part[r][c].copy()))
            sent[r] += seg
        for dst, c, v in msgs:
            part[dst][c] = part[dst][c] + v
    return [part[r][r] for r in range(p)], sent


def all_reduce(vecs):
    """Ring all-reduce = reduce-scatter then all-gather (Rabenseifner).

    Lengths not divisible by p are zero-padded and trimmed.
    Each member sends 2(p-1)/p·n elements.
    """
    p = len(vecs)
    n = len(vecs[0])
    if p == 1:
        return [np.array(vecs[0], dtype=np.float64)], [0]
    pad = (-n) % p
    padded = [np.concatenate([np.asarray(v, dtype=np.float64), np.zeros(pad)]) for v in vecs]
    segs, sent_rs = reduce_scatter(padded)
    full, sent_ag = all_gather(segs)
    return [f[:n] for f in full], [a + b for a, b in zip(sent_rs, sent_ag)]
