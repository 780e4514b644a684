"""Algorithm 1 simulated over every rank of a 4D grid.

For each rank g_{i,j,k} of each data-parallel replica d the simulation does,
in the paper's order and notation:

  forward  (Alg. 1 lines 1-7)
    line 2  W_{j,i} = all-gather_z(Ŵ_{j,i})
    line 3  Ô_{k,i} = I_{k,j} × W_{j,i}
    line 4  O_{k,i} = all-reduce_y(Ô_{k,i})
    line 5  cache I_{k,j}, W_{j,i}
  backward (Alg. 1 lines 9-15)
    line 11 dÎ_{k,j} = dO_{k,i} × W_{j,i}ᵀ
    line 12 dI_{k,j} = all-reduce_x(dÎ_{k,j})
    line 13 dŴpart   = I_{k,j}ᵀ × dO_{k,i}
    line 14 dŴ_{j,i} = reduce-scatter_z(dŴpart)
  data parallel: dŴ summed over the G_data replicas.

Readings:
  R1 follow Alg. 1's indices (contraction over Y, forward all-reduce over Y,
     backward all-reduce over X), not the Fig. 1 prose.
  R2 transposed layers swap the roles of X and Y:
     contraction over X, forward all-reduce over X, backward over Y.
  R4 Ŵ_{j,i} = k-th contiguous flat slice of W_{j,i} stored [k_l][n_l]
     row-major (PAPER.md:361-363 leave the order open).
  R5 m in Eqs. 3-4 is the per-replica row count m/G_data.
  R6 global row block of rank (k, d) is d·G_z + k (data outermost).
  R9 the data-parallel reduction is a sum.

Collectives go through ``oracle.ring`` so the per-rank bytes each collective
sends are recorded and can be compared with Eqs. 1-5 exactly.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import grid as gridmod
from . import ring


@dataclass(frozen=True)
class Geometry:
    """Shard geometry of one rank for one layer."""
    m_l: int        # rows of I_local / O_local
    k_l: int        # cols of I_local = rows of W_local
    n_l: int        # cols of W_local / O_local
    row0: int       # first global row of I_local / O_local
    in_col0: int    # first global column of I_local (= first row of W_local in W)
    out_col0: int   # first global column of O_local (= first col of W_local in W)
    what_off: int   # offset of Ŵ inside flat(W_local)
    what_len: int   # S = k_l·n_l / G_z


def check_shape(m, k, n, cfg, transposed=False) -> None:
    """Shape errors naming the axis; no padding."""
    gx, gy, gz, gd = cfg
    ga, gb = (gx, gy) if transposed else (gy, gx)   # contraction, output-col extents
    na, nb = ("Gx", "Gy") if transposed else ("Gy", "Gx")
    if m < 0 or k < 0 or n < 0:
        raise ValueError("shape error: negative dimension")
    if m % (gz * gd):
        raise ValueError(f"shape error: m={m} not divisible by Gz*Gd={gz * gd}")
    if k % ga:
        raise ValueError(f"shape error: k={k} not divisible by {na}={ga}")
    if n % gb:
        raise ValueError(f"shape error: n={n} not divisible by {nb}={gb}")
    if ((k // ga) * (n // gb)) % gz:
        raise ValueError(f"shape error: k_l*n_l={(k // ga) * (n // gb)} not divisible by Gz={gz}")


def geometry(m, k, n, cfg, rank, transposed=False) -> Geometry:
    """Placement of I_{k,j}, W_{j,i}, Ŵ_{j,i}, O_{k,i} on ``rank`` (Alg. 1)."""
    check_shape(m, k, n, cfg, transposed)
    gx, gy, gz, gd = cfg
    i, j, kz, d = gridmod.rank_to_coords(rank, cfg)
    m_l = m // (gz * gd)
    if transposed:                   # R2: rows of W over X, columns over Y
        k_l, n_l, a, b = k // gx, n // gy, i, j
    else:                            # R1: rows of W over Y, columns over X
        k_l, n_l, a, b = k // gy, n // gx, j, i
    S = (k_l * n_l) // gz
    return Geometry(m_l, k_l, n_l, (d * gz + kz) * m_l, a * k_l, b * n_l, kz * S, S)


def shard(X, W, dO, cfg, rank, transposed=False):
    """Slice I_local, Ŵ (flat), dO_local of ``rank`` from the global tensors."""
    m, k = X.shape
    n = W.shape[1]
    g = geometry(m, k, n, cfg, rank, transposed)
    I_loc = X[g.row0:g.row0 + g.m_l, g.in_col0:g.in_col0 + g.k_l]
    W_loc = W[g.in_col0:g.in_col0 + g.k_l, g.out_col0:g.out_col0 + g.n_l]
    W_hat = np.ascontiguousarray(W_loc).reshape(-1)[g.what_off:g.what_off + g.what_len]
    dO_loc = dO[g.row0:g.row0 + g.m_l, g.out_col0:g.out_col0 + g.n_l]
    return (np.array(I_loc, dtype=np.float64), np.array(W_hat, dtype=np.float64),
            np.array(dO_loc, dtype=np.float64))


@dataclass
class GridResult:
    """Per-rank outputs and per-rank bytes sent, per collective kind."""
    O: dict = field(default_factory=dict)       # rank -> O_{k,i} [m_l, n_l]
    dI: dict = field(default_factory=dict)      # rank -> dI_{k,j} [m_l, k_l]
    dW_hat: dict = field(default_factory=dict)  # rank -> dŴ_{j,i} flat [S]
    W_full: dict = field(default_factory=dict)  # rank -> gathered W_{j,i} [k_l, n_l]
    sent: dict = field(default_factory=dict)    # (kind, rank) -> elements sent


def _acc(sent, kind, members, counts):
    for r, c in zip(members, counts):
        sent[(kind, r)] = sent.get((kind, r), 0) + c


def simulate(X, W, dO, cfg, transposed=False) -> GridResult:
    """Run Algorithm 1 on every rank of ``cfg`` for one FC layer.

    X [m,k], W [k,n], dO [m,n] are the global tensors (fp64 exact copies of
    the bf16 inputs).  Returns per-rank results; gather them with
    :func:`gather_outputs` to compare with the unsharded ``oracle.fc``.
    """
    gx, gy, gz, gd = cfg
    G = gx * gy * gz * gd
    m, k = X.shape
    n = W.shape[1]
    check_shape(m, k, n, cfg, transposed)
    geo = {r: geometry(m, k, n, cfg, r, transposed) for r in range(G)}
    loc = {r: shard(X, W, dO, cfg, r, transposed) for r in range(G)}
    # Axis of the forward (contraction) all-reduce and of the backward dI one.
    ax_fwd, ax_bwd = ("x", "y") if transposed else ("y", "x")
    res = GridResult()

    # line 2: W_{j,i} = all-gather_z(Ŵ_{j,i})
    for grp in gridmod.groups(cfg, "z"):
        outs, sent = ring.all_gather([loc[r][1] for r in grp])
        _acc(res.sent, "ag_z", grp, sent)
        for r, w in zip(grp, outs):
            g = geo[r]
            res.W_full[r] = w.reshape(g.k_l, g.n_l)

    # line 3: Ô_{k,i} = I_{k,j} × W_{j,i}
    O_hat = {r: loc[r][0] @ res.W_full[r] for r in range(G)}

    # line 4: O_{k,i} = all-reduce_y(Ô_{k,i})   (over X for transposed layers)
    for grp in gridmod.groups(cfg, ax_fwd):
        outs, sent = ring.all_reduce([O_hat[r].reshape(-1) for r in grp])
        _acc(res.sent, "ar_fwd", grp, sent)
        for r, o in zip(grp, outs):
            res.O[r] = o.reshape(O_hat[r].shape)

    # line 11: dÎ_{k,j} = dO_{k,i} × W_{j,i}ᵀ
    dI_hat = {r: loc[r][2] @ res.W_full[r].T for r in range(G)}

    # line 12: dI_{k,j} = all-reduce_x(dÎ_{k,j})   (over Y for transposed layers)
    for grp in gridmod.groups(cfg, ax_bwd):
        outs, sent = ring.all_reduce([dI_hat[r].reshape(-1) for r in grp])
        _acc(res.sent, "ar_bwd", grp, sent)
        for r, v in zip(grp, outs):
            res.dI[r] = v.reshape(dI_hat[r].shape)

    # line 13: dŴpart = I_{k,j}ᵀ × dO_{k,i}
    dW_part = {r: (loc[r][0].T @ loc[r][2]).reshape(-1) for r in range(G)}

    # line 14: dŴ_{j,i} = reduce-scatter_z(dŴpart)
    dW_hat = {}
    for grp in gridmod.groups(cfg, "z"):
        outs, sent = ring.reduce_scatter([dW_part[r] for r in grp])
        _acc(res.sent, "rs_z", grp, sent)
        for r, v in zip(grp, outs):
            dW_hat[r] = v

    # data parallelism: all-reduce dŴ over the replicas (sum, R9)
    for grp in gridmod.groups(cfg, "d"):
        outs, sent = ring.all_reduce([dW_hat[r] for r in grp])
        _acc(res.sent, "ar_d", grp, sent)
        for r, v in zip(grp, outs):
            res.dW_hat[r] = v
    return res


def gather_outputs(res: GridResult, m, k, n, cfg, transposed=False):
    """Reassemble global O [m,n], dI [m,k], dW [k,n] from the per-rank shards.

    Also checks that replicas hold identical copies (every member of an
    all-reduce group must hold the same result).
    """
    G = cfg[0] * cfg[1] * cfg[2] * cfg[3]
    O = np.full((m, n), np.nan)
    dI = np.full((m, k), np.nan)
    dW = np.full((k, n), np.nan)
    for r in range(G):
        g = geometry(m, k, n, cfg, r, transposed)
        for dst, val, r0, c0 in ((O, res.O[r], g.row0, g.out_col0),
                                 (dI, res.dI[r], g.row0, g.in_col0)):
            blk = dst[r0:r0 + val.shape[0], c0:c0 + val.shape[1]]
            if not np.all(np.isnan(blk)) and not np.array_equal(blk, val):
                raise AssertionError("replicas disagree")
            dst[r0:r0 + val.shape[0], c0:c0 + val.shape[1]] = val
        wblk = dW[g.in_col0:g.in_col0 + g.k_l, g.out_col0:g.out_col0 + g.n_l]
        flat = wblk.reshape(-1).copy()
        seg = flat[g.what_off:g.what_off + g.what_len]
        if not np.all(np.isnan(seg)) and not np.array_equal(seg, res.dW_hat[r]):
            raise AssertionError("data-parallel replicas disagree on dŴ")
        flat[g.what_off:g.what_off + g.what_len] = res.dW_hat[r]
        dW[g.in_col0:g.in_col0 + g.k_l, g.out_col0:g.out_col0 + g.n_l] = flat.reshape(g.k_l, g.n_l)
    return O, dI, dW


def bytes_sent(res: GridResult, kind: str, rank: int, bytes_per_elem: int = 2) -> int:
    """Bytes one rank sent in one collective kind ('ag_z','ar_fwd','ar_bwd','rs_z','ar_d')."""
    return res.sent.get((kind, rank), 0) * bytes_per_elem
