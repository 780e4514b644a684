"""The paper's communication model (Eqs. 1-7) and the ranked configuration list.

PAPER.md:458-480 Eqs. 1-5 — ring-collective times of one layer:
  t_AG,z   = (1/β)·(Gz-1)·kn/(GxGyGz)                 (Eq. 1)
  t_RS,z   = (1/β)·((Gz-1)/Gz)·kn/(GxGy)              (Eq. 2)
  t_AR,y   = (2/β)·((Gy-1)/Gy)·mn/(GzGx)              (Eq. 3)
  t_AR,x   = (2/β)·((Gx-1)/Gx)·mk/(GzGy)              (Eq. 4)
  t_AR,data= (2/β)·((Gd-1)/Gd)·kn/(GxGyGz)            (Eq. 5)
PAPER.md:482-492 Eq. 6 — t_comm is their sum; transposed layers swap Gx and
Gy; the network time is the sum over layers.
PAPER.md:505-537 Case 1 — a group inside a node takes its bandwidth from a
profiled database keyed by (G0 = ∏_{j<i} G_j, G1 = G_i).
PAPER.md:547-593 Case 2, Eq. 7 — β_i = β_inter / min(G_node, ∏_{j<i} G_j).
PAPER.md:594-597 — "create an ordered list of configurations".

Readings: Eqs. count elements, multiplied by bytes per element b
(R7, b = 2 for bf16); m is the per-replica row count m/G_data (R5); β_z goes
with Eqs. 1-2, β_y with Eq. 3, β_x with Eq. 4, β_data with Eq. 5 and
transposed layers swap both G and β of X and Y (R10); singleton groups
contribute exactly 0 (R11); ties are broken lexicographically on
(Gx, Gy, Gz, Gd) (R12).

The oracle computes bytes exactly (``fractions.Fraction``) and times as exact
rationals of the (binary-exact) float bandwidths, so its ranking has no
rounding-order ambiguity.
"""
from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction
from math import inf

from . import grid as gridmod


@dataclass(frozen=True)
class Layer:
    m: int          # global tokens (rows of X) of the whole data-parallel job
    k: int          # input features
    n: int          # output features
    transposed: bool = False


def gpt_block(h: int, m: int, phase: str = "A"):
    """The four FC layers of one GPT block (Table II shapes).

    QKV h->3h, proj h->h, fc1 h->4h, fc2 4h->h (12h² weights per block).
    Phase A transposes proj and fc2; phase B transposes QKV and fc1
    (reading R2b: the paper fixes only the alternation).
    """
    if phase not in ("A", "B"):
        raise ValueError(f"phase must be 'A' or 'B' (reading R2b), got {phase!r}")
    shapes = [(h, 3 * h), (h, h), (h, 4 * h), (4 * h, h)]
    flags = [False, True, False, True] if phase == "A" else [True, False, True, False]
    return [Layer(m, k, n, t) for (k, n), t in zip(shapes, flags)]


def effective_bandwidths(cfg, g_node: int, table: dict, beta_inter: float):
    """β⃗ = (β_x, β_y, β_z, β_data) for the hierarchy X, Y, Z, DATA.

    Case 1 (∏_{j<=i} G_j <= G_node): table[(∏_{j<i} G_j, G_i)].
    Case 2: Eq. 7, β_inter / min(G_node, ∏_{j<i} G_j).
    Singleton groups get +inf (no communication, R11).
    """
    betas = []
    inner = 1
    for gi in cfg:
        if gi == 1:
            betas.append(inf)
        elif inner * gi <= g_node:
            key = (inner, gi)
            if key not in table:
                raise KeyError(f"configuration error: bandwidth table has no entry (G0={inner}, G1={gi})")
            betas.append(float(table[key]))
        else:
            betas.append(float(beta_inter) / min(g_node, inner))
        inner *= gi
    return tuple(betas)


def layer_bytes(layer: Layer, cfg, b: int = 2, b_grad: int | None = None):
    """Per-rank bytes of Eqs. 1-5 for one layer, exact.

    Returns dict with keys ag_z, rs_z, ar_y (Eq. 3 form: the forward
    all-reduce), ar_x (Eq. 4 form: the backward dI all-reduce), ar_d, and
    the axes they physically run on.  b_grad (default b) is the element size
    of the two gradient reductions, Eqs. 2 and 5 (reading R17: gradients
    reduced in fp32 while weights and activations move in bf16).
    """
    bg = b if b_grad is None else b_grad
    gx, gy, gz, gd = cfg
    if layer.transposed:               # swap Gx and Gy
        gx, gy = gy, gx
    m = Fraction(layer.m, gd)          # R5: per-replica rows
    k, n = layer.k, layer.n
    F = Fraction
    return {
        "ag_z": F(gz - 1) * F(k * n, gx * gy * gz) * b,
        "rs_z": F(gz - 1, gz) * F(k * n, gx * gy) * bg,
        "ar_y": 2 * F(gy - 1, gy) * m * F(n, gz * gx) * b,
        "ar_x": 2 * F(gx - 1, gx) * m * F(k, gz * gy) * b,
        "ar_d": 2 * F(gd - 1, gd) * F(k * n, gx * gy * gz) * bg,
    }


def layer_times(layer: Layer, cfg, betas, b: int = 2, b_grad: int | None = None):
    """Eqs. 1-6 for one layer: exact rational seconds per term and t_comm."""
    bx, by, bz, bd = betas
    if layer.transposed:               # swap β of X and Y with G (R10)
        bx, by = by, bx
    by_term = {"ag_z": bz, "rs_z": bz, "ar_y": by, "ar_x": bx, "ar_d": bd}
    byts = layer_bytes(layer, cfg, b, b_grad)
    t = {}
    for key, nbytes in byts.items():
        beta = by_term[key]
        t[key] = Fraction(0) if nbytes == 0 or beta == inf else nbytes / Fraction(beta)
    t["comm"] = sum(t[key] for key in byts)  # Eq. 6
    return t


def feasible(layer: Layer, cfg) -> bool:
    """Divisibility of the shards (no padding)."""
    gx, gy, gz, gd = cfg
    ga, gb = (gx, gy) if layer.transposed else (gy, gx)
    if layer.m % (gz * gd) or layer.k % ga or layer.n % gb:
        return False
    return ((layer.k // ga) * (layer.n // gb)) % gz == 0


def network_times(layers, cfg, betas, b: int = 2, b_grad: int | None = None):
    """Sum of Eq. 6 over all layers."""
    tot = {key: Fraction(0) for key in ("ag_z", "rs_z", "ar_y", "ar_x", "ar_d", "comm")}
    for L in layers:
        t = layer_times(L, cfg, betas, b, b_grad)
        for key in tot:
            tot[key] += t[key]
    return tot


def rank_configs(layers, G: int, g_node: int, table: dict, beta_inter: float,
                 b: int = 2, fixed_gd: int = 0, b_grad: int | None = None):
    """Ordered list of (cfg, times) — the model's ranking.

    Enumerates every (Gx, Gy, Gz, Gd) with product G, drops the ones that do
    not divide every layer, scores each by Σ_layers t_comm and sorts
    ascending, ties broken by (Gx, Gy, Gz, Gd).  Raises on an empty set
    ("no feasible configuration").
    """
    out = []
    for cfg in gridmod.enumerate_configs(G, fixed_gd):
        if not all(feasible(L, cfg) for L in layers):
            continue
        betas = effective_bandwidths(cfg, g_node, table, beta_inter)
        out.append((cfg, network_times(layers, cfg, betas, b, b_grad)))
    if not out:
        raise ValueError("infeasible: no configuration divides every layer")
    out.sort(key=lambda e: (e[1]["comm"], e[0]))
    return out


def uniform_table(G_node: int, beta: float) -> dict:
    """A Case-1 database with the same β for every (G0, G1), G0·G1 <= G_node."""
    return {(g0, g1): beta for g0 in range(1, G_node + 1) for g1 in range(2, G_node + 1)
            if g0 * g1 <= G_node}
