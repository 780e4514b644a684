#!/usr/bin/env python
"""Case 2 / Eq. 7 exercised: how the performance model's
ranking moves when the grid spans nodes (g_node < G).

For G = 8 and 16 GPUs, g_node in {1, 2, 4, 8} (< G), the GPT 20B / 40B / 80B
blocks (Table II, m = 16384 tokens, phase A) are ranked by axonn_grid_select:
levels whose group fits in a node (prod_{j<=i} G_j <= g_node) take the
measured Case-1 table of this B200 pool (profiles/case1_table.json, entries
it lacks take the mean of the measured ones), the others Eq. 7,
beta_inter / min(g_node, prod_{j<i} G_j).  beta_inter is
the node-pair bidirectional bandwidth: 4 Slingshot-11 NICs x 25 GB/s
 and, for a B200-era node, 8 x 50 GB/s.
Host-only (the model is pure host code); writes profiles/r02_case2_sweep.json.
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2502_08145_b200 as ax  # noqa: E402
from bench import HIDDEN, block_layers, case1_table  # noqa: E402


def levels(cfg, g_node):
    """'1' (Case 1, in-node table) or '2' (Eq. 7) per level X, Y, Z, DATA; '-' if G_i = 1."""
    out, inner = "", 1
    for gi in cfg:
        out += "-" if gi == 1 else ("1" if inner * gi <= g_node else "2")
        inner *= gi
    return out


def main():
    tb, src = case1_table()
    res = {"table": src, "beta_inter_GBps": [100, 400], "cases": []}
    for G in (8, 16):
        for g_node in (1, 2, 4, 8):
            if g_node >= G:
                continue
            for binter in (100e9, 400e9):
                for model in ("20B", "40B", "80B"):
                    layers = block_layers(HIDDEN[model], 16384)
                    # the Case-1 table only covers groups inside one node
                    t = {k: v for k, v in tb.items() if k[0] * k[1] <= g_node}
                    ranked = ax.axonn_grid_select(layers, G, g_node, t, binter, 2, 0)
                    top = [{"grid": [r["gx"], r["gy"], r["gz"], r["gd"]],
                            "t_comm_ms": r["t_comm"] * 1e3,
                            "levels": levels((r["gx"], r["gy"], r["gz"], r["gd"]), g_node)}
                           for r in ranked[:5]]
                    res["cases"].append({
                        "G": G, "g_node": g_node, "beta_inter_GBps": binter / 1e9, "model": model,
                        "n_grids": len(ranked), "top5": top})
    out = os.path.join(ROOT, "profiles", "r02_case2_sweep.json")
    json.dump(res, open(out, "w"), indent=1)
    for c in res["cases"]:
        t = c["top5"]
        print(f"G={c['G']:2d} g_node={c['g_node']} beta_inter={c['beta_inter_GBps']:.0f} GB/s "
              f"{c['model']}: " + "; ".join(f"{tuple(x['grid'])} {x['t_comm_ms']:.1f} ms [{x['levels']}]"
                                             for x in t[:3]))


if __name__ == "__main__":
    main()
