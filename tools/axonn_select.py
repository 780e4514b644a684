#!/usr/bin/env python
"""The paper's offline configuration selection (Eqs. 1-7) as
a command: rank every (Gx, Gy, Gz, Gd) of G GPUs for a GPT block by its
modelled communication time, with the Case-1 bandwidth table measured on this
box (profiles/case1_table.json; missing entries at their mean) or uniform β,
and Eq. 7 for groups that cross `--gnode`.  Runs on the host (libaxonn's
axonn_grid_select), no GPU needed.

    python tools/axonn_select.py --model 20B --gpus 8 [--tokens 16384] [--gnode 8]
                                 [--phase A] [--top 10] [--fixed-gd 0] [--grad-f32]
                                 [--uniform GBps] [--beta-inter GBps]
"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def rank(model, gpus, tokens=16384, gnode=8, phase="A", fixed_gd=0, grad_f32=False,
         uniform=None, beta_inter=25.0):
    import paper_2502_08145_b200 as ax
    from bench import HIDDEN, block_layers, case1_table
    layers = block_layers(HIDDEN[model], tokens, phase)
    if uniform:
        full = [(g0, g1) for g0 in range(1, gnode + 1) for g1 in range(2, gnode + 1)
                if g0 * g1 <= gnode]
        table, src = {k: uniform * 1e9 for k in full}, f"uniform {uniform} GB/s"
    else:
        table, src = case1_table()
    rows = ax.axonn_grid_select(layers, gpus, gnode, table, beta_inter * 1e9, 2, fixed_gd,
                                grad_bytes_per_elem=4 if grad_f32 else None)
    return rows, src


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--model", default="20B", choices=["5B", "10B", "20B", "40B", "80B"])
    ap.add_argument("--gpus", type=int, default=8)
    ap.add_argument("--tokens", type=int, default=16384, help="global tokens per step (m)")
    ap.add_argument("--gnode", type=int, default=8, help="GPUs per node (Case 1 inside)")
    ap.add_argument("--phase", default="A", choices=["A", "B"])
    ap.add_argument("--top", type=int, default=10)
    ap.add_argument("--fixed-gd", type=int, default=0)
    ap.add_argument("--grad-f32", action="store_true", help="b = 4 in Eqs. 2 and 5")
    ap.add_argument("--uniform", type=float, default=None, help="uniform intra-node GB/s")
    ap.add_argument("--beta-inter", type=float, default=25.0, help="inter-node GB/s (Eq. 7)")
    a = ap.parse_args(argv)
    rows, src = rank(a.model, a.gpus, a.tokens, a.gnode, a.phase, a.fixed_gd, a.grad_f32,
                     a.uniform, a.beta_inter)
    print(f"# GPT-{a.model} block, m = {a.tokens}, G = {a.gpus}, g_node = {a.gnode}, phase {a.phase}; "
          f"bandwidths: {src}")
    print(f"{'rank':>4} {'Gx,Gy,Gz,Gd':>12} {'AG_z':>8} {'RS_z':>8} {'AR_y':>8} {'AR_x':>8} "
          f"{'AR_d':>8} {'t_comm ms':>10}")
    for i, r in enumerate(rows[:a.top]):
        g = f"{r['gx']},{r['gy']},{r['gz']},{r['gd']}"
        print(f"{i + 1:>4} {g:>12} " + " ".join(f"{r[k] * 1e3:8.3f}" for k in
                                                ("t_ag_z", "t_rs_z", "t_ar_y", "t_ar_x", "t_ar_data"))
              + f" {r['t_comm'] * 1e3:10.3f}")
    return rows


if __name__ == "__main__":
    main()
