#!/usr/bin/env python
"""Rank statistics of saved grid sweeps (profiles/r01_grid_sweep_*.json):
tie-aware Spearman (average ranks; the model's exact Z-vs-DP ties, R12) and
Kendall's tau-b of predicted t_comm vs measured step time, plus top-3 hits.

    python tools/sweep_stats.py profiles/r01_grid_sweep_G4_20B_fused.json ...
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from grid_sweep import kendall_tau_b, spearman  # noqa: E402


def stats(path):
    d = json.load(open(path))
    g = d["grids"]
    t = [x["ms_per_step"] for x in g]
    out = {"file": os.path.basename(path), "G": d["G"], "model": d["model"], "grids": len(g)}
    for tag, key in (("uniform", "model_t_comm_uniform"), ("measured", "model_t_comm_measured_beta")):
        p = [x[key] for x in g]
        out[f"spearman_{tag}"] = spearman(p, t)
        out[f"kendall_{tag}"] = kendall_tau_b(p, t)
    out["top3_hits_uniform"] = d.get("top3_hits_uniform")
    return out


if __name__ == "__main__":
    for f in sys.argv[1:]:
        s = stats(f)
        print(f"| {s['model']} | {s['G']} | {s['grids']} | {s['spearman_uniform']:.3f} | "
              f"{s['kendall_uniform']:.3f} | {s['spearman_measured']:.3f} | "
              f"{s['kendall_measured']:.3f} | {s['top3_hits_uniform']}/3 |")
