"""Model-flop accounting and efficiency (Table III).

Per FC layer step the paper runs one forward MM and two backward MMs
(PAPER.md:330-335), each 2·m·k·n flops: 6·m·k·n per layer step.
Activation checkpointing re-runs the forward MM: 8·m·k·n.
"""
from __future__ import annotations


def layer_flops(m: int, k: int, n: int, recompute: bool = False) -> int:
    """2mkn forward + 2·2mkn backward (+2mkn with recompute)."""
    return (8 if recompute else 6) * m * k * n


def network_flops(layers, recompute: bool = False) -> int:
    """Sum of layer_flops over (m, k, n) triples."""
    return sum(layer_flops(m, k, n, recompute) for (m, k, n) in layers)


def efficiency(total_flops_per_s: float, workers: int, advertised: float, empirical: float):
    """Per-worker flop/s and % of advertised / empirical peak."""
    per = total_flops_per_s / workers
    return {"per_worker": per,
            "pct_advertised": 100.0 * per / advertised,
            "pct_empirical": 100.0 * per / empirical}
