"""The rank statistics the model validation reports (tools/grid_sweep.py)."""
import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
gs = pytest.importorskip("grid_sweep")


def test_tie_ranks_average():
    assert list(gs.tie_ranks([3.0, 1.0, 1.0, 2.0])) == [4.0, 1.5, 1.5, 3.0]
    # R12 tolerance: values equal to 1e-12 relative are one tie
    assert list(gs.tie_ranks([1.0, 1.0 + 1e-15, 2.0])) == [1.5, 1.5, 3.0]


def test_spearman_and_kendall_perfect_reversed_and_tied():
    a = [1.0, 2.0, 3.0, 4.0]
    assert gs.spearman(a, [10, 20, 30, 40]) == pytest.approx(1.0)
    assert gs.spearman(a, [40, 30, 20, 10]) == pytest.approx(-1.0)
    assert gs.kendall_tau_b(a, [10, 20, 30, 40]) == pytest.approx(1.0)
    assert gs.kendall_tau_b(a, [40, 30, 20, 10]) == pytest.approx(-1.0)
    # a tie in the prediction is not scored as a disagreement either way
    p = [1.0, 1.0, 2.0, 3.0]
    assert gs.spearman(p, [1, 2, 3, 4]) == pytest.approx(gs.spearman(p, [2, 1, 3, 4]))
    assert gs.kendall_tau_b(p, [1, 2, 3, 4]) == pytest.approx(gs.kendall_tau_b(p, [2, 1, 3, 4]))
    # tau-b with one tied pair out of six: (5 - 0) / sqrt(5 * 6)
    assert gs.kendall_tau_b(p, [1, 2, 3, 4]) == pytest.approx(5 / (5 * 6) ** 0.5)
