"""Pins of oracle.act (GeLU between fc1 and fc2, reading R18) against what
the mathematics fixes: printed normal-CDF values, the odd-part identity, the
derivative by central differences, and the block's gradients by finite
differences of L = Σ O ⊙ dY."""
import math

import numpy as np
import pytest

from oracle import act


def test_table_values():
    # Φ(1), Φ(2) from standard normal tables (Abramowitz & Stegun 26.2)
    assert act.gelu(1.0) == pytest.approx(0.8413447460685429, abs=1e-15)
    assert act.gelu(-1.0) == pytest.approx(-0.15865525393145707, abs=1e-15)
    assert act.gelu(2.0) == pytest.approx(2 * 0.9772498680518208, abs=1e-15)
    assert act.gelu(0.0) == 0.0
    assert act.gelu_grad(0.0) == 0.5            # Φ(0) + 0·φ(0)


def test_odd_part_identity():
    # Φ(x) + Φ(-x) = 1  =>  GELU(x) - GELU(-x) = x
    x = np.linspace(-6, 6, 241)
    np.testing.assert_allclose(act.gelu(x) - act.gelu(-x), x, rtol=0, atol=1e-14)
    # large |x|: GELU(x) -> x (x > 0), -> 0 (x < 0)
    assert act.gelu(10.0) == pytest.approx(10.0, abs=1e-15)
    assert abs(act.gelu(-10.0)) < 1e-20


def test_derivative_by_central_differences():
    x = np.linspace(-4, 4, 81)
    h = 1e-6
    fd = (act.gelu(x + h) - act.gelu(x - h)) / (2 * h)
    np.testing.assert_allclose(act.gelu_grad(x), fd, rtol=0, atol=1e-8)


def test_mlp_gradients_by_finite_differences():
    rng = np.random.default_rng(5)
    m, h, f = 5, 4, 6
    X = rng.uniform(-1, 1, (m, h))
    W1 = rng.uniform(-1, 1, (h, f))
    W2 = rng.uniform(-1, 1, (f, h))
    dY = rng.uniform(-1, 1, (m, h))
    r = act.mlp(X, W1, W2, dY)

    def loss(X_, W1_, W2_):
        return float(np.sum(act.mlp(X_, W1_, W2_, dY)["O"] * dY))
    eps = 1e-6
    for name, arr, grad in (("X", X, r["dX"]), ("W1", W1, r["dW1"]), ("W2", W2, r["dW2"])):
        for idx in [(0, 0), (1, 2), (arr.shape[0] - 1, arr.shape[1] - 1)]:
            a, b = arr.copy(), arr.copy()
            a[idx] += eps
            b[idx] -= eps
            args_a = {"X": X, "W1": W1, "W2": W2}
            args_b = dict(args_a)
            args_a[name], args_b[name] = a, b
            fd = (loss(**{k + "_": v for k, v in args_a.items()}) -
                  loss(**{k + "_": v for k, v in args_b.items()})) / (2 * eps)
            assert grad[idx] == pytest.approx(fd, rel=1e-6, abs=1e-8), (name, idx)
    # the pieces the library's kernels produce
    np.testing.assert_array_equal(r["A"], act.gelu(r["Z"]))
    np.testing.assert_allclose(r["dZ"], r["dA"] * act.gelu_grad(r["Z"]), rtol=0, atol=0)
