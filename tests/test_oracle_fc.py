"""Pins of oracle.fc (the unsharded layer).

Pinned against: a brute-force triple loop on tiny inputs, central finite
differences of a scalar loss (fixes operand order / transposes of the two
backward products independently of their formulas), the identity special
case, and the zero-gradient case.
"""
import numpy as np
import pytest

from oracle import fc
import synthdata


@pytest.mark.parametrize("M,K,N", [(1, 1, 1), (3, 5, 7), (8, 16, 4), (17, 9, 32)])
def test_matmul_matches_triple_loop(M, K, N):
    rng = np.random.default_rng(M * 100 + K * 10 + N)
    A = rng.standard_normal((M, K))
    B = rng.standard_normal((K, N))
    np.testing.assert_allclose(fc.fc_forward(A, B), fc.naive_matmul(A, B), rtol=1e-12, atol=1e-12)


def _loss(X, W, G):
    # L = Σ_ij (X W)_ij · G_ij — linear in each of X and W, so a central
    # difference is exact up to rounding.
    return float(np.sum(fc.naive_matmul(X, W) * G))


def test_backward_products_match_finite_differences():
    rng = np.random.default_rng(7)
    m, k, n = 4, 3, 5
    X = rng.standard_normal((m, k))
    W = rng.standard_normal((k, n))
    dO = rng.standard_normal((m, n))   # ∂L/∂O for L = Σ O ⊙ dO
    h = 1e-3
    gX = np.zeros_like(X)
    for a in range(m):
        for b in range(k):
            Xp, Xm = X.copy(), X.copy()
            Xp[a, b] += h
            Xm[a, b] -= h
            gX[a, b] = (_loss(Xp, W, dO) - _loss(Xm, W, dO)) / (2 * h)
    gW = np.zeros_like(W)
    for a in range(k):
        for b in range(n):
            Wp, Wm = W.copy(), W.copy()
            Wp[a, b] += h
            Wm[a, b] -= h
            gW[a, b] = (_loss(X, Wp, dO) - _loss(X, Wm, dO)) / (2 * h)
    np.testing.assert_allclose(fc.fc_backward_input(dO, W), gX, rtol=1e-8, atol=1e-9)
    np.testing.assert_allclose(fc.fc_backward_weight(X, dO), gW, rtol=1e-8, atol=1e-9)


def test_identity_input_returns_weight():
    W = synthdata.tensor((6, 9), 5)
    np.testing.assert_array_equal(fc.fc_forward(np.eye(6), W), W.astype(np.float64))


def test_zero_output_gradient_gives_zero_gradients():
    X, W, _ = synthdata.layer_tensors(8, 6, 10)
    dO = np.zeros((8, 10))
    assert not fc.fc_backward_input(dO, W).any()
    assert not fc.fc_backward_weight(X, dO).any()


def test_integer_inputs_give_exact_integers():
    X, W, dO = synthdata.layer_tensors(64, 48, 80, kind="int")
    O, dI, dW = fc.fc_layer(X, W, dO)
    for R in (O, dI, dW):
        assert np.array_equal(R, np.round(R))
    # exact against the triple loop on a corner
    np.testing.assert_array_equal(O[:4, :6], fc.naive_matmul(X[:4], W[:, :6]))
    np.testing.assert_array_equal(dI[:4, :6], fc.naive_matmul(dO[:4], W[:6].T))
    np.testing.assert_array_equal(dW[:4, :6], fc.naive_matmul(X[:, :4].T, dO[:, :6]))


def test_dot_entries_matches_brute_force():
    rng = np.random.default_rng(3)
    A = rng.standard_normal((13, 11))
    B = rng.standard_normal((11, 17))
    rows = rng.integers(0, 13, 50)
    cols = rng.integers(0, 17, 50)
    full = fc.naive_matmul(A, B)
    np.testing.assert_allclose(fc.dot_entries(A, B, rows, cols), full[rows, cols], rtol=1e-12)


def test_synthdata_bf16_round_is_rne():
    # 1 + 2^-8 is a tie between 1 and 1 + 2^-7 -> even (1.0);
    # 1 + 3·2^-8 ties between 1+2^-7 and 1+2^-6 -> even (1 + 2^-6)
    x = np.array([1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, 1.0 + 2 ** -9, -2.5], dtype=np.float32)
    r = synthdata.bf16_round(x)
    np.testing.assert_array_equal(r, np.array([1.0, 1.0 + 2 ** -6, 1.0, -2.5], dtype=np.float32))
    bits = synthdata.bf16_bits(r)
    np.testing.assert_array_equal(synthdata.bits_to_f32(bits), r)
