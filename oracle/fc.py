"""Unsharded FC layer in fp64 — the plain definition the 3D PMM must reproduce.

PAPER.md:329-337 (§IV-A, "3D Parallel Matrix Multiplication"): "Each FC layer
computes one half-precision ... matrix multiplication (input activation, I
multiplied by the layer's weight matrix, W) in the forward pass and two
half-precision matrix multiplications (MMs) in the backward pass
(∂L/∂O × Wᵀ and Iᵀ × ∂L/∂O ...)".

The oracle evaluates these three products in fp64 on the bf16-valued inputs
(converted exactly).  The library primitive ``numpy.matmul`` is a step; there
is no blocking or reordering beyond it.  ``naive_matmul`` is the triple loop
used only to pin ``numpy.matmul`` on tiny inputs.
"""
from __future__ import annotations

import numpy as np


def _f64(a) -> np.ndarray:
    return np.asarray(a, dtype=np.float64)


def fc_forward(I, W) -> np.ndarray:
    """O = I × W  (Alg. 1 line 3 at grid 1×1×1)."""
    return _f64(I) @ _f64(W)


def fc_backward_input(dO, W) -> np.ndarray:
    """∂L/∂I = ∂L/∂O × Wᵀ  (Alg. 1 line 11 at grid 1×1×1)."""
    return _f64(dO) @ _f64(W).T


def fc_backward_weight(I, dO) -> np.ndarray:
    """∂L/∂W = Iᵀ × ∂L/∂O  (Alg. 1 line 13 at grid 1×1×1)."""
    return _f64(I).T @ _f64(dO)


def fc_layer(I, W, dO):
    """All three products of one FC layer step: (O, dI, dW)."""
    return fc_forward(I, W), fc_backward_input(dO, W), fc_backward_weight(I, dO)


def dot_entries(A, B, rows, cols) -> np.ndarray:
    """(A @ B)[rows[t], cols[t]] for sampled t, each an exact fp64 dot product.

    Used for parity at full size where the whole product is too slow on the
    CPU (SURVEY.md §8(d) "sampled entries ... each an exact fp64 dot
    product").  A is [M,K], B is [K,N].
    """
    A = _f64(A)
    B = _f64(B)
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    return np.einsum("tk,kt->t", A[rows, :], B[:, cols])


def naive_matmul(A, B) -> np.ndarray:
    """Triple loop C[i,j] = Σ_p A[i,p]·B[p,j] — brute force for tiny pins only."""
    A = _f64(A)
    B = _f64(B)
    M, K = A.shape
    K2, N = B.shape
    if K != K2:
        raise ValueError("inner dimensions differ")
    C = np.zeros((M, N), dtype=np.float64)
    for i in range(M):
        for j in range(N):
            s = 0.0
            for p in range(K):
                s += A[i, p] * B[p, j]
            C[i, j] = s
    return C
