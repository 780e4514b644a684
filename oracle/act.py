"""GeLU between fc1 and fc2 of a GPT block — test oracle (plain fp64).

The paper trains GPT-style transformers (citing GPT-3),
whose MLP is fc1 (h -> 4h), GeLU, fc2 (4h -> h).  The paper never spells the
activation out; reading R18: the exact GeLU of Hendrycks & Gimpel,

    GELU(x)  = x · Φ(x),          Φ(x) = (1 + erf(x / √2)) / 2,
    GELU'(x) = Φ(x) + x · φ(x),   φ(x) = exp(-x² / 2) / √(2π),

evaluated elementwise in fp64 (``math.erf`` / ``math.exp`` as the library
steps).  ``mlp`` composes it with the two FC products of oracle.fc in the
order the block runs them (forward fc1, GeLU, fc2; backward fc2, dGeLU, fc1).

Test infrastructure: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline leg may import this package.
"""
from __future__ import annotations

import math

import numpy as np

from . import fc

_erf = np.vectorize(math.erf, otypes=[np.float64])
_exp = np.vectorize(math.exp, otypes=[np.float64])


def Phi(x) -> np.ndarray:
    """Standard normal CDF, (1 + erf(x/√2)) / 2."""
    return 0.5 * (1.0 + _erf(np.asarray(x, dtype=np.float64) / math.sqrt(2.0)))


def phi(x) -> np.ndarray:
    """Standard normal density."""
    x = np.asarray(x, dtype=np.float64)
    return _exp(-0.5 * x * x) / math.sqrt(2.0 * math.pi)


def gelu(x) -> np.ndarray:
    """GELU(x) = x Φ(x)."""
    x = np.asarray(x, dtype=np.float64)
    return x * Phi(x)


def gelu_grad(x) -> np.ndarray:
    """d GELU / dx = Φ(x) + x φ(x)."""
    x = np.asarray(x, dtype=np.float64)
    return Phi(x) + x * phi(x)


def mlp(X, W1, W2, dY):
    """fc1 -> GeLU -> fc2, forward and backward, unsharded, fp64.

    Returns dict: Z (fc1 output, pre-activation), A = GELU(Z) (fc2 input),
    O = A W2, dA = dY W2ᵀ (fc2's dI), dW2 = Aᵀ dY, dZ = dA ⊙ GELU'(Z)
    (fc1's dO), dX = dZ W1ᵀ, dW1 = Xᵀ dZ.
    """
    Z = fc.fc_forward(X, W1)
    A = gelu(Z)
    O = fc.fc_forward(A, W2)
    dA = fc.fc_backward_input(dY, W2)
    dW2 = fc.fc_backward_weight(A, dY)
    dZ = dA * gelu_grad(Z)
    dX = fc.fc_backward_input(dZ, W1)
    dW1 = fc.fc_backward_weight(X, dZ)
    return {"Z": Z, "A": A, "O": O, "dA": dA, "dW2": dW2, "dZ": dZ, "dX": dX, "dW1": dW1}
