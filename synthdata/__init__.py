"""Seeded synthetic inputs shared by the CPU oracle and the CUDA path.

This module holds NO arithmetic of the method (no matmul, no collective, no
shard geometry).  It only draws numbers and encodes them as bf16, so that the
oracle (``oracle/``) and the GPU path (``paper_2502_08145_b200``) can be fed
bit-identical inputs without sharing any code that computes a result.

Recipe:
  * every global tensor is drawn from numpy's PCG64 seeded with
    ``(seed, tensor_id)`` — independent streams per tensor;
  * ``kind="uniform"``: U(-1, 1) ("seeded uniform(-1,1)"), then
    rounded round-to-nearest-even to bf16 — the paper trains in bf16
    (PAPER.md:724-728);
  * ``kind="int"``: integers in [-4, 4]; every product and partial sum of the
    three FC products is then an exact integer < 2^24 (SURVEY.md §8(c) pins);
  * base seed 42.
"""
from __future__ import annotations

import numpy as np

BASE_SEED = 42

# Stable tensor ids per role, so that "X of layer 2" is the same array
# wherever it is generated.
TENSOR_IDS = {"X": 1, "W": 2, "dY": 3}


def _rng(seed: int, tensor_id: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64([int(seed), int(tensor_id)]))


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round float32/float64 values to the nearest bf16 (ties to even).

    Returns float32 holding exactly representable bf16 values.  Inputs are
    finite (generator output), so NaN/Inf handling is not needed.
    """
    f = np.ascontiguousarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    r = ((u + np.uint64(0x7FFF) + lsb) & np.uint64(0xFFFF0000)).astype(np.uint32)
    return r.view(np.float32).reshape(f.shape)


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """bf16 bit patterns (uint16) of values already representable in bf16."""
    f = np.ascontiguousarray(x, dtype=np.float32)
    return (f.view(np.uint32) >> np.uint32(16)).astype(np.uint16).reshape(f.shape)


def bits_to_f32(bits: np.ndarray) -> np.ndarray:
    """Inverse of :func:`bf16_bits`: uint16 bf16 patterns -> float32 values."""
    b = np.ascontiguousarray(bits, dtype=np.uint16)
    return (b.astype(np.uint32) << np.uint32(16)).view(np.float32).reshape(b.shape)


def tensor(shape, tensor_id: int, seed: int = BASE_SEED, kind: str = "uniform") -> np.ndarray:
    """A seeded global tensor as float32 holding bf16-representable values."""
    rng = _rng(seed, tensor_id)
    shape = tuple(int(s) for s in shape)
    if kind == "uniform":
        return bf16_round(rng.uniform(-1.0, 1.0, size=shape).astype(np.float32))
    if kind == "int":
        return rng.integers(-4, 5, size=shape).astype(np.float32)
    raise ValueError(f"unknown kind {kind!r}")


def layer_tensors(m: int, k: int, n: int, layer_id: int = 0, seed: int = BASE_SEED,
                  kind: str = "uniform"):
    """Global X [m,k], W [k,n], dY [m,n] of one FC layer (float32, bf16 values)."""
    base = 16 * int(layer_id)
    X = tensor((m, k), base + TENSOR_IDS["X"], seed, kind)
    W = tensor((k, n), base + TENSOR_IDS["W"], seed, kind)
    dY = tensor((m, n), base + TENSOR_IDS["dY"], seed, kind)
    return X, W, dY
