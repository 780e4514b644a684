"""Helpers for the -m gpu parity tests: seeded inputs -> device tensors, and the
comparison metrics.  No arithmetic of the method lives here."""
import numpy as np

import synthdata


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("-m gpu tests need a CUDA device (B200)")
    return torch


def to_dev(a32: np.ndarray, dtype, ld=None):
    """float32 array holding bf16 values -> device tensor [rows][cols] with row
    stride `ld` (>= cols), returned as a view of the padded buffer."""
    torch = require_cuda()
    rows, cols = a32.shape
    ld = cols if ld is None else ld
    if dtype == torch.bfloat16:
        bits = synthdata.bf16_bits(a32).view(np.int16)
        host = torch.from_numpy(np.ascontiguousarray(bits)).view(torch.bfloat16)
    else:
        host = torch.from_numpy(np.ascontiguousarray(a32, dtype=np.float32))
    buf = torch.zeros((max(rows, 1), max(ld, 1)), dtype=dtype, device="cuda")
    if rows and cols:
        buf[:rows, :cols].copy_(host.cuda())
    return buf[:rows, :cols]


def empty_dev(rows, cols, dtype, ld=None):
    torch = require_cuda()
    ld = cols if ld is None else ld
    buf = torch.full((max(rows, 1), max(ld, 1)), float("nan"), dtype=dtype, device="cuda")
    return buf[:rows, :cols]


def to_host_f64(t) -> np.ndarray:
    import torch
    return t.detach().float().cpu().numpy().astype(np.float64)


def bf16_bits_of(t) -> np.ndarray:
    import torch
    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def normwise_err(got: np.ndarray, ref: np.ndarray) -> float:
    """max|got - ref| / max|ref|."""
    den = np.max(np.abs(ref)) if ref.size else 0.0
    if den == 0.0:
        return float(np.max(np.abs(got))) if got.size else 0.0
    return float(np.max(np.abs(got - ref)) / den)


def round_up(x, a=8):
    return (x + a - 1) // a * a
