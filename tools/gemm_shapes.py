#!/usr/bin/env python
"""Per-launch timing of the 12 local products of one C2 step (GPT-5B block,
m = 16384, grid 1x1x1x1), libaxonn vs torch.matmul (cuBLAS) on the same
operands, alternating, each in its own short (burst-clock) window.

    python tools/gemm_shapes.py [--reps 10] [--rounds 3] [--no-cublas] [--label NAME]

Prints one JSON line: per shape the best-of-rounds TF/s of each side and the
sum of per-shape times (the step's GEMM time at the measured rates).  The
library reads its AXONN_* switches once per process, so A/B of kernel
configurations runs this script once per setting (tools/ab_gemm.sh).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2502_08145_b200 as ax  # noqa: E402

H, M = 4096, 16384
# (name, op, M, N, K): fwd NN (m x k x n), dI NT (m x n x k... M=m, N=k, K=n), dW TN (M=k, N=n, K=m)
LAYERS = [("qkv", H, 3 * H), ("proj", H, H), ("fc1", H, 4 * H), ("fc2", 4 * H, H)]


def shapes():
    out = []
    for name, k, n in LAYERS:
        out.append((f"{name}_fwd", 0, M, n, k))
        out.append((f"{name}_dI", 1, M, k, n))
        out.append((f"{name}_dW", 2, k, n, M))
    return out


def operands(op, Mm, Nn, Kk, dev):
    bf = torch.bfloat16
    a_shape = (Kk, Mm) if op == 2 else (Mm, Kk)
    b_shape = (Nn, Kk) if op == 1 else (Kk, Nn)
    A = torch.empty(a_shape, dtype=bf, device=dev).uniform_(-1, 1)
    B = torch.empty(b_shape, dtype=bf, device=dev).uniform_(-1, 1)
    C = torch.empty(Mm, Nn, dtype=bf, device=dev)
    return A, B, C


def time_it(fn, reps, s, warm=True):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if warm:
        fn()
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--no-cublas", action="store_true")
    ap.add_argument("--label", default=os.environ.get("AB_LABEL", "default"))
    ap.add_argument("--only", default=None, help="comma-separated shape names")
    ap.add_argument("--no-warm", action="store_true", help="no warm-up launch (ncu captures)")
    args = ap.parse_args()
    dev = "cuda"
    torch.cuda.set_device(0)
    s = torch.cuda.current_stream()
    res = {}
    sel = set(args.only.split(",")) if args.only else None
    for name, op, Mm, Nn, Kk in shapes():
        if sel and name not in sel:
            continue
        A, B, C = operands(op, Mm, Nn, Kk, dev)
        lda, ldb = A.stride(0), B.stride(0)

        def ours():
            ax.axonn_gemm(op, ax.AXONN_BF16, Mm, Nn, Kk, A, lda, B, ldb, C, Nn, s)

        if op == 0:
            def cub():
                torch.matmul(A, B, out=C)
        elif op == 1:
            def cub():
                torch.matmul(A, B.t(), out=C)
        else:
            def cub():
                torch.matmul(A.t(), B, out=C)
        t_ax, t_cb = [], []
        for _ in range(args.rounds):
            t_ax.append(time_it(ours, args.reps, s, not args.no_warm))
            if not args.no_cublas:
                t_cb.append(time_it(cub, args.reps, s))
        fl = 2.0 * Mm * Nn * Kk
        res[name] = {"shape": [op, Mm, Nn, Kk], "axonn_ms": min(t_ax),
                     "axonn_tflops": fl / min(t_ax) / 1e9}
        if t_cb:
            res[name].update({"cublas_ms": min(t_cb), "cublas_tflops": fl / min(t_cb) / 1e9})
        del A, B, C
    tot_ax = sum(r["axonn_ms"] for r in res.values())
    line = {"label": args.label, "reps": args.reps, "rounds": args.rounds,
            "sum_axonn_ms": tot_ax, "shapes": res}
    if not args.no_cublas:
        line["sum_cublas_ms"] = sum(r["cublas_ms"] for r in res.values())
    print(json.dumps(line))


if __name__ == "__main__":
    main()
