#!/usr/bin/env python
"""Same-box comparison of the C2 step's 12 local products: libaxonn's tcgen05
kernel vs cuBLAS (torch.matmul on the same operand layouts, as views).

Both are timed the same way (CUDA events around K back-to-back steps, several
seconds so both run at the power-capped sustained clock), alternating
A-B-A-B on one GPU.  cuBLAS here is a reference point, not part of the product.

    python tools/cublas_compare.py [--seconds 4] [--rounds 2]
"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2502_08145_b200 as ax  # noqa: E402
from bench import block_layers, model_flops  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=4.0)
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--once", action="store_true", help="1 warm-up + 1 step of each (for ncu)")
    ap.add_argument("--cool", type=float, default=0.0,
                    help="idle seconds before each timed window (short windows then start from "
                         "a rested power state, as a fresh bench run does)")
    ap.add_argument("--per-op", action="store_true",
                    help="also time each of the 12 products separately (CUDA events per launch)")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    bf = torch.bfloat16
    layers = block_layers(args.hidden, 16384)
    T = []
    for (m, k, n, _) in layers:
        T.append({"I": torch.empty(m, k, dtype=bf, device="cuda").uniform_(-1, 1),
                  "W": torch.empty(k, n, dtype=bf, device="cuda").uniform_(-1, 1),
                  "dO": torch.empty(m, n, dtype=bf, device="cuda").uniform_(-1, 1),
                  "O": torch.empty(m, n, dtype=bf, device="cuda"),
                  "dI": torch.empty(m, k, dtype=bf, device="cuda"),
                  "dW": torch.empty(k, n, dtype=bf, device="cuda"), "mkn": (m, k, n)})
    s = torch.cuda.Stream()

    def step_axonn():
        for t in T:
            m, k, n = t["mkn"]
            ax.axonn_gemm(0, 0, m, n, k, t["I"], k, t["W"], n, t["O"], n, s)
        for t in reversed(T):
            m, k, n = t["mkn"]
            ax.axonn_gemm(1, 0, m, k, n, t["dO"], n, t["W"], n, t["dI"], k, s)
            ax.axonn_gemm(2, 0, k, n, m, t["I"], k, t["dO"], n, t["dW"], n, s)

    def step_cublas():
        with torch.cuda.stream(s):
            for t in T:
                torch.matmul(t["I"], t["W"], out=t["O"])
            for t in reversed(T):
                torch.matmul(t["dO"], t["W"].t(), out=t["dI"])
                torch.matmul(t["I"].t(), t["dO"], out=t["dW"])

    flops = model_flops(layers)

    def ops_axonn():
        out = []
        for t in T:
            m, k, n = t["mkn"]
            out.append((f"fwd NN {m}x{n}x{k}", 2 * m * n * k,
                        lambda t=t, m=m, k=k, n=n: ax.axonn_gemm(0, 0, m, n, k, t["I"], k, t["W"], n, t["O"], n, s)))
        for t in reversed(T):
            m, k, n = t["mkn"]
            out.append((f"dI NT {m}x{k}x{n}", 2 * m * n * k,
                        lambda t=t, m=m, k=k, n=n: ax.axonn_gemm(1, 0, m, k, n, t["dO"], n, t["W"], n, t["dI"], k, s)))
            out.append((f"dW TN {k}x{n}x{m}", 2 * m * n * k,
                        lambda t=t, m=m, k=k, n=n: ax.axonn_gemm(2, 0, k, n, m, t["I"], k, t["dO"], n, t["dW"], n, s)))
        return out

    def ops_cublas():
        out = []
        for t in T:
            m, k, n = t["mkn"]
            out.append((f"fwd NN {m}x{n}x{k}", 2 * m * n * k,
                        lambda t=t: torch.matmul(t["I"], t["W"], out=t["O"])))
        for t in reversed(T):
            m, k, n = t["mkn"]
            out.append((f"dI NT {m}x{k}x{n}", 2 * m * n * k,
                        lambda t=t: torch.matmul(t["dO"], t["W"].t(), out=t["dI"])))
            out.append((f"dW TN {k}x{n}x{m}", 2 * m * n * k,
                        lambda t=t: torch.matmul(t["I"].t(), t["dO"], out=t["dW"])))
        return out

    def per_op(ops, steps):
        evs = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                for _ in ops] for _ in range(steps)]
        with torch.cuda.stream(s):
            for st in range(steps):
                for (name, fl, fn), (a, b) in zip(ops, evs[st]):
                    a.record(s)
                    fn()
                    b.record(s)
        torch.cuda.synchronize()
        return [(name, fl / (sum(evs[st][i][0].elapsed_time(evs[st][i][1]) for st in range(steps)) / steps * 1e-3) / 1e12)
                for i, (name, fl, _) in enumerate(ops)]

    def timed(fn):
        import time as _t
        if args.cool > 0:
            torch.cuda.synchronize()
            _t.sleep(args.cool)
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn()
        e1.record(s)
        torch.cuda.synchronize()
        per = e0.elapsed_time(e1)
        k = max(5, int(args.seconds * 1e3 / per))
        e0.record(s)
        for _ in range(k):
            fn()
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / k
        return flops / (ms * 1e-3) / 1e12, ms, k

    if args.once:
        for fn in (step_axonn, step_cublas, step_axonn, step_cublas):
            fn()
        torch.cuda.synchronize()
        return
    res = {"axonn": [], "cublas": []}
    for r in range(args.rounds):
        for name, fn in (("axonn", step_axonn), ("cublas", step_cublas)):
            tf, ms, k = timed(fn)
            res[name].append(tf)
            print(f"round {r} {name:7s}: {tf:8.1f} TFLOP/s  {ms:.3f} ms/step  ({k} steps)", flush=True)
    a = max(res["axonn"])
    c = max(res["cublas"])
    print(f"best: axonn {a:.1f} TFLOP/s, cublas {c:.1f} TFLOP/s, ratio {a / c:.3f}")
    if args.per_op:
        import time as _t
        for name, ops in (("axonn", ops_axonn()), ("cublas", ops_cublas())):
            torch.cuda.synchronize()
            if args.cool > 0:
                _t.sleep(args.cool)
            for _, _, fn in ops:
                fn()
            r = per_op(ops, 3)
            for op, tf in r:
                print(f"per-op {name:7s} {op:28s} {tf:8.1f} TFLOP/s", flush=True)


if __name__ == "__main__":
    main()
