#!/usr/bin/env python
"""Where the time of one fused Alg. 1 layer goes, per phase, under torchrun:

    python -m torch.distributed.run --nproc-per-node 4 tools/layer_phases.py \
        --model 20B --tokens 8192 --grid 2,2,1,1 [--phase A] [--out FILE]

For each FC layer of the GPT block, with the ranks aligned before every call
(barrier + synchronize, so no skew carries between calls), reports the max
over ranks of:
  fwd_ms        axonn_fc_forward (lines 2-4) on the stream, CUDA events;
  fwd_gemm_ms   the GEMM inside it (the library's own events: epilogue incl.
                its NVLink traffic);
  gemm_alone_ms the same local product through axonn_gemm (plain stores);
  bwd_ms / bwd_gemm_ms / bwd_alone_ms  the same for axonn_fc_backward
                (lines 11-14) + grads_sync.
fwd_ms - fwd_gemm_ms is what follows the GEMM (barriers, owner phase / local
sum, completion waits); fwd_gemm_ms - gemm_alone_ms is the epilogue's cost.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2502_08145_b200 as ax  # noqa: E402
from bench import HIDDEN, block_layers  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="20B", choices=sorted(HIDDEN))
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--grid", default="2,2,1,1")
    ap.add_argument("--phase", default="A")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank = dist.get_rank()
    ax.bootstrap_from_torch_distributed(local)
    cfg = [int(x) for x in args.grid.split(",")]
    ax.axonn_grid_init(*cfg)
    bf = torch.bfloat16
    s = torch.cuda.Stream()
    names = ["qkv", "proj", "fc1", "fc2"]
    res = []

    def tmax(x):
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(fn, prof=False):
        """mean ms of fn on s over iters, ranks aligned before each call; with
        prof, also the library's GEMM ms inside it."""
        tot = 0.0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        gm = 0.0
        for _ in range(args.iters):
            dist.barrier()
            torch.cuda.synchronize()
            if prof:
                ax.axonn_profile_read()
                ax.axonn_profile_enable(True)
            e0.record(s)
            fn()
            e1.record(s)
            torch.cuda.synchronize()
            if prof:
                ax.axonn_profile_enable(False)
                gm += ax.axonn_profile_read()[1]
            tot += e0.elapsed_time(e1)
        return tot / args.iters, gm / args.iters

    for name, (m, k, n, t) in zip(names, block_layers(HIDDEN[args.model], args.tokens, args.phase)):
        h = ax.axonn_fc_create(m, k, n, t, ax.AXONN_BF16)
        g = ax.axonn_fc_geometry(h)
        a = (3.0 / k) ** 0.5
        I = torch.empty(g.m_l, g.k_l, dtype=bf, device="cuda").uniform_(-1, 1)
        W = torch.empty(g.what_len, dtype=bf, device="cuda").uniform_(-a, a)
        dO = torch.empty(g.m_l, g.n_l, dtype=bf, device="cuda").uniform_(-1, 1)
        Wf = torch.empty(g.k_l, g.n_l, dtype=bf, device="cuda").uniform_(-a, a)
        outs = []
        for which, shape in ((0, (g.m_l, g.n_l)), (1, (g.m_l, g.k_l)), (2, (g.what_len,))):
            p = ax.axonn_fc_output_buffer(h, which)
            outs.append(p if p else torch.empty(shape, dtype=bf, device="cuda"))
        O2 = torch.empty(g.m_l, g.n_l, dtype=bf, device="cuda")
        dI2 = torch.empty(g.m_l, g.k_l, dtype=bf, device="cuda")
        dW2 = torch.empty(g.k_l, g.n_l, dtype=bf, device="cuda")

        def fwd():
            ax.axonn_fc_forward(h, I, W, outs[0], s)

        def bwd():
            ax.axonn_fc_backward(h, dO, outs[1], outs[2], s)
            ax.axonn_grads_sync(s)

        def fwd_alone():
            ax.axonn_gemm(0, 0, g.m_l, g.n_l, g.k_l, I, g.k_l, Wf, g.n_l, O2, g.n_l, s)

        def bwd_alone():
            ax.axonn_gemm(1, 0, g.m_l, g.k_l, g.n_l, dO, g.n_l, Wf, g.n_l, dI2, g.k_l, s)
            ax.axonn_gemm(2, 0, g.k_l, g.n_l, g.m_l, I, g.k_l, dO, g.n_l, dW2, g.n_l, s)

        with torch.cuda.stream(s):
            for _ in range(3):
                fwd()
                bwd()
                fwd_alone()
                bwd_alone()
            torch.cuda.synchronize()
            f_ms, f_g = timed(fwd, True)
            fa, _ = timed(fwd_alone)
            b_tot = 0.0
            bg = 0.0
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for _ in range(args.iters):
                fwd()
                dist.barrier()
                torch.cuda.synchronize()
                ax.axonn_profile_read()
                ax.axonn_profile_enable(True)
                e0.record(s)
                bwd()
                e1.record(s)
                torch.cuda.synchronize()
                ax.axonn_profile_enable(False)
                bg += ax.axonn_profile_read()[1]
                b_tot += e0.elapsed_time(e1)
            b_ms, b_g = b_tot / args.iters, bg / args.iters
            ba, _ = timed(bwd_alone)
        rec = {"layer": name, "grid": cfg, "m": m, "k": k, "n": n, "transposed": t,
               "local_gemm": [g.m_l, g.k_l, g.n_l],
               "fwd_ms": tmax(f_ms), "fwd_gemm_ms": tmax(f_g), "gemm_alone_ms": tmax(fa),
               "bwd_ms": tmax(b_ms), "bwd_gemm_ms": tmax(b_g), "bwd_alone_ms": tmax(ba),
               "fused": {a_: ax.axonn_fused_status(a_) for a_ in "xyzd"}}
        if rank == 0:
            print(json.dumps(rec), flush=True)
            res.append(rec)
        ax.axonn_fc_destroy(h)
        del I, W, dO, Wf, outs, O2, dI2, dW2
    if rank == 0 and args.out:
        json.dump(res, open(args.out, "w"), indent=1)
    ax.axonn_grid_finalize()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
