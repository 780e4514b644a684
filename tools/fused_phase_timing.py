#!/usr/bin/env python
"""Time one layer's fused forward (GEMM + epilogue collective + owner phase)
against its GEMM alone, on a given grid.  Run under torchrun:

    python -m torch.distributed.run --nproc-per-node 2 tools/fused_phase_timing.py \
        --tokens 65536 --kin 7168 --nout 7168 --transposed --grid 2,1,1,1

Prints, per rank 0: mean forward ms (CUDA events around axonn_fc_forward), the
mean GEMM ms inside it (the library's own profiling events), and the rest
(barriers + owner phase + waits on the peer).
"""
import argparse
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2502_08145_b200 as ax  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=65536)
    ap.add_argument("--kin", type=int, default=7168)
    ap.add_argument("--nout", type=int, default=7168)
    ap.add_argument("--transposed", action="store_true")
    ap.add_argument("--grid", default="2,1,1,1")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--backward", action="store_true", help="time backward instead")
    args = ap.parse_args()
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ax.bootstrap_from_torch_distributed(local)
    ax.axonn_grid_init(*[int(x) for x in args.grid.split(",")])
    h = ax.axonn_fc_create(args.tokens, args.kin, args.nout, args.transposed, ax.AXONN_BF16)
    g = ax.axonn_fc_geometry(h)
    bf = torch.bfloat16
    I = torch.empty(g.m_l, g.k_l, dtype=bf, device="cuda").uniform_(-1, 1)
    W = torch.empty(g.what_len, dtype=bf, device="cuda").uniform_(-0.02, 0.02)
    dO = torch.empty(g.m_l, g.n_l, dtype=bf, device="cuda").uniform_(-1, 1)
    outs = []
    for which, shape in ((0, (g.m_l, g.n_l)), (1, (g.m_l, g.k_l)), (2, (g.what_len,))):
        p = ax.axonn_fc_output_buffer(h, which)
        outs.append(p if p else torch.empty(shape, dtype=bf, device="cuda"))
    s = torch.cuda.Stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def one():
        ax.axonn_fc_forward(h, I, W, outs[0], s)
        if args.backward:
            ax.axonn_fc_backward(h, dO, outs[1], outs[2], s)
            ax.axonn_grads_sync(s)

    with torch.cuda.stream(s):
        for _ in range(3):
            one()
    torch.cuda.synchronize()
    tot = 0.0
    ax.axonn_profile_read()
    ax.axonn_profile_enable(True)
    for _ in range(args.iters):
        dist.barrier()
        torch.cuda.synchronize()
        if args.backward:
            ax.axonn_fc_forward(h, I, W, outs[0], s)
        e0.record(s)
        if args.backward:
            ax.axonn_fc_backward(h, dO, outs[1], outs[2], s)
            ax.axonn_grads_sync(s)
        else:
            ax.axonn_fc_forward(h, I, W, outs[0], s)
        e1.record(s)
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    ax.axonn_profile_enable(False)
    n, gemm_ms, _ = ax.axonn_profile_read()
    per_call = 2 if args.backward else 1
    gemm = gemm_ms / args.iters * (per_call / (per_call + (1 if args.backward else 0)))
    if args.backward:  # the profile also holds the untimed forwards' GEMMs
        gemm = None
    t = tot / args.iters
    if dist.get_rank() == 0:
        print(f"grid {args.grid} m={args.tokens} k={args.kin} n={args.nout} T={args.transposed} "
              f"{'bwd' if args.backward else 'fwd'}: {t:.3f} ms per call, gemm {gemm_ms / args.iters:.3f} ms "
              f"({n // args.iters} gemm launches/iter), rest {t - gemm_ms / args.iters:.3f} ms; "
              f"fused: {ax.axonn_fused_status('x')}", flush=True)
    ax.axonn_fc_destroy(h)
    ax.axonn_grid_finalize()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
