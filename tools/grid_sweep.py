#!/usr/bin/env python
"""Case-1 bandwidth database and performance-model validation on one box.

Run under torchrun, one process per GPU:

    python -m torch.distributed.run --nproc-per-node G tools/grid_sweep.py \
        --model 20B --tokens 16384 --steps 20 --out gpurun_out/sweep_G.json

1. Case-1 database: for every (G0, G1) with G0*G1 <= G,
   all G/G1 groups of size G1 whose members are G0 ranks apart all-reduce
   1 GiB simultaneously; beta = per-rank ring bytes 2(G1-1)/G1 * S / time
   (the quantity Eqs. 1-5 divide by).  Reading R13.
2. Every feasible grid (Gx, Gy, Gz, Gd) of G is timed on the GPT block (Alg. 1
   fwd+bwd of its 4 FC layers through libaxonn) and compared with the model's
   ranking under uniform beta and under the measured table (Spearman rank
   correlation and top-k overlap, cf. Fig. 2).
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
from bench import HIDDEN, block_layers, model_flops  # noqa: E402


def measure_beta(rank, world, nbytes, iters=5):
    table = {}
    for g0 in range(1, world + 1):
        for g1 in range(2, world + 1):
            if g0 * g1 > world or world % (g0 * g1):
                continue
            # groups: ranks r with the same (r mod g0, r // (g0*g1)), members g0 apart
            groups = {}
            for r in range(world):
                key = (r % g0, r // (g0 * g1))
                groups.setdefault(key, []).append(r)
            pgs = {k: dist.new_group(v) for k, v in sorted(groups.items())}
            mine = [k for k, v in groups.items() if rank in v][0]
            t = torch.empty(nbytes // 2, dtype=torch.bfloat16, device="cuda").fill_(1.0)
            for _ in range(2):
                dist.all_reduce(t, group=pgs[mine])
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(iters):
                dist.all_reduce(t, group=pgs[mine])
            e1.record()
            torch.cuda.synchronize()
            ms = torch.tensor([e0.elapsed_time(e1) / iters], device="cuda", dtype=torch.float64)
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
            sec = float(ms.item()) / 1e3
            table[(g0, g1)] = 2 * (g1 - 1) / g1 * nbytes / sec
            del t
            for pg in pgs.values():
                dist.destroy_process_group(pg)
    return table


def time_grid(cfg, layers, steps, warmup, chunks):
    ax.axonn_grid_init(*cfg)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(42 + dist.get_rank())
    bf = torch.bfloat16

    def rnd(*shape):
        x = torch.empty(shape, dtype=torch.float32, device="cuda")
        x.uniform_(-1, 1, generator=gen)
        return x.to(bf)

    L = []
    for (m, k, n, t) in layers:
        h = ax.axonn_fc_create(m, k, n, t, ax.AXONN_BF16, chunks)
        g = ax.axonn_fc_geometry(h)
        L.append({"h": h, "I": rnd(g.m_l, g.k_l), "W": rnd(g.what_len),
                  "O": torch.empty(g.m_l, g.n_l, dtype=bf, device="cuda"), "dO": rnd(g.m_l, g.n_l),
                  "dI": torch.empty(g.m_l, g.k_l, dtype=bf, device="cuda"),
                  "dW": torch.empty(g.what_len, dtype=bf, device="cuda")})
    s = torch.cuda.Stream()

    def step():
        for i, l in enumerate(L):
            if i + 1 < len(L):  # OAG: next layer's gather beside this layer's GEMM
                ax.axonn_fc_prefetch(L[i + 1]["h"], L[i + 1]["W"], s)
            ax.axonn_fc_forward(l["h"], l["I"], l["W"], l["O"], s)
        for l in reversed(L):
            ax.axonn_fc_backward(l["h"], l["dO"], l["dI"], l["dW"], s)
        ax.axonn_grads_sync(s)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(steps):
        step()
    e1.record(s)
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1) / steps], device="cuda", dtype=torch.float64)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    for l in L:
        ax.axonn_fc_destroy(l["h"])
    ax.axonn_grid_finalize()
    del L
    torch.cuda.empty_cache()
    return float(ms.item())


def tie_ranks(v, rel=1e-12):
    """Average ranks (1-based), values equal within `rel` (R12's tolerance) tied."""
    import numpy as np
    v = np.asarray(v, dtype=np.float64)
    order = np.argsort(v, kind="stable")
    ranks = np.empty(len(v))
    i = 0
    while i < len(v):
        j = i
        while j + 1 < len(v) and abs(v[order[j + 1]] - v[order[i]]) <= rel * max(abs(v[order[i]]), 1e-300):
            j += 1
        ranks[order[i:j + 1]] = (i + j) / 2.0 + 1.0
        i = j + 1
    return ranks


def spearman(a, b):
    """Spearman's rho with average ranks for ties (the model's exact Z-vs-DP
    ties, R12, are not ordered arbitrarily)."""
    import numpy as np
    ra, rb = tie_ranks(a), tie_ranks(b)
    if np.std(ra) == 0 or np.std(rb) == 0:
        return float("nan")
    return float(np.corrcoef(ra, rb)[0, 1])


def kendall_tau_b(a, b, rel=1e-12):
    """Kendall's tau-b (tie-corrected) between predicted and measured orders."""
    import math
    n = len(a)
    conc = disc = ta = tb = 0
    for i in range(n):
        for j in range(i + 1, n):
            da = 0 if abs(a[i] - a[j]) <= rel * max(abs(a[i]), abs(a[j]), 1e-300) else (1 if a[i] > a[j] else -1)
            db = 0 if abs(b[i] - b[j]) <= rel * max(abs(b[i]), abs(b[j]), 1e-300) else (1 if b[i] > b[j] else -1)
            if da == 0 and db == 0:
                continue
            if da == 0:
                ta += 1
            elif db == 0:
                tb += 1
            elif da == db:
                conc += 1
            else:
                disc += 1
    den = math.sqrt((conc + disc + ta) * (conc + disc + tb))
    return (conc - disc) / den if den else float("nan")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="20B", choices=sorted(HIDDEN))
    ap.add_argument("--tokens", type=int, default=16384)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--chunks", type=int, default=4)
    ap.add_argument("--beta-bytes", type=int, default=1 << 30)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ax.bootstrap_from_torch_distributed(local)

    table = measure_beta(rank, world, args.beta_bytes)
    layers = block_layers(HIDDEN[args.model], args.tokens)
    flops = model_flops(layers)
    uni = {k: 1e11 for k in table} if table else {}
    rank_uni = ax.axonn_grid_select(layers, world, world, uni or {(1, 2): 1e11}, 1e11)
    rank_meas = ax.axonn_grid_select(layers, world, world, table or {(1, 2): 1e11}, 1e11)
    meas = {}
    for r in rank_uni:
        cfg = (r["gx"], r["gy"], r["gz"], r["gd"])
        meas[cfg] = time_grid(cfg, layers, args.steps, args.warmup, args.chunks)
        if rank == 0:
            print(f"grid {cfg}: {meas[cfg]:.3f} ms/step, {flops / meas[cfg] / 1e9 / world:.1f} TF/s/GPU",
                  file=sys.stderr, flush=True)
    if rank == 0:
        cfgs = list(meas)
        t = [meas[c] for c in cfgs]
        pu = [next(r["t_comm"] for r in rank_uni if (r["gx"], r["gy"], r["gz"], r["gd"]) == c) for c in cfgs]
        pm = [next(r["t_comm"] for r in rank_meas if (r["gx"], r["gy"], r["gz"], r["gd"]) == c) for c in cfgs]
        k = min(3, len(cfgs))
        fastest = set(sorted(cfgs, key=lambda c: meas[c])[:k])
        top_u = {(r["gx"], r["gy"], r["gz"], r["gd"]) for r in rank_uni[:k]}
        top_m = {(r["gx"], r["gy"], r["gz"], r["gd"]) for r in rank_meas[:k]}
        out = {"G": world, "model": args.model, "tokens": args.tokens,
               "beta_table_GBps": {f"{a},{b}": v / 1e9 for (a, b), v in table.items()},
               "grids": [{"grid": list(c), "ms_per_step": meas[c],
                          "tflops_per_gpu": flops / meas[c] / 1e9 / world,
                          "model_t_comm_uniform": u, "model_t_comm_measured_beta": p}
                         for c, u, p in zip(cfgs, pu, pm)],
               "spearman_uniform": spearman(pu, t), "spearman_measured_beta": spearman(pm, t),
               "kendall_tau_b_uniform": kendall_tau_b(pu, t),
               "kendall_tau_b_measured_beta": kendall_tau_b(pm, t),
               f"top{k}_hits_uniform": len(top_u & fastest),
               f"top{k}_hits_measured_beta": len(top_m & fastest)}
        s = json.dumps(out, indent=1)
        print(s)
        if args.out:
            open(args.out, "w").write(s)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
