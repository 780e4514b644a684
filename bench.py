#!/usr/bin/env python
"""Benchmark of the 3D-PMM FC hot path (AxoNN, arXiv 2502.08145) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                    [--grid gx,gy,gz,gd] [--model 5B|10B|20B|40B|80B] [--tokens-per-gpu T]

A "step" is one pass of the whole hot path over one batch: Alg. 1 forward of
the four FC layers of one GPT block (QKV h->3h, proj h->h, fc1 h->4h, fc2
4h->h; Table II shapes; proj and fc2 transposed,
PAPER.md:402-414), then their backward in reverse order, then the ORS /
data-parallel wait point (axonn_grads_sync).

N = 1: BASELINE.json configs[1] (C2): GPT-5B block, m = 16,384 tokens, grid
1x1x1x1.  N > 1: the same block weak-scaled (16,384 tokens per GPU, global
m = 16,384 N) on the grid the paper's performance model ranks first
(axonn_grid_select, uniform NVSwitch bandwidth), unless --grid is given.

value = model flops of the step (6 m k n per layer, PAPER.md:786-795,
SPEC.md:443) summed over ranks / device time of the step (CUDA events on the
launching stream, max over ranks), in TFLOP/s.  e2e = the same metric with the
per-step inputs copied host->device from pinned memory and the weight
gradients read back, inside the timed region.  The block is chained the way
the paper's alternating transposed layers allow: proj's
output shard IS fc1's input shard and fc1's output shard IS fc2's (no
communication between them), and in backward fc2's dI is fc1's dO and fc1's
dI is proj's dO.  The step's external inputs are therefore the block input X
(QKV), the attention output (proj's input; attention is outside the FC path),
the loss gradient at fc2's output and attention-backward's gradient at QKV's
output.  --no-chain runs the four layers on independent inputs instead (and
then e2e uploads every layer's I and dO).
--impl reference times the CPU fp64 oracle (oracle/) on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "bf16 TFLOP/s per GPU (fraction of peak) for 3D-PMM FC fwd+bwd at 1/2/4/8 B200"
HIDDEN = {"5B": 4096, "10B": 5120, "20B": 7168, "40B": 9216, "80B": 12288}
FALLBACK_PEAKS = {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0}


def block_layers(h: int, m: int):
    """(m, k, n, transposed) of the four FC layers of one GPT block, phase A (R2b)."""
    return [(m, h, 3 * h, False), (m, h, h, True), (m, h, 4 * h, False), (m, 4 * h, h, True)]


def chain_plan(n_layers: int, chain: bool = True):
    """Which layers of a run of GPT blocks (4 FC layers each, phase A) take
    external inputs.  Chained: layer i's I is layer i-1's O
    and its dO is layer i+1's dI, except the first QKV input, every proj input
    (attention output), the last fc2's dO (loss gradient) and every QKV dO
    (attention backward).  Returns (ext_I ascending, ext_dO in backward order)."""
    if not chain:
        return list(range(n_layers)), list(reversed(range(n_layers)))
    ext_I = [i for i in range(n_layers) if i == 0 or i % 4 == 1]
    ext_dO = [i for i in reversed(range(n_layers)) if i == n_layers - 1 or i % 4 == 0]
    return ext_I, ext_dO


def model_flops(layers) -> float:
    return float(sum(6 * m * k * n for m, k, n, _ in layers))


_JSON_OUT = None


def emit(obj) -> None:
    f = _JSON_OUT or sys.stdout
    f.write(json.dumps(obj) + "\n")
    f.flush()


def copy_raw(dst: int, src: int, nbytes: int, stream) -> None:
    """cudaMemcpyAsync between raw addresses (a library-owned buffer) on `stream`."""
    import ctypes
    rt = ctypes.CDLL("libcudart.so.12")
    rc = rt.cudaMemcpyAsync(ctypes.c_void_p(dst), ctypes.c_void_p(src), ctypes.c_size_t(nbytes),
                            4, ctypes.c_void_p(stream.cuda_stream))
    if rc != 0:
        raise RuntimeError(f"cudaMemcpyAsync failed ({rc})")


def reduce_max(x: float, device: str = "cuda") -> float:
    """Max of a per-rank float over all ranks (device timing is max over ranks)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def read_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured (MEASURED_PEAKS.json)"
    return dict(FALLBACK_PEAKS), "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during timing."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                self.out, _ = self.proc.communicate()

    def summary(self):
        rows = []
        for line in (self.out or "").strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) != 7:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[3:]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for _, _, r in rows for n, v in zip(names, r) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows),
                "sm_max_mhz": max(r[1] for r in rows), "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------ CPU oracle legs
def oracle_sample(h: int, m_sample: int, min_seconds: float):
    """Time the fp64 oracle (oracle.fc) on the block's layers with m_sample rows,
    repeating until min_seconds elapsed.  Returns (TFLOP/s, threads, description)."""
    import numpy as np
    from oracle import fc
    import synthdata
    try:
        from threadpoolctl import threadpool_info
        threads = max((i.get("num_threads", 1) for i in threadpool_info()), default=os.cpu_count())
    except Exception:  # pragma: no cover
        threads = os.cpu_count()
    layers = block_layers(h, m_sample)
    data = [synthdata.layer_tensors(m, k, n, i) for i, (m, k, n, _) in enumerate(layers)]
    data = [tuple(a.astype(np.float64) for a in d) for d in data]
    flops, t0, reps = 0.0, time.perf_counter(), 0
    while True:
        for (X, W, dY), L in zip(data, layers):
            fc.fc_layer(X, W, dY)
            flops += model_flops([L])
        reps += 1
        el = time.perf_counter() - t0
        if el >= min_seconds or reps >= 50:
            break
    desc = (f"oracle.fc fp64 (numpy BLAS) on the GPT block's 4 FC layers fwd+bwd with "
            f"{m_sample} of the workload's token rows (h={h}), {reps} rep(s), {el:.1f} s")
    return flops / el / 1e12, threads, desc


def run_reference(args):
    """--impl reference: the oracle as it stands, on the host cores, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy  # noqa: F401  (load BLAS before lifting its thread limit)
    try:
        # torchrun exports OMP_NUM_THREADS=1 to every rank; this rank alone
        # works, so the oracle gets every host core it may run on
        from threadpoolctl import threadpool_limits
        _blas = threadpool_limits(limits=len(os.sched_getaffinity(0)))  # noqa: F841
    except Exception:  # pragma: no cover
        pass
    n = args.gpus
    h = HIDDEN[args.model]
    m_ref = 256
    import numpy as np
    from oracle import fc
    import synthdata
    layers = block_layers(h, m_ref)
    data = [tuple(a.astype(np.float64) for a in synthdata.layer_tensors(m, k, nn, i))
            for i, (m, k, nn, _) in enumerate(layers)]
    def step():
        for X, W, dY in data:
            fc.fc_layer(X, W, dY)
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = time.perf_counter() - t0
    val = model_flops(layers) * args.steps / el / 1e12
    try:
        from threadpoolctl import threadpool_info
        threads = max((i.get("num_threads", 1) for i in threadpool_info()), default=os.cpu_count())
    except Exception:  # pragma: no cover
        threads = os.cpu_count()
    sample = (f"oracle.fc fp64 on the GPT-{args.model} block's 4 FC layers fwd+bwd, {m_ref} token "
              f"rows per step (bounded sample of the {16384 * n}-token workload)")
    out = {"metric": METRIC, "value": val, "unit": "TFLOP/s", "impl": "reference", "n_gpus": n,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": workload_config(args.model, n, None),
           "cpu_baseline": {"value": val, "unit": "TFLOP/s", "cores": threads, "kind": "oracle",
                            "sample": sample},
           "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(out)


def workload_config(model, n, grid, tpg=16384, blocks=1):
    h = HIDDEN[model]
    return {"workload": ((f"{blocks} chained " if blocks > 1 else "") + f"GPT-{model} block FC layers (QKV h->3h, proj h->h, fc1 h->4h, fc2 4h->h; "
                         f"h={h}) Alg. 1 fwd+bwd, {tpg} tokens per GPU"
                         + (" (BASELINE.json configs[1], C2)"
                            if n == 1 and model == "5B" and tpg == 16384 and blocks == 1
                            else f", global m={tpg * n}")),
            "grid": list(grid) if grid else [1, 1, 1, 1], "tokens": tpg * n, "hidden": h,
            "phase": "A (proj, fc2 transposed)",
            "l2": "no flush: per-step operands (>= 134 MB each for I/dO of the fc2 layer) exceed the 126 MB L2"}


def bind_numa_local(device: int):
    """Pin this rank's host threads to the CPUs NVML reports as local to its
    GPU, before any pinned host buffer is allocated, so first-touch places the
    e2e staging buffers on the GPU's NUMA node (a cross-socket hop halves
    PCIe upload bandwidth when several ranks upload at once).  Returns the
    CPU count bound to, or None if NVML cannot say."""
    try:
        import pynvml
        import torch
        pr = torch.cuda.get_device_properties(device)
        pynvml.nvmlInit()
        hnd = pynvml.nvmlDeviceGetHandleByPciBusId(
            f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0")
        words = pynvml.nvmlDeviceGetCpuAffinity(hnd, (os.cpu_count() + 63) // 64)
        cpus = {64 * w + b for w, word in enumerate(words) for b in range(64) if word >> b & 1}
        cpus &= os.sched_getaffinity(0)
        if not cpus:
            return None
        os.sched_setaffinity(0, cpus)
        return len(cpus)
    except Exception:
        return None


# ------------------------------------------------------------------ GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="axonn", choices=["axonn", "reference"])
    ap.add_argument("--grid", default=None, help="gx,gy,gz,gd (default: model-selected)")
    ap.add_argument("--model", default="5B", choices=sorted(HIDDEN))
    ap.add_argument("--tokens-per-gpu", type=int, default=16384,
                    help="global m = tokens-per-gpu x N (BASELINE.json: 16384)")
    ap.add_argument("--chunks", type=int, default=4, help="forward AR pipelining chunks")
    ap.add_argument("--gemm-sms", type=int, default=0, help="SM budget of the GEMM grid (0 = all)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--graph", action="store_true",
                    help="capture one step in a CUDA graph and time its replays")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--w-init", default="scaled", choices=["scaled", "uniform"],
                    help="weights U(+-sqrt(3/k)) (random init) or U(-1,1)")
    ap.add_argument("--blocks", type=int, default=1,
                    help="GPT blocks per step, chained fc2 -> next QKV (SURVEY.md §8(f) f-1)")
    ap.add_argument("--grad-f32", action="store_true",
                    help="AXONN_BF16_GRADF32: dW in fp32, RS_z / data-parallel sums in fp32 (R17)")
    ap.add_argument("--recompute", action="store_true",
                    help="activation checkpointing (PAPER.md:722-723): each layer's forward re-runs "
                         "before its backward; flops counted 8mkn as Narayanan et al.'s formula does")
    ap.add_argument("--no-chain", action="store_true",
                    help="independent per-layer inputs (default: proj->fc1->fc2 chained)")
    args = ap.parse_args()
    # Exactly one JSON line on stdout: libraries (NCCL prints its version line)
    # write to fd 1, so fd 1 is pointed at stderr and the JSON goes to a copy.
    out_fd = os.dup(1)
    os.dup2(2, 1)
    global _JSON_OUT
    _JSON_OUT = os.fdopen(out_fd, "w")
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2502_08145_b200 as ax

    h = HIDDEN[args.model]
    m = args.tokens_per_gpu * world
    layers = block_layers(h, m) * args.blocks
    if args.grid:
        grid = tuple(int(x) for x in args.grid.split(","))
    elif world == 1:
        grid = (1, 1, 1, 1)
    else:
        tb = {(g0, g1): 1.0e11 for g0 in range(1, 9) for g1 in range(2, 9) if g0 * g1 <= 8}
        best = ax.axonn_grid_select(layers, world, 8, tb, 1.0e11, 2, 0, cap=1)[0]
        grid = (best["gx"], best["gy"], best["gz"], best["gd"])

    if world > 1:
        ax.bootstrap_from_torch_distributed(local)
    ax.axonn_grid_init(*grid)
    if args.gemm_sms:
        ax.axonn_set_gemm_sms(args.gemm_sms)

    stream = torch.cuda.Stream()
    gen = torch.Generator(device="cuda")
    gen.manual_seed(42 + rank)
    bf = torch.bfloat16

    def rnd(*shape, scale=1.0):
        t = torch.empty(shape, dtype=torch.float32, device="cuda")
        t.uniform_(-scale, scale, generator=gen)
        return t.to(bf)

    chain = not args.no_chain
    gdt = torch.float32 if args.grad_f32 else bf   # dŴ storage
    gsz = 4 if args.grad_f32 else 2
    gcode = ax.AXONN_BF16_GRADF32 if args.grad_f32 else ax.AXONN_BF16  # dW product dtype
    L = []
    for (mm, k, n, t) in layers:
        hd = ax.axonn_fc_create(mm, k, n, t,
                                ax.AXONN_BF16_GRADF32 if args.grad_f32 else ax.AXONN_BF16,
                                args.chunks)
        g = ax.axonn_fc_geometry(hd)
        # random-init weights, variance preserving (U(+-sqrt(3/k)): unit-variance
        # outputs for unit-variance inputs), so chained activations stay O(1)
        wscale = (3.0 / k) ** 0.5 if args.w_init == "scaled" else 1.0
        rec = {"h": hd, "g": g, "W": rnd(g.what_len, scale=wscale),
               "O": torch.empty(g.m_l, g.n_l, dtype=bf, device="cuda"),
               "dI": torch.empty(g.m_l, g.k_l, dtype=bf, device="cuda"),
               "dW": torch.empty(g.what_len, dtype=gdt, device="cuda")}
        # outputs of fused (NVLS) all-reduces live in handle-owned symmetric
        # buffers; writing there avoids the final copy (include/axonn.h)
        for key, which in (("O", 0), ("dI", 1), ("dW", 2)):
            ptr = ax.axonn_fc_output_buffer(hd, which)
            if ptr:
                rec[key] = ptr
        L.append(rec)
    # inputs: external (uniform(-1,1), uploaded by e2e) or chained
    # chained: inside a block proj -> fc1 -> fc2; across blocks fc2 (transposed,
    # columns over Y) -> the next block's QKV (normal, input columns over Y).
    # External: the first QKV input, every proj input (attention output), the
    # last fc2's dO (loss gradient) and every QKV dO (attention backward).
    nL = len(layers)
    ext_I, ext_dO = chain_plan(nL, chain)
    for i, l in enumerate(L):
        g = l["g"]
        if i in ext_I:
            l["I"] = rnd(g.m_l, g.k_l)
        else:
            # a transposed layer's input shard is the previous
            # (normal) layer's output shard and vice versa — same rows, same columns
            p = L[i - 1]["g"]
            assert (p.m_l, p.row0, p.n_l, p.out_col0) == (g.m_l, g.row0, g.k_l, g.in_col0), (p, g)
            l["I"] = L[i - 1]["O"]
        if i in ext_dO:
            l["dO"] = rnd(g.m_l, g.n_l)
        else:
            l["dO"] = L[i + 1]["dI"]

    def step(s):
        for i, l in enumerate(L):
            # OAG: the next layer's all-gather is issued before
            # this layer's forward, so it runs on the copy engines beside this GEMM
            if i + 1 < len(L):
                ax.axonn_fc_prefetch(L[i + 1]["h"], L[i + 1]["W"], s)
            ax.axonn_fc_forward(l["h"], l["I"], l["W"], l["O"], s)
        for l in reversed(L):
            if args.recompute:  # checkpointing: Alg. 1 lines 1-7 again, then 9-15
                ax.axonn_fc_forward(l["h"], l["I"], l["W"], l["O"], s)
            ax.axonn_fc_backward(l["h"], l["dO"], l["dI"], l["dW"], s)
        ax.axonn_grads_sync(s)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        return reduce_max(x, "cuda")

    ax.axonn_comm_bytes(reset=True)
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step(stream)
    barrier()

    # ---------------------------------------------------------------- timed region
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    graph = None
    if args.graph:
        # one whole step (every kernel, NCCL call, barrier, copy, cross-stream
        # event) captured once; profiling events inside it report the last replay
        ax.axonn_profile_read()
        ax.axonn_profile_enable(True)
        launches0 = ax.axonn_kernel_launches()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream, capture_error_mode="thread_local"):
            step(stream)
        ax.axonn_profile_enable(False)
        per_step_launches = ax.axonn_kernel_launches() - launches0
        for _ in range(2):
            graph.replay()
        barrier()
    launches0 = ax.axonn_kernel_launches()
    if not args.graph:
        ax.axonn_profile_read()
        ax.axonn_profile_enable(True)
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        with torch.cuda.stream(stream):
            for _ in range(args.steps):
                if graph is not None:
                    graph.replay()
                else:
                    step(stream)
        ev1.record(stream)
        barrier()
    ax.axonn_profile_enable(False)
    launches = ax.axonn_kernel_launches() - launches0
    if graph is not None:
        launches = per_step_launches * args.steps
    comm0 = ax.axonn_comm_bytes(reset=True)
    gemm_n, gemm_ms, gemm_flops = ax.axonn_profile_read()
    if graph is not None:  # events captured once hold the last replay: one step
        gemm_n, gemm_ms, gemm_flops = gemm_n * args.steps, gemm_ms * args.steps, gemm_flops * args.steps
    t_ms = max_over_ranks(ev0.elapsed_time(ev1)) / args.steps
    # whole job (all ranks): 6mkn per layer, 8mkn with recomputation
    flops_step = model_flops(layers) * (8.0 / 6.0 if args.recompute else 1.0)
    value = flops_step / (t_ms * 1e-3) / 1e12

    peaks, peaks_src = read_peaks()
    achieved = gemm_flops / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else 0.0
    peak = float(peaks.get("bf16_tflops_sustained", FALLBACK_PEAKS["bf16_tflops_sustained"]))
    burst = float(peaks.get("bf16_tflops", FALLBACK_PEAKS["bf16_tflops"]))
    traffic = None
    tf = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    if os.path.exists(tf):
        traffic = json.load(open(tf)).get("dram_bytes_per_launch")

    # ---------------------------------------------------------------- e2e
    e2e = None
    if not args.no_e2e:
        cpus0 = os.sched_getaffinity(0)
        numa_cpus = bind_numa_local(local)
        # Host buffers: each step uploads the block's external inputs (pinned;
        # with --no-chain every layer's I and dO) and reads every dW back.
        # Device inputs are double-buffered so step s+1's uploads (copy stream,
        # in consumption order) overlap step s's compute; read-backs run on a
        # third stream (PCIe is full duplex).
        hI = {i: L[i]["I"].cpu().pin_memory() for i in ext_I}
        hdO = {i: L[i]["dO"].cpu().pin_memory() for i in ext_dO}
        # the step's result, the weight gradient, crosses to the host once:
        # the Gd data-parallel replicas hold identical dŴ, so each reads back
        # the 1/Gd slice its DATA coordinate selects (the union over ranks is
        # every dŴ element exactly once)
        _, _, _, dcoord = ax.axonn_grid_coords()
        gd = grid[3]
        wsl = []
        for l in L:
            S_ = l["g"].what_len
            lo, hi = S_ * dcoord // gd, S_ * (dcoord + 1) // gd
            wsl.append((lo, hi))
        hdW = [torch.empty(hi - lo, dtype=gdt).pin_memory() for lo, hi in wsl]
        dev_sets = [[(l["I"], l["dO"]) for l in L],
                    [(torch.empty_like(L[i]["I"]) if i in ext_I else L[i]["I"],
                      torch.empty_like(L[i]["dO"]) if i in ext_dO else L[i]["dO"])
                     for i in range(len(L))]]
        up, down = torch.cuda.Stream(), torch.cuda.Stream()
        evI = [[torch.cuda.Event() for _ in L] for _ in range(2)]
        evO = [[torch.cuda.Event() for _ in L] for _ in range(2)]
        ev_free = [torch.cuda.Event(), torch.cuda.Event()]
        ev_done = torch.cuda.Event()
        ev_read = [torch.cuda.Event() for _ in L]
        bi = sum(t.numel() * 2 for t in list(hI.values()) + list(hdO.values()))
        bo = sum(t.numel() * gsz for t in hdW)
        # whole job: the slices' union is every weight-gradient element once
        bo_total = sum(gsz * k * n for (_, k, n, _) in layers)
        assert world > 1 or bo == bo_total

        def upload(s_idx):
            b = s_idx % 2
            with torch.cuda.stream(up):
                up.wait_event(ev_free[b])             # compute of step s-2 done with set b
                for i in ext_I:
                    dev_sets[b][i][0].copy_(hI[i], non_blocking=True)
                    evI[b][i].record(up)
                for i in ext_dO:
                    dev_sets[b][i][1].copy_(hdO[i], non_blocking=True)
                    evO[b][i].record(up)

        def compute(s_idx):
            b = s_idx % 2
            with torch.cuda.stream(stream):
                for i, l in enumerate(L):
                    if i + 1 < len(L):
                        ax.axonn_fc_prefetch(L[i + 1]["h"], L[i + 1]["W"], stream)
                    if i in ext_I:
                        stream.wait_event(evI[b][i])
                    ax.axonn_fc_forward(l["h"], dev_sets[b][i][0], l["W"], l["O"], stream)
                for i in reversed(range(len(L))):
                    if i in ext_dO:
                        stream.wait_event(evO[b][i])
                    stream.wait_event(ev_read[i])    # previous step's dŴ has reached the host
                    if args.recompute:
                        ax.axonn_fc_forward(L[i]["h"], dev_sets[b][i][0], L[i]["W"], L[i]["O"],
                                            stream)
                    ax.axonn_fc_backward(L[i]["h"], dev_sets[b][i][1], L[i]["dI"], L[i]["dW"], stream)
                ax.axonn_grads_sync(stream)
                ev_free[b].record(stream)
                ev_done.record(stream)
            with torch.cuda.stream(down):
                down.wait_event(ev_done)
                for i in reversed(range(len(L))):    # in the next step's backward order
                    l = L[i]
                    if isinstance(l["dW"], int):
                        copy_raw(hdW[i].data_ptr(), l["dW"] + gsz * wsl[i][0], hdW[i].numel() * gsz,
                                 down)
                    else:
                        hdW[i].copy_(l["dW"][wsl[i][0]:wsl[i][1]], non_blocking=True)
                    ev_read[i].record(down)

        def e2e_run(n):
            upload(0)
            for s_idx in range(n):
                if s_idx + 1 < n:
                    upload(s_idx + 1)
                compute(s_idx)

        e2e_run(2)
        barrier()
        ksteps = max(3, min(args.steps, 10))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record(stream)
        stream.wait_stream(torch.cuda.current_stream())
        up.wait_event(e0)
        down.wait_event(e0)
        e2e_run(ksteps)
        stream.wait_stream(down)
        stream.wait_stream(up)
        e1.record(stream)
        barrier()
        te = max_over_ranks(e0.elapsed_time(e1)) / ksteps
        e2e = {"value": flops_step / (te * 1e-3) / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": bi * world, "d2h_bytes_per_step": bo_total,
               "ms_per_step": te, "steps": ksteps,
               "numa_local_cpus": numa_cpus,
               "inputs": ("block input X, attention output (proj input), loss gradient at fc2 "
                          "output, attention-backward gradient at QKV output; proj->fc1->fc2 chained "
                          "on device (PAPER.md:402-414)") if chain else "every layer's I and dO",
               "path": "pinned host -> device uploads (double-buffered, copy stream) + "
                       "axonn_fc_forward/backward + grads_sync + dW device->host (third stream),"
                       " all inside the timed region"}

        os.sched_setaffinity(0, cpus0)   # the CPU baseline below uses every core

    # ---------------------------------------------------------------- GEMM-only (exposed comm)
    exposed = None
    if world > 1:
        scratch = []
        for l, (_, k_glob, _, _) in zip(L, layers):
            g = l["g"]
            a = (3.0 / k_glob) ** 0.5 if args.w_init == "scaled" else 1.0  # as the Alg. 1 step
            scratch.append((g, torch.empty(g.k_l, g.n_l, dtype=bf, device="cuda").uniform_(-a, a),
                            torch.empty(g.k_l, g.n_l, dtype=gdt, device="cuda")))

        def gemm_step(s):
            for l, (g, Wf, _) in zip(L, scratch):
                ax.axonn_gemm(0, 0, g.m_l, g.n_l, g.k_l, l["I"], g.k_l, Wf, g.n_l, l["O"], g.n_l, s)
            for l, (g, Wf, dWf) in zip(reversed(L), reversed(scratch)):
                if args.recompute:
                    ax.axonn_gemm(0, 0, g.m_l, g.n_l, g.k_l, l["I"], g.k_l, Wf, g.n_l, l["O"], g.n_l, s)
                ax.axonn_gemm(1, 0, g.m_l, g.k_l, g.n_l, l["dO"], g.n_l, Wf, g.n_l, l["dI"], g.k_l, s)
                ax.axonn_gemm(2, gcode, g.k_l, g.n_l, g.m_l, l["I"], g.k_l, l["dO"], g.n_l, dWf, g.n_l, s)

        for _ in range(2):
            gemm_step(stream)
        barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(args.steps):
            gemm_step(stream)
        g1.record(stream)
        barrier()
        t_gemm = max_over_ranks(g0.elapsed_time(g1)) / args.steps

        # per layer: Alg. 1 forward / backward through the ABI vs the same
        # local products alone (SURVEY.md §8(d) "per layer and per block")
        names = [["qkv", "proj", "fc1", "fc2"][i % 4] + (f"{i // 4}" if args.blocks > 1 else "")
                 for i in range(nL)]
        nrep = max(3, min(args.steps, 20))
        ev = {key: [torch.cuda.Event(enable_timing=True) for _ in range(2 * nrep)]
              for key in [f"{n_}_{ph}" for n_ in names for ph in ("fwd", "bwd", "fwd_gemm", "bwd_gemm")]
              + ["sync"]}
        acc_ms = {key: 0.0 for key in ev}
        for rep in range(nrep):
            with torch.cuda.stream(stream):
                for i, l in enumerate(L):
                    if i + 1 < len(L):
                        ax.axonn_fc_prefetch(L[i + 1]["h"], L[i + 1]["W"], stream)
                    ev[f"{names[i]}_fwd"][2 * rep].record(stream)
                    ax.axonn_fc_forward(l["h"], l["I"], l["W"], l["O"], stream)
                    ev[f"{names[i]}_fwd"][2 * rep + 1].record(stream)
                for i in reversed(range(len(L))):
                    l = L[i]
                    ev[f"{names[i]}_bwd"][2 * rep].record(stream)
                    ax.axonn_fc_backward(l["h"], l["dO"], l["dI"], l["dW"], stream)
                    ev[f"{names[i]}_bwd"][2 * rep + 1].record(stream)
                ev["sync"][2 * rep].record(stream)
                ax.axonn_grads_sync(stream)
                ev["sync"][2 * rep + 1].record(stream)
                for i, (l, (g, Wf, dWf)) in enumerate(zip(L, scratch)):
                    ev[f"{names[i]}_fwd_gemm"][2 * rep].record(stream)
                    ax.axonn_gemm(0, 0, g.m_l, g.n_l, g.k_l, l["I"], g.k_l, Wf, g.n_l, l["O"], g.n_l, stream)
                    ev[f"{names[i]}_fwd_gemm"][2 * rep + 1].record(stream)
                    ev[f"{names[i]}_bwd_gemm"][2 * rep].record(stream)
                    ax.axonn_gemm(1, 0, g.m_l, g.k_l, g.n_l, l["dO"], g.n_l, Wf, g.n_l, l["dI"], g.k_l, stream)
                    ax.axonn_gemm(2, gcode, g.k_l, g.n_l, g.m_l, l["I"], g.k_l, l["dO"], g.n_l, dWf, g.n_l, stream)
                    ev[f"{names[i]}_bwd_gemm"][2 * rep + 1].record(stream)
        barrier()
        for key, lst in ev.items():
            acc_ms[key] = max_over_ranks(sum(lst[2 * r].elapsed_time(lst[2 * r + 1])
                                             for r in range(nrep)) / nrep)
        per_layer = {}
        for n_ in names:
            for ph in ("fwd", "bwd"):
                t_op, t_g = acc_ms[f"{n_}_{ph}"], acc_ms[f"{n_}_{ph}_gemm"]
                per_layer[f"{n_}_{ph}"] = {"ms": t_op, "gemm_only_ms": t_g,
                                           "exposed_frac": max(0.0, (t_op - t_g) / t_op) if t_op else 0.0}
        per_layer["grads_sync"] = {"ms": acc_ms["sync"]}
        exposed = {"t_step_ms": t_ms, "t_gemm_only_ms": t_gemm, "per_layer": per_layer,
                   "exposed_comm_frac": max(0.0, (t_ms - t_gemm) / t_ms),
                   "comm_bytes_per_rank_per_step": {k: v // max(1, args.steps + args.warmup)
                                                    for k, v in comm0.items()}}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, thr, desc = oracle_sample(h, 2048, 10.0)
        cpu = {"value": v, "unit": "TFLOP/s", "cores": thr, "kind": "oracle", "sample": desc}

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": ("synthetic (inputs uniform(-1,1) bf16, weights "
                     + ("U(+-sqrt(3/k)) random init" if args.w_init == "scaled" else "U(-1,1)")
                     + ", device-generated, seeded)"),
            "config": {**workload_config(args.model, world, grid, args.tokens_per_gpu, args.blocks),
                       "chained": chain, "recompute": bool(args.recompute),
                       "grad_f32": bool(args.grad_f32),
                       "flops_per_layer": "8mkn (forward recomputed)" if args.recompute else "6mkn"},
            "per_gpu_tflops": value / world,
            "frac_of_peak": {"advertised_2250": value / world / 2250.0,
                             "measured_burst": value / world / burst,
                             "measured_sustained": value / world / peak, "peaks": peaks_src},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak,
                         "unit": "TFLOP/s", "frac": achieved / peak if peak else None,
                         "traffic": traffic,
                         "kernel": "gemm_bf16_tcgen05 (all NN/NT/TN launches of the timed region;"
                                   " achieved = sum 2MNK / sum event time)",
                         "peak_kind": f"bf16_tflops_sustained, {peaks_src}",
                         "frac_of_burst": achieved / burst if burst else None,
                         "gemm_launches": gemm_n, "gemm_ms_per_step": gemm_ms / args.steps},
            "cuda_graph": bool(args.graph),
            "gpu_launches": launches,
            "overlap": exposed,
            "clocks": clk.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        emit(out)
    ax.axonn_grid_finalize()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
