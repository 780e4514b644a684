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
1x1x1x1.  N > 1 measures the 3D PMM on tensor grids (PRIMARY below): N = 8
is C3 exactly (GPT-20B block, m = 16,384, grid 2x2x2x1); N = 4 the C3 proxy
(m = 8192 on 2x2x1x1: C3's local GEMMs and all-reduce sizes); N = 2 the
20B block on 2x1x1x1 at C3's per-GPU flops.  Sub-records of the same line
(SUB): the C4a / C4b (80B, phase B) and C5 (40B, tensor x data) configs or
their 4-GPU proxies, and the data-parallel weak-scaling line (5B, 16,384
tokens per GPU, the grid the paper's performance model ranks first with the
measured Case-1 table).  --grid / --model / --tokens override the plan.

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


def block_layers(h: int, m: int, phase: str = "A"):
    """(m, k, n, transposed) of the four FC layers of one GPT block (Table II
    shapes).  Phase A transposes proj and fc2, phase B QKV and fc1 (R2b)."""
    if phase not in ("A", "B"):
        raise ValueError(f"phase must be 'A' or 'B', got {phase!r}")
    t = [False, True, False, True] if phase == "A" else [True, False, True, False]
    return [(m, h, 3 * h, t[0]), (m, h, h, t[1]), (m, h, 4 * h, t[2]), (m, 4 * h, h, t[3])]


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


def write_trace(path, c, ev, t_base, nrep, spec) -> None:
    """Chrome-trace JSON (chrome://tracing, Perfetto) of the instrumented
    per-layer steps: one complete event per layer phase and repetition on the
    launching stream, CUDA-event timestamps relative to the first, one process
    per rank (rank 0 gathers and writes)."""
    import torch.distributed as dist
    events = []
    rank = dist.get_rank() if dist.is_available() and dist.is_initialized() else 0
    for key, lst in ev.items():
        cat = "gemm_only" if key.endswith("_gemm") else ("sync" if key == "sync" else "alg1")
        for r in range(nrep):
            t0 = t_base.elapsed_time(lst[2 * r]) * 1e3
            dur = lst[2 * r].elapsed_time(lst[2 * r + 1]) * 1e3
            events.append({"name": key, "cat": cat, "ph": "X", "ts": round(t0, 3),
                           "dur": round(dur, 3), "pid": rank, "tid": "compute stream",
                           "args": {"rep": r}})
    allr = [events]
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        allr = [None] * dist.get_world_size()
        dist.all_gather_object(allr, events)
    if rank == 0:
        meta = [{"name": "process_name", "ph": "M", "pid": r, "args": {"name": f"rank {r}"}}
                for r in range(len(allr))]
        json.dump({"traceEvents": meta + [e for evs in allr for e in evs],
                   "displayTimeUnit": "ms",
                   "otherData": {"workload": spec.get("label", ""), "grid": spec.get("grid")}},
                  open(path, "w"))


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


def torch_cpu_bf16_sample(h: int, m_sample: int, min_seconds: float):
    """The same block's products with torch CPU bf16 matmuls (oneDNN, AMX where
    the host has it): the CPU bf16 throughput BASELINE.md quotes beside the
    oracle.  Returns (TFLOP/s, threads)."""
    import torch
    layers = block_layers(h, m_sample)
    g = torch.Generator().manual_seed(42)
    data = [(torch.rand(m, k, generator=g).bfloat16(), torch.rand(k, n, generator=g).bfloat16(),
             torch.rand(m, n, generator=g).bfloat16()) for m, k, n, _ in layers]
    flops, t0, reps = 0.0, time.perf_counter(), 0
    while True:
        for (X, W, dY), L in zip(data, layers):
            X @ W
            dY @ W.t()
            X.t() @ dY
            flops += model_flops([L])
        reps += 1
        el = time.perf_counter() - t0
        if el >= min_seconds or reps >= 50:
            break
    return flops / el / 1e12, torch.get_num_threads()


def run_reference(args):
    """--impl reference: the oracle as it stands, on the host cores, rank 0 only,
    on a bounded sample of the primary workload of this GPU count."""
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
    spec = PRIMARY.get(n) if not (args.model or args.grid or args.tokens or args.tokens_per_gpu) else None
    if spec is None:
        model = args.model or "5B"
        spec = dict(model=model, m=args.tokens or (args.tokens_per_gpu or 16384) * n,
                    grid=tuple(int(x) for x in args.grid.split(",")) if args.grid else None,
                    phase=args.phase or "A", label="custom")
    h = HIDDEN[spec["model"]]
    m_ref = 256
    import numpy as np
    from oracle import fc
    import synthdata
    layers = block_layers(h, m_ref, spec.get("phase", "A"))
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
    sample = (f"oracle.fc fp64 on the GPT-{spec['model']} block's 4 FC layers fwd+bwd, {m_ref} token "
              f"rows per step (bounded sample of the {spec['m']}-token workload)")
    out = {"metric": METRIC, "value": val, "unit": "TFLOP/s", "impl": "reference", "n_gpus": n,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic",
           "config": {**workload_config(spec["model"], n, spec.get("grid"), spec["m"], 1,
                                        spec.get("phase", "A")), "label": spec.get("label", "")},
           "cpu_baseline": {"value": val, "unit": "TFLOP/s", "cores": threads, "kind": "oracle",
                            "sample": sample},
           "e2e": {"value": val, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(out)


def workload_config(model, n, grid, m, blocks=1, phase="A"):
    """config of the JSON line: the workload named by BASELINE.json."""
    h = HIDDEN[model]
    c2 = n == 1 and model == "5B" and m == 16384 and blocks == 1 and tuple(grid or (1, 1, 1, 1)) == (1, 1, 1, 1)
    return {"workload": ((f"{blocks} chained " if blocks > 1 else "")
                         + f"GPT-{model} block FC layers (QKV h->3h, proj h->h, fc1 h->4h, fc2 4h->h; "
                         f"h={h}) Alg. 1 fwd+bwd, m={m} global tokens on {n} GPU(s)"
                         + (" (BASELINE.json configs[1], C2)" if c2 else "")),
            "grid": list(grid) if grid else [1, 1, 1, 1], "tokens": m, "hidden": h,
            "phase": "A (proj, fc2 transposed)" if phase == "A" else "B (QKV, fc1 transposed)",
            "l2": "no flush: per-step operands (>= 58 MB each, most >= 134 MB) exceed the 126 MB "
                  "L2 across the step's 12+ GEMMs"}


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


# ------------------------------------------------------------------ configurations
# Default workloads per GPU count (BASELINE.json configs).
#   N = 1: C2, the GPT-5B block on 1x1x1x1 (configs[1]).
#   N = 8: C3 exactly: the GPT-20B block, m = 16384 global tokens, 2x2x2x1.
#   N = 4: the C3 proxy (2,2,1,1) at m = 8192: every rank runs C3's local GEMM
#          shapes and C3's AR_x / AR_y message sizes (one Z level fewer).
#   N = 2: (2,1,1,1) at m = 4096: C3's per-GPU flops on a 2-GPU tensor grid.
# Per-GPU work is C3's at N = 2, 4, 8 (weak scaling of the C3 workload).
# Sub-records of the same JSON line (N = 4 proxies / N = 8 exact): C4a / C4b
# (80B, the model's phase-B pair 1x4x2 and 2x4x1) and C5 (40B,
# 2x2x1 x Gd=2), plus the data-parallel weak-scaling line (5B block, 16384
# tokens per GPU, the grid the performance model ranks first).
PRIMARY = {
    1: dict(label="C2", model="5B", m=16384, grid=(1, 1, 1, 1), phase="A"),
    2: dict(label="C3 family at N=2 (C3's per-GPU flops)", model="20B", m=4096,
            grid=(2, 1, 1, 1), phase="A"),
    4: dict(label="C3 proxy (C3's local shapes and AR sizes)", model="20B", m=8192,
            grid=(2, 2, 1, 1), phase="A"),
    8: dict(label="C3", model="20B", m=16384, grid=(2, 2, 2, 1), phase="A"),
}
SUB = {
    4: [dict(label="C4a proxy (80B, phase B)", model="80B", m=16384, grid=(1, 2, 2, 1), phase="B"),
        dict(label="C4b proxy (80B, phase B)", model="80B", m=16384, grid=(2, 2, 1, 1), phase="B"),
        dict(label="C5 proxy (40B, tensor x data)", model="40B", m=16384, grid=(2, 1, 1, 2),
             phase="A")],
    8: [dict(label="C4a", model="80B", m=16384, grid=(1, 4, 2, 1), phase="B"),
        dict(label="C4b", model="80B", m=16384, grid=(2, 4, 1, 1), phase="B"),
        dict(label="C5", model="40B", m=16384, grid=(2, 2, 1, 2), phase="A")],
}


def case1_table(path=None):
    """Measured Case-1 database for grid selection:
    {(G0, G1): bytes/s}.  Entries missing from the measured file (e.g. the
    8-GPU groups of a 4-GPU measurement) take the mean of the measured ones;
    with no file, uniform 1e11 (Case 1 with equal beta).  Returns (table, source)."""
    path = path or os.path.join(ROOT, "profiles", "case1_table.json")
    full = [(g0, g1) for g0 in range(1, 9) for g1 in range(2, 9) if g0 * g1 <= 8]
    if os.path.exists(path):
        d = json.load(open(path))
        meas = {tuple(int(x) for x in k.split(",")): float(v) * 1e9
                for k, v in d["beta_GBps"].items()}
        fill = sum(meas.values()) / len(meas)
        return ({k: meas.get(k, fill) for k in full},
                f"measured {os.path.relpath(path, ROOT)} ({len(meas)} entries; others = their mean)")
    return {k: 1.0e11 for k in full}, "uniform beta 1e11 (no measured table)"


def model_top1(ax, layers, world, fixed_gd=0):
    tb, src = case1_table()
    best = ax.axonn_grid_select(layers, world, 8, tb, 1.0e11, 2, fixed_gd, cap=1)[0]
    return (best["gx"], best["gy"], best["gz"], best["gd"]), src


# ------------------------------------------------------------------ GPU arm
class Ctx:
    pass


def run_config(c, spec, steps, warmup, e2e_on, exposure_on):
    """Time one workload: `spec` = dict(model, m (global tokens), grid, phase,
    blocks, chain, label).  Returns the record (value, overlap, e2e, ...)."""
    ax, torch, dist, args = c.ax, c.torch, c.dist, c.args
    world, rank, local = c.world, c.rank, c.local
    h = HIDDEN[spec["model"]]
    m = spec["m"]
    grid = tuple(spec["grid"])
    blocks = spec.get("blocks", 1)
    chain = spec.get("chain", True)
    layers = block_layers(h, m, spec.get("phase", "A")) * blocks
    ax.axonn_grid_init(*grid)
    stream = c.stream
    gen = torch.Generator(device="cuda")
    gen.manual_seed(42 + rank)
    bf = torch.bfloat16

    def rnd(*shape, scale=1.0):
        t = torch.empty(shape, dtype=torch.float32, device="cuda")
        t.uniform_(-scale, scale, generator=gen)
        return t.to(bf)

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
    # chained: inside a block proj -> fc1 -> fc2; across blocks fc2 -> the next
    # block's QKV (alternating normal/transposed layers share shard layouts).
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
        for _ in range(warmup):
            step(stream)
    barrier()
    if args.soak > 0:
        # untimed steps until the power cap has settled the clocks (the
        # default stays 0: the timed region is exactly --steps steps)
        t0 = time.perf_counter()
        with torch.cuda.stream(stream):
            while time.perf_counter() - t0 < args.soak:
                step(stream)
                torch.cuda.synchronize()
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
    ax.axonn_comm_bytes(reset=True)
    launches0 = ax.axonn_kernel_launches()
    if not args.graph:
        ax.axonn_profile_read()
        ax.axonn_profile_enable(True)
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        with torch.cuda.stream(stream):
            for _ in range(steps):
                if graph is not None:
                    graph.replay()
                else:
                    step(stream)
        ev1.record(stream)
        barrier()
    ax.axonn_profile_enable(False)
    launches = ax.axonn_kernel_launches() - launches0
    if graph is not None:
        launches = per_step_launches * steps
    comm0 = ax.axonn_comm_bytes(reset=True)
    gemm_n, gemm_ms, gemm_flops = ax.axonn_profile_read()
    if graph is not None:  # events captured once hold the last replay: one step
        gemm_n, gemm_ms, gemm_flops = gemm_n * steps, gemm_ms * steps, gemm_flops * steps
    t_ms = max_over_ranks(ev0.elapsed_time(ev1)) / steps
    # whole job (all ranks): 6mkn per layer, 8mkn with recomputation
    flops_step = model_flops(layers) * (8.0 / 6.0 if args.recompute else 1.0)
    value = flops_step / (t_ms * 1e-3) / 1e12
    clocks = clk.summary()

    # ---------------------------------------------------------------- e2e
    e2e = None
    if e2e_on:
        cpus0 = os.sched_getaffinity(0)
        numa_cpus = bind_numa_local(local)
        # Host buffers: each step uploads the block's external inputs (pinned;
        # with --no-chain every layer's I and dO) and reads the step's results
        # back: every dŴ, the block output O (last fc2) and the block input
        # gradient dX (first QKV's dI).  Device inputs are double-buffered so
        # step s+1's uploads (copy stream, in consumption order) overlap step
        # s's compute; read-backs run on a third stream (PCIe is full duplex).
        hI = {i: L[i]["I"].cpu().pin_memory() for i in ext_I}
        hdO = {i: L[i]["dO"].cpu().pin_memory() for i in ext_dO}
        # the weight gradient crosses to the host once: the Gd data-parallel
        # replicas hold identical dŴ, so each reads back the 1/Gd slice its
        # DATA coordinate selects (the union over ranks is every dŴ element once)
        _, _, _, dcoord = ax.axonn_grid_coords()
        gd = grid[3]
        wsl = []
        for l in L:
            S_ = l["g"].what_len
            lo, hi = S_ * dcoord // gd, S_ * (dcoord + 1) // gd
            wsl.append((lo, hi))
        hdW = [torch.empty(hi - lo, dtype=gdt).pin_memory() for lo, hi in wsl]
        gl, g0_ = L[-1]["g"], L[0]["g"]
        hO = torch.empty(gl.m_l * gl.n_l, dtype=bf).pin_memory()    # block output O
        hdX = torch.empty(g0_.m_l * g0_.k_l, dtype=bf).pin_memory()  # block input gradient
        dev_sets = [[(l["I"], l["dO"]) for l in L],
                    [(torch.empty_like(L[i]["I"]) if i in ext_I else L[i]["I"],
                      torch.empty_like(L[i]["dO"]) if i in ext_dO else L[i]["dO"])
                     for i in range(len(L))]]
        up, down = torch.cuda.Stream(), torch.cuda.Stream()
        evI = [[torch.cuda.Event() for _ in L] for _ in range(2)]
        evO = [[torch.cuda.Event() for _ in L] for _ in range(2)]
        ev_free = [torch.cuda.Event(), torch.cuda.Event()]
        ev_done = torch.cuda.Event()
        ev_fwd = torch.cuda.Event()
        ev_read = [torch.cuda.Event() for _ in L]
        ev_readO, ev_readX = torch.cuda.Event(), torch.cuda.Event()
        bi = sum(t.numel() * 2 for t in list(hI.values()) + list(hdO.values()))
        bo = sum(t.numel() * gsz for t in hdW) + 2 * (hO.numel() + hdX.numel())

        def raw_read(dst_t, src, nbytes, off=0):
            if isinstance(src, int):
                copy_raw(dst_t.data_ptr(), src + off, nbytes, down)
            else:
                dst_t.copy_(src.reshape(-1)[off // dst_t.element_size():
                                            (off + nbytes) // dst_t.element_size()],
                            non_blocking=True)

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
                    if i == len(L) - 1:
                        stream.wait_event(ev_readO)  # previous step's O has reached the host
                    ax.axonn_fc_forward(l["h"], dev_sets[b][i][0], l["W"], l["O"], stream)
                ev_fwd.record(stream)
                for i in reversed(range(len(L))):
                    if i in ext_dO:
                        stream.wait_event(evO[b][i])
                    stream.wait_event(ev_read[i])    # previous step's dŴ has reached the host
                    if i == 0:
                        stream.wait_event(ev_readX)
                    if args.recompute:
                        ax.axonn_fc_forward(L[i]["h"], dev_sets[b][i][0], L[i]["W"], L[i]["O"],
                                            stream)
                    ax.axonn_fc_backward(L[i]["h"], dev_sets[b][i][1], L[i]["dI"], L[i]["dW"], stream)
                ax.axonn_grads_sync(stream)
                ev_free[b].record(stream)
                ev_done.record(stream)
            with torch.cuda.stream(down):
                down.wait_event(ev_fwd)              # the block output, during the backward
                raw_read(hO, L[-1]["O"], 2 * hO.numel())
                ev_readO.record(down)
                down.wait_event(ev_done)
                raw_read(hdX, L[0]["dI"], 2 * hdX.numel())
                ev_readX.record(down)
                for i in reversed(range(len(L))):    # in the next step's backward order
                    raw_read(hdW[i], L[i]["dW"], hdW[i].numel() * gsz, gsz * wsl[i][0])
                    ev_read[i].record(down)

        def e2e_run(n):
            upload(0)
            for s_idx in range(n):
                if s_idx + 1 < n:
                    upload(s_idx + 1)
                compute(s_idx)

        e2e_run(2)
        barrier()
        ksteps = max(3, min(steps, 10))
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
               "h2d_bytes_per_step": bi * world, "d2h_bytes_per_step": bo * world,
               "ms_per_step": te, "steps": ksteps,
               "numa_local_cpus": numa_cpus,
               "inputs": ("block input X, attention output (proj input), loss gradient at fc2 "
                          "output, attention-backward gradient at QKV output; proj->fc1->fc2 chained "
                          "on device (PAPER.md:402-414)") if chain else "every layer's I and dO",
               "outputs": ("every weight gradient dŴ (each data-parallel replica its 1/Gd slice), "
                           "the block output O (last fc2's output shard) and the block input "
                           "gradient dX (first QKV's dI shard), per rank"),
               "path": "pinned host -> device uploads (double-buffered, copy stream) + "
                       "axonn_fc_forward/backward + grads_sync + results device->host (third "
                       "stream), all inside the timed region"}
        os.sched_setaffinity(0, cpus0)   # the CPU baseline uses every core

    # ---------------------------------------------------------------- GEMM-only (exposed comm)
    exposed = None
    if exposure_on and world > 1:
        scratch = []
        for l, (_, k_glob, _, _) in zip(L, layers):
            g = l["g"]
            a = (3.0 / k_glob) ** 0.5 if args.w_init == "scaled" else 1.0  # as the Alg. 1 step
            scratch.append((g, torch.empty(g.k_l, g.n_l, dtype=bf, device="cuda").uniform_(-a, a),
                            torch.empty(g.k_l, g.n_l, dtype=gdt, device="cuda")))

        # the GEMM-only reference writes its forward outputs to scratch: the
        # handle-owned output buffers are read-only for the caller
        # (include/axonn.h, axonn_fc_output_buffer)
        Oscr = [torch.empty(l["g"].m_l, l["g"].n_l, dtype=bf, device="cuda") for l in L]
        dIscr = [torch.empty(l["g"].m_l, l["g"].k_l, dtype=bf, device="cuda") for l in L]

        def gemm_step(s):
            for l, (g, Wf, _), Os in zip(L, scratch, Oscr):
                ax.axonn_gemm(0, 0, g.m_l, g.n_l, g.k_l, l["I"], g.k_l, Wf, g.n_l, Os, g.n_l, s)
            for l, (g, Wf, dWf), Os, dIs in zip(reversed(L), reversed(scratch), reversed(Oscr),
                                                 reversed(dIscr)):
                if args.recompute:
                    ax.axonn_gemm(0, 0, g.m_l, g.n_l, g.k_l, l["I"], g.k_l, Wf, g.n_l, Os, g.n_l, s)
                ax.axonn_gemm(1, 0, g.m_l, g.k_l, g.n_l, l["dO"], g.n_l, Wf, g.n_l, dIs, g.k_l, s)
                ax.axonn_gemm(2, gcode, g.k_l, g.n_l, g.m_l, l["I"], g.k_l, l["dO"], g.n_l, dWf, g.n_l, s)

        for _ in range(2):
            gemm_step(stream)
        barrier()
        # exposure from interleaved windows (fused step, then the same local
        # GEMMs alone, three times), so both see the same power state; the
        # headline window above stays one contiguous region
        kk = max(3, steps // 3)
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t_ab, t_g = 0.0, 0.0
        for _ in range(3):
            barrier()
            g0.record(stream)
            with torch.cuda.stream(stream):
                for _ in range(kk):
                    if graph is not None:
                        graph.replay()
                    else:
                        step(stream)
            g1.record(stream)
            barrier()
            t_ab += g0.elapsed_time(g1)
            g0.record(stream)
            for _ in range(kk):
                gemm_step(stream)
            g1.record(stream)
            barrier()
            t_g += g0.elapsed_time(g1)
        t_step_ab = max_over_ranks(t_ab) / (3 * kk)
        t_gemm = max_over_ranks(t_g) / (3 * kk)

        # per layer: Alg. 1 forward / backward through the ABI vs the same
        # local products alone (SURVEY.md §8(d) "per layer and per block")
        names = [["qkv", "proj", "fc1", "fc2"][i % 4] + (f"{i // 4}" if blocks > 1 else "")
                 for i in range(nL)]
        nrep = max(3, min(steps, 20))
        ev = {key: [torch.cuda.Event(enable_timing=True) for _ in range(2 * nrep)]
              for key in [f"{n_}_{ph}" for n_ in names for ph in ("fwd", "bwd", "fwd_gemm", "bwd_gemm")]
              + ["sync"]}
        acc_ms = {key: 0.0 for key in ev}
        t_base = torch.cuda.Event(enable_timing=True)
        t_base.record(stream)
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
                    ax.axonn_gemm(0, 0, g.m_l, g.n_l, g.k_l, l["I"], g.k_l, Wf, g.n_l, Oscr[i], g.n_l, stream)
                    ev[f"{names[i]}_fwd_gemm"][2 * rep + 1].record(stream)
                    ev[f"{names[i]}_bwd_gemm"][2 * rep].record(stream)
                    ax.axonn_gemm(1, 0, g.m_l, g.k_l, g.n_l, l["dO"], g.n_l, Wf, g.n_l, dIscr[i], g.k_l, stream)
                    ax.axonn_gemm(2, gcode, g.k_l, g.n_l, g.m_l, l["I"], g.k_l, l["dO"], g.n_l, dWf, g.n_l, stream)
                    ev[f"{names[i]}_bwd_gemm"][2 * rep + 1].record(stream)
        barrier()
        for key, lst in ev.items():
            acc_ms[key] = max_over_ranks(sum(lst[2 * r].elapsed_time(lst[2 * r + 1])
                                             for r in range(nrep)) / nrep)
        if getattr(args, "trace", None) and spec.get("primary", True):
            write_trace(args.trace, c, ev, t_base, nrep, spec)
        per_layer = {}
        for n_ in names:
            for ph in ("fwd", "bwd"):
                t_op, t_g = acc_ms[f"{n_}_{ph}"], acc_ms[f"{n_}_{ph}_gemm"]
                per_layer[f"{n_}_{ph}"] = {"ms": t_op, "gemm_only_ms": t_g,
                                           "exposed_frac": max(0.0, (t_op - t_g) / t_op) if t_op else 0.0}
        per_layer["grads_sync"] = {"ms": acc_ms["sync"]}
        exposed = {"t_step_ms": t_ms, "t_step_interleaved_ms": t_step_ab,
                   "t_gemm_only_ms": t_gemm, "per_layer": per_layer,
                   "exposed_comm_frac": max(0.0, (t_step_ab - t_gemm) / t_step_ab),
                   "exposure_method": "interleaved windows: 3 x (fused steps, then the same local "
                                      "GEMMs alone, outputs to scratch), max over ranks",
                   "comm_bytes_per_rank_per_step": {k: v // max(1, steps)
                                                    for k, v in comm0.items()},
                   "comm_bytes_note": "bytes the collectives of one step send per rank "
                                      "(ring formulas of Eqs. 1-5 on the element counts issued)"}
    fused = {a: ax.axonn_fused_status(a) for a in ("x", "y", "z", "d")}
    for l in L:
        ax.axonn_fc_destroy(l["h"])
    ax.axonn_grid_finalize()
    del L
    torch.cuda.empty_cache()
    rec = {"label": spec.get("label", ""), "value": value, "per_gpu_tflops": value / world,
           "ms_per_step": t_ms, "steps": steps, "warmup": warmup,
           "config": {**workload_config(spec["model"], world, grid, m, blocks, spec.get("phase", "A")),
                      "chained": chain, "recompute": bool(args.recompute),
                      "grad_f32": bool(args.grad_f32),
                      "flops_per_layer": "8mkn (forward recomputed)" if args.recompute else "6mkn"},
           "gpu_launches": launches, "overlap": exposed, "clocks": clocks, "e2e": e2e,
           "fused_axes": fused,
           "gemm": {"launches": gemm_n, "ms": gemm_ms, "flops": gemm_flops}}
    if "grid_source" in spec:
        rec["config"]["grid_source"] = spec["grid_source"]
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="axonn", choices=["axonn", "reference"])
    ap.add_argument("--grid", default=None, help="gx,gy,gz,gd (default: per-N plan, see PRIMARY)")
    ap.add_argument("--model", default=None, choices=sorted(HIDDEN))
    ap.add_argument("--tokens", type=int, default=None, help="global m (default: per-N plan)")
    ap.add_argument("--tokens-per-gpu", type=int, default=None,
                    help="global m = tokens-per-gpu x N (the data-parallel weak-scaling family)")
    ap.add_argument("--phase", default=None, choices=["A", "B"])
    ap.add_argument("--chunks", type=int, default=4, help="forward AR pipelining chunks")
    ap.add_argument("--gemm-sms", type=int, default=0, help="SM budget of the GEMM grid (0 = all)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sub", action="store_true", help="skip the sub-records (C4a/C4b/C5, DP)")
    ap.add_argument("--sub-steps", type=int, default=20, help="timed steps of each sub-record")
    ap.add_argument("--graph", action="store_true",
                    help="capture one step in a CUDA graph and time its replays")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--soak", type=float, default=0.0,
                    help="untimed seconds of steps before timing (settles the power-capped clock)")
    ap.add_argument("--w-init", default="scaled", choices=["scaled", "uniform"],
                    help="weights U(+-sqrt(3/k)) (random init) or U(-1,1)")
    ap.add_argument("--blocks", type=int, default=1,
                    help="GPT blocks per step, chained fc2 -> next QKV (SURVEY.md §8(f) f-1)")
    ap.add_argument("--grad-f32", action="store_true",
                    help="AXONN_BF16_GRADF32: dW in fp32, RS_z / data-parallel sums in fp32 (R17)")
    ap.add_argument("--recompute", action="store_true",
                    help="activation checkpointing (PAPER.md:722-723): each layer's forward re-runs "
                         "before its backward; flops counted 8mkn as Narayanan et al.'s formula does")
    ap.add_argument("--trace", default=None,
                    help="write a Chrome-trace JSON of the per-layer phases (N > 1) to this path")
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
    if world > 1:
        ax.bootstrap_from_torch_distributed(local)
    if args.gemm_sms:
        ax.axonn_set_gemm_sms(args.gemm_sms)
    c = Ctx()
    c.ax, c.torch, c.dist, c.args = ax, torch, dist, args
    c.world, c.rank, c.local = world, rank, local
    c.stream = torch.cuda.Stream()

    # the primary workload: the per-N plan, unless overridden
    default = PRIMARY.get(world)
    custom = (args.grid or args.model or args.tokens or args.tokens_per_gpu or args.phase
              or default is None)
    if custom:
        model = args.model or "5B"
        m = (args.tokens if args.tokens else (args.tokens_per_gpu or 16384) * world)
        phase = args.phase or "A"
        spec = dict(label="custom", model=model, m=m, phase=phase)
        if args.grid:
            spec["grid"] = tuple(int(x) for x in args.grid.split(","))
        elif world == 1:
            spec["grid"] = (1, 1, 1, 1)
        else:
            spec["grid"], spec["grid_source"] = model_top1(ax, block_layers(HIDDEN[model], m, phase), world)
    else:
        spec = dict(default)
    spec["blocks"] = args.blocks
    spec["chain"] = not args.no_chain
    prim = run_config(c, spec, args.steps, args.warmup, not args.no_e2e, True)

    subs = []
    if not args.no_sub and not custom and world > 1:
        plan = [dict(s) for s in SUB.get(world, [])]
        # the data-parallel weak-scaling line: 5B block, 16384 tokens per GPU,
        # the model's top-ranked grid (round-1 headline, kept as a sub-record)
        dp_layers = block_layers(HIDDEN["5B"], 16384 * world)
        g, src = model_top1(ax, dp_layers, world)
        plan.append(dict(label="data-parallel weak scaling (5B, 16384 tokens/GPU, model top-1)",
                         model="5B", m=16384 * world, grid=g, phase="A", grid_source=src))
        for sp in plan:
            sp["blocks"], sp["chain"], sp["primary"] = 1, not args.no_chain, False
            r = run_config(c, sp, args.sub_steps, max(3, args.warmup), False, True)
            subs.append({k: r[k] for k in ("label", "value", "per_gpu_tflops", "ms_per_step",
                                           "steps", "config", "overlap", "clocks",
                                           "gpu_launches", "fused_axes")})

    peaks, peaks_src = read_peaks()
    gemm_n, gemm_ms, gemm_flops = prim["gemm"]["launches"], prim["gemm"]["ms"], prim["gemm"]["flops"]
    achieved = gemm_flops / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else 0.0
    sustained = float(peaks.get("bf16_tflops_sustained", FALLBACK_PEAKS["bf16_tflops_sustained"]))
    burst = float(peaks.get("bf16_tflops", FALLBACK_PEAKS["bf16_tflops"]))
    # The measured peaks are cuBLAS at burst clocks (best of 10) and back to
    # back for 4 s (sustained, power-capped).  The timed region takes the
    # peak measured the way it runs: a window of >= 4 s (or one whose median
    # SM clock sat well below the maximum for >= 1 s) is in the sustained
    # regime; shorter windows, which start from a rested power state, take
    # the burst peak — never a denominator the window could exceed.
    clk = prim["clocks"]
    window_s = prim["ms_per_step"] * args.steps / 1e3
    below_max = bool(clk.get("sm_mhz") and clk.get("sm_max_mhz")
                     and clk["sm_mhz"] < 0.97 * clk["sm_max_mhz"])
    at_max = not (window_s >= 4.0 or (window_s >= 1.0 and below_max))
    peak = burst if at_max else sustained
    traffic = None
    tf = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    if os.path.exists(tf):
        traffic = json.load(open(tf)).get("dram_bytes_per_launch")

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, thr, desc = oracle_sample(HIDDEN[spec["model"]], 2048, 10.0)
        cpu = {"value": v, "unit": "TFLOP/s", "cores": thr, "kind": "oracle", "sample": desc}
        try:
            tv, tthr = torch_cpu_bf16_sample(HIDDEN[spec["model"]], 2048, 5.0)
            cpu["torch_cpu_bf16"] = {"value": tv, "unit": "TFLOP/s", "threads": tthr,
                                     "sample": "torch CPU bf16 matmuls of the same block products, "
                                               "2048 token rows"}
        except Exception as e:  # pragma: no cover
            cpu["torch_cpu_bf16"] = {"error": str(e)[:200]}

    if rank == 0:
        value = prim["value"]
        out = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": prim["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": ("synthetic (inputs uniform(-1,1) bf16, weights "
                     + ("U(+-sqrt(3/k)) random init" if args.w_init == "scaled" else "U(-1,1)")
                     + ", device-generated, seeded)"),
            "config": {**prim["config"], "label": prim["label"]},
            "per_gpu_tflops": value / world,
            "frac_of_peak": {"advertised_2250": value / world / 2250.0,
                             "measured_burst": value / world / burst,
                             "measured_sustained": value / world / sustained, "peaks": peaks_src},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak,
                         "unit": "TFLOP/s", "frac": achieved / peak if peak else None,
                         "traffic": traffic,
                         "kernel": "gemm_bf16_tcgen05_pair (all NN/NT/TN launches of the timed "
                                   "region; achieved = sum 2MNK / sum event time on the launching "
                                   "stream)",
                         "peak_kind": (f"bf16_tflops (burst: a {window_s:.2f} s window)" if at_max else
                                       f"bf16_tflops_sustained (a {window_s:.2f} s window in the "
                                       "power-capped regime)")
                                      + f", {peaks_src}",
                         "frac_of_burst": achieved / burst if burst else None,
                         "frac_of_sustained": achieved / sustained if sustained else None,
                         "gemm_launches": gemm_n, "gemm_ms_per_step": gemm_ms / args.steps},
            "cuda_graph": bool(args.graph),
            "gpu_launches": prim["gpu_launches"],
            "overlap": prim["overlap"],
            "fused_axes": prim["fused_axes"],
            "clocks": prim["clocks"],
            "e2e": prim["e2e"],
            "cpu_baseline": cpu,
            "sub_records": subs or None,
        }
        emit(out)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
