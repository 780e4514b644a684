#!/usr/bin/env python
"""NVLink bytes and rates of the fused collectives, from the GPU's own NVLink
counters (NVML field values), per launch — run under torchrun with 2 ranks:

    python -m torch.distributed.run --nproc-per-node 2 tools/nvlink_counters.py \
        --out profiles/r02_nvlink_counters.json

For one FC layer per collective site (Alg. 1 line 4 forward all-reduce, line
12 backward all-reduce, lines 2/14 AG_z / RS_z, the data-parallel sum of
PAPER.md:313-317) on the 2-rank grid that isolates it, each rank reads its
NVLink TX/RX data counters (NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX/RX, KiB,
summed over links) around `iters` calls, with the calls timed by CUDA events
on the launching stream.  Reported per call and rank: bytes sent / received,
the closed-form bytes of Eqs. 1-5 for that collective (ring volumes), and
the achieved GB/s over the call's device time.  Shapes: the GPT-20B block's
QKV layer at m = 8192 (K = 7168 / 2 = 3584 < 8192: the short-K 2-rank mode)
and its fc2 layer (K >= 8192: multimem.red), so both 2-rank fused modes show.
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

# (tx, rx, bytes per unit): NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX/_RX (KiB),
# NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES / _RCV_BYTES (bytes), tried in order
FIELDS = [(138, 139, 1024), (202, 204, 1)]


def nvml_handle(local):
    import pynvml
    pynvml.nvmlInit()
    global _SMI_BUS
    pr = torch.cuda.get_device_properties(local)
    _SMI_BUS = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
    return pynvml.nvmlDeviceGetHandleByPciBusId(_SMI_BUS)


_FIELD = None


_SMI_BUS = None
_UNITS = {"B": 1, "KiB": 1024, "MiB": 1024 ** 2, "GiB": 1024 ** 3, "TiB": 1024 ** 4}


def smi_counters():
    """(tx, rx) data bytes summed over this GPU's links from
    `nvidia-smi nvlink -gt d -i <bus id>` (the driver's per-link data
    throughput counters), or None."""
    import re
    import subprocess
    try:
        out = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", _SMI_BUS],
                             capture_output=True, text=True, timeout=30).stdout
    except Exception:
        return None
    tot = [0, 0]
    hit = False
    for key, i in (("Tx", 0), ("Rx", 1)):
        for v, u in re.findall(rf"Data {key}:\s*([0-9]+)\s*([KMGT]?i?B)", out):
            tot[i] += int(v) * _UNITS.get(u, 1)
            hit = True
    return tuple(tot) if hit else None


def counters(h, nlinks=18):
    """(tx, rx) bytes summed over links (or the device total); None if no field
    is available.  The first field set and scope that answers is kept; the
    nvidia-smi per-link counters are the fallback."""
    import pynvml
    global _FIELD
    if _FIELD == "smi":
        return smi_counters()
    cands = [_FIELD] if _FIELD else [(f, sc) for f in FIELDS for sc in ("links", "all")]
    for (tx, rx, unit), scope in cands:
        scopes = range(nlinks) if scope == "links" else [0xFFFFFFFF]
        tot, ok = [0, 0], False
        for link in scopes:
            try:
                vals = pynvml.nvmlDeviceGetFieldValues(h, [(tx, link), (rx, link)])
            except Exception:
                continue
            for i, v in enumerate(vals):
                if v.nvmlReturn == 0:
                    ok = True
                    tot[i] += int(v.value.ullVal) * unit
        if ok:
            _FIELD = ((tx, rx, unit), scope)
            return tuple(tot)
    c = smi_counters()
    if c is not None:
        _FIELD = "smi"
    return c


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "nvlink_counters.json"))
    args = ap.parse_args()
    local = int(os.environ["LOCAL_RANK"])
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    assert world == 2, "run with 2 ranks"
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ax.bootstrap_from_torch_distributed(local)
    nv = nvml_handle(local)
    h7 = 7168
    # (site, grid, layer (m, k, n, transposed), phase to time)
    sites = [("AR_y fwd, K=3584 (line 4)", (1, 2, 1, 1), (8192, h7, 3 * h7, False), "fwd"),
             ("AR_y fwd, K=14336 (line 4)", (1, 2, 1, 1), (8192, 4 * h7, h7, False), "fwd"),
             ("AR_x bwd, K=10752 (line 12)", (2, 1, 1, 1), (8192, h7, 3 * h7, False), "bwd"),
             ("AR_x bwd, K=3584 (line 12)", (2, 1, 1, 1), (8192, h7, h7, False), "bwd"),
             ("AG_z (line 2, prefetched)", (1, 1, 2, 1), (8192, h7, 3 * h7, False), "ag"),
             ("RS_z (line 14)", (1, 1, 2, 1), (8192, h7, 3 * h7, False), "bwd"),
             ("AR_data (Eq. 5)", (1, 1, 1, 2), (8192, h7, 3 * h7, False), "bwd")]
    s = torch.cuda.current_stream()
    res = []
    for name, cfg, (m, k, n, t), what in sites:
        ax.axonn_grid_init(*cfg)
        hd = ax.axonn_fc_create(m, k, n, t, ax.AXONN_BF16, 1)
        g = ax.axonn_fc_geometry(hd)
        I = torch.empty(g.m_l, g.k_l, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
        W = torch.empty(g.what_len, dtype=torch.bfloat16, device="cuda").uniform_(-0.02, 0.02)
        dO = torch.empty(g.m_l, g.n_l, dtype=torch.bfloat16, device="cuda").uniform_(-1, 1)
        outs = []
        for which, shape in ((0, (g.m_l, g.n_l)), (1, (g.m_l, g.k_l)), (2, (g.what_len,))):
            p = ax.axonn_fc_output_buffer(hd, which)
            outs.append(p if p else torch.empty(shape, dtype=torch.bfloat16, device="cuda"))

        def call():
            if what == "ag":
                ax.axonn_fc_prefetch(hd, W, s)
            if what in ("fwd", "ag", "bwd"):
                ax.axonn_fc_forward(hd, I, W, outs[0], s)
            if what == "bwd":
                ax.axonn_fc_backward(hd, dO, outs[1], outs[2], s)
                ax.axonn_grads_sync(s)

        for _ in range(3):
            call()
        torch.cuda.synchronize()
        dist.barrier()
        # align the two GPUs' starts (a device-side collective right before the timed calls)
        z = torch.zeros(1, device="cuda")
        with torch.cuda.stream(s):
            dist.all_reduce(z)
        # the forward alone, to subtract from "bwd" sites (its collective may be idle there)
        ax.axonn_comm_bytes(reset=True)
        c0 = counters(nv)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(args.iters):
            call()
        e1.record(s)
        torch.cuda.synchronize()
        c1 = counters(nv)
        ms = e0.elapsed_time(e1) / args.iters
        eq = ax.axonn_comm_bytes(reset=True)
        eq = {k: v // args.iters for k, v in eq.items()}
        rec = {"site": name, "grid": list(cfg), "layer": [m, k, n, t], "rank": rank,
               "field": str(_FIELD),
               "ms_per_call": ms, "eqs_1_5_bytes_per_call": eq,
               "fused_axes": {a: ax.axonn_fused_status(a) for a in "xyzd"}}
        if c0 and c1:
            tx, rx = (c1[0] - c0[0]) / args.iters, (c1[1] - c0[1]) / args.iters
            rec.update({"nvlink_tx_bytes_per_call": tx, "nvlink_rx_bytes_per_call": rx,
                        "tx_GBps_over_call": tx / (ms * 1e-3) / 1e9,
                        "tx_over_eqs": tx / max(1, sum(eq.values()))})
        else:
            rec["nvlink_counters"] = "unavailable (NVML field values 138/139, nvidia-smi nvlink -gt d)"
        allr = [None] * world
        dist.all_gather_object(allr, rec)
        if rank == 0:
            res.extend(allr)
            for r in allr:
                print(json.dumps({k: r[k] for k in r if k != "fused_axes"}), flush=True)
        ax.axonn_fc_destroy(hd)
        ax.axonn_grid_finalize()
        dist.barrier()
    if rank == 0:
        os.makedirs(os.path.dirname(args.out), exist_ok=True)
        json.dump(res, open(args.out, "w"), indent=1)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
