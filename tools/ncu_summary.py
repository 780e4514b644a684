"""Summarise an ncu report (raw page) of the GEMM launches into a markdown table
and the per-launch DRAM traffic file bench.py reports as roofline.traffic.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_gemm_ncu.md
"""
import csv
import io
import json
import os
import subprocess
import sys

M = {
    "time_ms": ("gpu__time_duration.sum", 1e-6),       # ns -> ms (unit checked below)
    "dram_rd": ("dram__bytes_read.sum", 1.0),
    "dram_wr": ("dram__bytes_write.sum", 1.0),
    "tc_pct": ("sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed", 1.0),
    "hmma_pipe_pct": ("sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "sm_ghz": ("sm__cycles_elapsed.avg.per_second", 1.0),
    "l2_rd_sect": ("lts__t_sectors_srcunit_tex_op_read.sum", 1.0),
    "regs": ("launch__registers_per_thread", 1.0),
}
SCALE = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "hz": 1e-9, "Khz": 1e-6, "Mhz": 1e-3, "Ghz": 1.0}


SHAPE_NAMES = [f"{l}_{p}" for l in ("qkv", "proj", "fc1", "fc2") for p in ("fwd", "dI", "dW")]


def main(rep, out_md, traffic_json=None, pick=None):
    """pick="odd": keep launches 1, 3, 5, ... (tools/gemm_shapes.py --reps 1
    --rounds 1 runs each C2 shape twice: warm-up, then the measured launch)."""
    if rep.endswith(".csv"):  # an exported raw page (ncu -i REP --page raw --csv)
        raw = open(rep).read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    recs = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0].replace("void ", ""),
             "grid": r[h.index("Grid Size")], "block": r[h.index("Block Size")]}
        for key, (col, _) in M.items():
            if col in h:
                i = h.index(col)
                v = float(r[i].replace(",", "")) if r[i] not in ("", "n/a") else float("nan")
                d[key] = v * SCALE.get(units[i], 1.0)
        recs.append(d)
    if pick == "odd":
        recs = recs[1::2]
        for d, name in zip(recs, SHAPE_NAMES):
            d["kernel"] = name + " " + d["kernel"].split("::")[-1]
    lines = ["| # | kernel | grid | time ms | DRAM read GB | DRAM write GB | UTCHMMA % peak | hmma pipe % active | SM GHz |",
             "|---|---|---|---|---|---|---|---|---|"]
    for i, d in enumerate(recs):
        lines.append(f"| {i} | {d['kernel'][-40:]} | {d['grid']} | {d.get('time_ms', 0):.3f} | "
                     f"{d.get('dram_rd', 0) / 1e9:.3f} | {d.get('dram_wr', 0) / 1e9:.3f} | "
                     f"{d.get('tc_pct', 0):.1f} | {d.get('hmma_pipe_pct', 0):.1f} | {d.get('sm_ghz', 0):.3f} |")
    n = len(recs)
    tot_t = sum(d.get("time_ms", 0) for d in recs)
    tot_b = sum(d.get("dram_rd", 0) + d.get("dram_wr", 0) for d in recs)
    wavg_tc = sum(d.get("tc_pct", 0) * d.get("time_ms", 0) for d in recs) / max(tot_t, 1e-12)
    lines += ["", f"launches: {n}; total {tot_t:.3f} ms; DRAM read+write {tot_b / 1e9:.3f} GB "
              f"({tot_b / max(n, 1) / 1e9:.3f} GB per launch); time-weighted UTCHMMA % of peak: {wavg_tc:.1f}"]
    open(out_md, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if traffic_json:
        json.dump({"source": os.path.basename(rep), "launches": n,
                   "dram_bytes_per_launch": tot_b / max(n, 1),
                   "note": "dram__bytes_read.sum + dram__bytes_write.sum averaged over the GEMM launches "
                           "of one C2 step (ncu --set full, cold-cache replays)"},
                  open(traffic_json, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 and sys.argv[3] != "-" else None,
         sys.argv[4] if len(sys.argv) > 4 else None)
