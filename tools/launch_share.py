"""Per-kernel share table of an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python tools/launch_share.py gpurun_out/launches.csv profiles/r02_launches.md "<command>"
"""
import collections
import csv
import sys


def main(path, out, cmd):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, rows = rows[0], rows[1:]
    ki, ui, vi = hdr.index("Kernel Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        name = r[ki][:100]
        tot[name] += float(r[vi].replace(",", "")) * scale[r[ui]]
        cnt[name] += 1
    allt = sum(tot.values())
    lines = [f"ncu --metrics gpu__time_duration.sum --clock-control none launch list of `{cmd}`.",
             "Cold-cache, serialised per-launch times: compare shares, not absolute times.", "",
             "| kernel | launches | total ms | share % |", "|---|---|---|---|"]
    for name, t in sorted(tot.items(), key=lambda kv: -kv[1]):
        lines.append(f"| {name.replace('|', '/')} | {cnt[name]} | {t:.3f} | {100 * t / allt:.1f} |")
    lines.append(f"| **total** | {sum(cnt.values())} | {allt:.3f} | 100 |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "bench.py")
