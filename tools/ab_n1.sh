#!/bin/bash
# Same-box A/B of GEMM tile configurations at N=1 (C2), short windows (burst
# clocks) and long windows (power-capped), alternating.  Usage: tools/ab_n1.sh OUTDIR
out=${1:-gpurun_out/ab}
mkdir -p $out
for rep in 1 2; do
  for cfg in "default:" "mt2k8192:AXONN_MT2_MIN_K=8192" "mt1:AXONN_PAIR_MT=1"; do
    name=${cfg%%:*}; env=${cfg#*:}
    env $env python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $out/${name}_short_$rep.json 2>/dev/null
    env $env python bench.py --steps 300 --warmup 5 --no-e2e --no-cpu-baseline > $out/${name}_long_$rep.json 2>/dev/null
  done
done
python - "$out" <<'PY'
import json, glob, sys, os
for f in sorted(glob.glob(os.path.join(sys.argv[1], "*.json"))):
    try:
        d = json.load(open(f))
        print(os.path.basename(f), round(d["value"], 1), "gemm", round(d["roofline"]["achieved"], 1),
              "clk", d["clocks"]["sm_mhz"])
    except Exception as e:
        print(os.path.basename(f), "failed", e)
PY
