#!/bin/bash
# raster band A/B on the 12 C2 launches (AXONN_GROUP_M, in 512-row tiles; default 8)
o=gpurun_out/gm; mkdir -p $o
for rep in 1 2 3; do
  for v in "g8:AXONN_GROUP_M=8" "g4:AXONN_GROUP_M=4" "g16:AXONN_GROUP_M=16" "g6:AXONN_GROUP_M=6"; do
    name=${v%%:*}; env=${v#*:}
    env $env AB_LABEL=$name timeout 300 python tools/gemm_shapes.py --reps 10 --rounds 2 --no-cublas > $o/${name}_$rep.json 2> $o/${name}_$rep.err
  done
done
python - $o <<'PY'
import json, glob, os, sys, collections
agg = collections.defaultdict(lambda: collections.defaultdict(list))
for f in sorted(glob.glob(os.path.join(sys.argv[1], "*.json"))):
    d = json.load(open(f)); name = os.path.basename(f).rsplit("_", 1)[0]
    for k, v in d["shapes"].items():
        agg[k][name].append(round(v["axonn_tflops"]))
    agg["SUM_ms"][name].append(round(d["sum_axonn_ms"], 3))
for k, v in agg.items():
    print(k, dict(v))
PY
