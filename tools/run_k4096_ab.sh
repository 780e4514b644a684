#!/bin/bash
# K=4096 launches of C2: 512x256 with 4 stages / 1 staging box (default) vs
# 3 stages / 2 boxes vs 256x256 (MT=1, double-buffered accumulators).
o=gpurun_out/k4; mkdir -p $o
sh="qkv_fwd,proj_fwd,proj_dI,fc1_fwd,fc2_dI"
for rep in 1 2 3; do
  for v in "deep:AXONN_SK=1" "deep0:AXONN_MT2_DEEP=0" "mt1:AXONN_MT2_MIN_K=8192"; do
    name=${v%%:*}; env=${v#*:}
    env $env AB_LABEL=$name timeout 300 python tools/gemm_shapes.py --reps 20 --rounds 3 --no-cublas --only $sh > $o/${name}_$rep.json 2> $o/${name}_$rep.err
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
