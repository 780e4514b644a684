#!/bin/bash
# Same-box A/B of GEMM kernel configurations on the 12 C2 launch shapes
# (tools/gemm_shapes.py, burst windows), alternating.  Usage:
#   tools/ab_gemm.sh OUTDIR "name:ENV=V ENV2=V" "name2:ENV=V" ...
out=${1:-gpurun_out/abg}; shift
mkdir -p $out
for rep in 1 2; do
  for cfg in "$@"; do
    name=${cfg%%:*}; env=${cfg#*:}
    cub=--no-cublas; [ $rep = 1 ] && [ "$cfg" = "$1" ] && cub=
    env $env AB_LABEL=$name timeout 300 python tools/gemm_shapes.py --reps 10 --rounds 3 $cub > $out/${name}_$rep.json 2> $out/${name}_$rep.err
  done
done
python - "$out" <<'PY'
import json, glob, sys, os
rows = {}
for f in sorted(glob.glob(os.path.join(sys.argv[1], "*.json"))):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(os.path.basename(f), "failed", e); continue
    print(f"{os.path.basename(f):28s} sum {d['sum_axonn_ms']:.3f} ms" +
          (f"  cublas {d['sum_cublas_ms']:.3f}" if 'sum_cublas_ms' in d else ""))
    for k, v in d["shapes"].items():
        rows.setdefault(k, {})[os.path.basename(f)[:-5]] = v["axonn_tflops"]
        if "cublas_tflops" in v: rows[k]["cublas"] = v["cublas_tflops"]
cols = sorted({c for r in rows.values() for c in r})
print("shape," + ",".join(cols))
for k, r in rows.items():
    print(k + "," + ",".join(f"{r.get(c, 0):.0f}" for c in cols))
PY
