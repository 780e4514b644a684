#!/bin/bash
# 2-rank modes per layer (20B, (1,2,1,1), m = 8192): exchange + local sum vs
# multimem.red at every K (AXONN_RED_MIN_K=0), ranks aligned per call.
o=gpurun_out/ra; mkdir -p $o
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
for v in "x0:AXONN_XSUM=0" "red:AXONN_RED_MIN_K=0" "x0b:AXONN_XSUM=0" "redb:AXONN_RED_MIN_K=0"; do
  name=${v%%:*}; env=${v#*:}
  env $env timeout 600 bash -c "$(declare -f tr); tr 2 29761 tools/layer_phases.py --model 20B --tokens 8192 --grid 1,2,1,1 --out $o/$name.json" > $o/$name.log 2>&1
done
python - $o <<'PY'
import json, glob, os, sys
for f in sorted(glob.glob(os.path.join(sys.argv[1], "*.json"))):
    print("==", os.path.basename(f))
    for r in json.load(open(f)):
        print(f"{r['layer']:5s} fwd {r['fwd_ms']:.3f} (gemm {r['fwd_gemm_ms']:.3f}, alone {r['gemm_alone_ms']:.3f}, post {r['fwd_ms']-r['fwd_gemm_ms']:.3f})  bwd {r['bwd_ms']:.3f} (gemm {r['bwd_gemm_ms']:.3f}, alone {r['bwd_alone_ms']:.3f}, post {r['bwd_ms']-r['bwd_gemm_ms']:.3f})")
PY
