#!/bin/bash
# kXSum cost breakdown on the C3-proxy layers (2 ranks, the Y axis of 2):
# the full mode, sums all left to the sweep (bit 0), and no fence (bit 1,
# timing only), against the exchange + local sum.
o=gpurun_out/xo; mkdir -p $o
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
for v in "x0:AXONN_XSUM=0" "x1:AXONN_XSUM=1" "x1o1:AXONN_XSUM=1 AXONN_XSUM_OPT=1" "x1o3:AXONN_XSUM=1 AXONN_XSUM_OPT=3" "x1o2:AXONN_XSUM=1 AXONN_XSUM_OPT=2" "x0nopdl:AXONN_XSUM=0 AXONN_PDL=0"; do
  name=${v%%:*}; env=${v#*:}
  env $env timeout 600 bash -c "$(declare -f tr); tr 2 29741 tools/layer_phases.py --model 20B --tokens 8192 --grid 1,2,1,1 --out $o/$name.json" > $o/$name.log 2>&1
done
python - $o <<'PY'
import json, glob, os, sys
for f in sorted(glob.glob(os.path.join(sys.argv[1], "*.json"))):
    print("==", os.path.basename(f))
    for r in json.load(open(f)):
        print(f"{r['layer']:5s} fwd {r['fwd_ms']:.3f} (gemm {r['fwd_gemm_ms']:.3f}, alone {r['gemm_alone_ms']:.3f}, post {r['fwd_ms']-r['fwd_gemm_ms']:.3f})  bwd {r['bwd_ms']:.3f} (gemm {r['bwd_gemm_ms']:.3f}, alone {r['bwd_alone_ms']:.3f}, post {r['bwd_ms']-r['bwd_gemm_ms']:.3f})")
PY
