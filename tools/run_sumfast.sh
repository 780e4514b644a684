#!/bin/bash
o=gpurun_out/sf; mkdir -p $o
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
timeout 900 python -m pytest tests/test_gpu_loopback.py -q -x > $o/pt_lb.log 2>&1; echo EXIT=$? >> $o/pt_lb.log
grep -q "EXIT=0" $o/pt_lb.log || exit 1
for rep in 1 2; do for v in f1 f0; do
  AXONN_SUM_FAST=${v#f} timeout 600 bash -c "$(declare -f tr); tr 2 29791 tools/layer_phases.py --model 20B --tokens 8192 --grid 1,2,1,1 --out $o/ph_${v}_$rep.json" > $o/ph_${v}_$rep.log 2>&1
done; done
python - $o <<'PY'
import json, glob, os, sys
for f in sorted(glob.glob(os.path.join(sys.argv[1], "ph_*.json"))):
    print("==", os.path.basename(f))
    for r in json.load(open(f)):
        print(f"{r['layer']:5s} fwd {r['fwd_ms']:.3f} (gemm {r['fwd_gemm_ms']:.3f}, post {r['fwd_ms']-r['fwd_gemm_ms']:.3f})  bwd {r['bwd_ms']:.3f} (gemm {r['bwd_gemm_ms']:.3f}, post {r['bwd_ms']-r['bwd_gemm_ms']:.3f})")
PY
