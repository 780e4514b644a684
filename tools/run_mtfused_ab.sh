#!/bin/bash
# fused short-K launches: 256x256 (default) vs 512x256 tiles (AXONN_PAIR_MT_FUSED=2),
# C3 proxy per-layer phases and N=4 bench
o=gpurun_out/mf; mkdir -p $o
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
for v in "d:AXONN_PAIR_MT_FUSED=0" "m2:AXONN_PAIR_MT_FUSED=2"; do
  name=${v%%:*}; env=${v#*:}
  env $env timeout 600 bash -c "$(declare -f tr); tr 4 29781 tools/layer_phases.py --model 20B --tokens 8192 --grid 2,2,1,1 --out $o/ph_$name.json" > $o/ph_$name.log 2>&1
done
for rep in 1 2; do for v in "d:AXONN_PAIR_MT_FUSED=0" "m2:AXONN_PAIR_MT_FUSED=2"; do
  name=${v%%:*}; env=${v#*:}
  env $env timeout 400 bash -c "$(declare -f tr); tr 4 29782 bench.py --gpus 4 --steps 30 --warmup 5 --no-sub --no-cpu-baseline --no-e2e" > $o/b_N4_${name}_$rep.json 2> $o/b_N4_${name}_$rep.err
done; done
python - $o <<'PY'
import json, glob, os, sys
for f in sorted(glob.glob(os.path.join(sys.argv[1], "ph_*.json"))):
    print("==", os.path.basename(f))
    for r in json.load(open(f)):
        print(f"{r['layer']:5s} fwd {r['fwd_ms']:.3f} (gemm {r['fwd_gemm_ms']:.3f}, post {r['fwd_ms']-r['fwd_gemm_ms']:.3f})  bwd {r['bwd_ms']:.3f} (gemm {r['bwd_gemm_ms']:.3f}, alone {r['bwd_alone_ms']:.3f}, post {r['bwd_ms']-r['bwd_gemm_ms']:.3f})")
for f in sorted(glob.glob(os.path.join(sys.argv[1], "b_N*.json"))):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        ov = d.get("overlap") or {}
        print(os.path.basename(f), round(d["per_gpu_tflops"], 1), "exposed", round(ov.get("exposed_comm_frac", 0), 4))
    except Exception as e:
        print(os.path.basename(f), "failed", e)
PY
