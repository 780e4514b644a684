#!/bin/bash
o=gpurun_out/rp; mkdir -p $o
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
timeout 900 python -m pytest tests/test_gpu_loopback.py -q -x > $o/pt_lb.log 2>&1; echo EXIT=$? >> $o/pt_lb.log
grep -q "EXIT=0" $o/pt_lb.log || exit 1
timeout 1200 bash -c "$(declare -f tr); tr 2 29801 tests/mp_worker.py" > $o/mp2.log 2>&1; echo EXIT=$? >> $o/mp2.log
grep -q "MP_OK" $o/mp2.log || exit 1
for v in r0 r1 r2; do
  AXONN_REDPAIR=${v#r} timeout 600 bash -c "$(declare -f tr); tr 2 29802 tools/layer_phases.py --model 20B --tokens 8192 --grid 1,2,1,1 --out $o/ph_$v.json" > $o/ph_$v.log 2>&1
done
for rep in 1 2; do for v in r0 r1 r2; do
  AXONN_REDPAIR=${v#r} timeout 400 bash -c "$(declare -f tr); tr 4 29803 bench.py --gpus 4 --steps 30 --warmup 5 --no-sub --no-cpu-baseline --no-e2e" > $o/b_N4_${v}_$rep.json 2> $o/b_N4_${v}_$rep.err
done; done
python - $o <<'PY'
import json, glob, os, sys
for f in sorted(glob.glob(os.path.join(sys.argv[1], "ph_*.json"))):
    print("==", os.path.basename(f))
    for r in json.load(open(f)):
        print(f"{r['layer']:5s} fwd {r['fwd_ms']:.3f} (gemm {r['fwd_gemm_ms']:.3f}, post {r['fwd_ms']-r['fwd_gemm_ms']:.3f})  bwd {r['bwd_ms']:.3f} (gemm {r['bwd_gemm_ms']:.3f}, post {r['bwd_ms']-r['bwd_gemm_ms']:.3f})")
for f in sorted(glob.glob(os.path.join(sys.argv[1], "b_N*.json"))):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        ov = d.get("overlap") or {}
        print(os.path.basename(f), round(d["per_gpu_tflops"], 1), "exposed", round(ov.get("exposed_comm_frac", 0), 4))
    except Exception as e:
        print(os.path.basename(f), "failed", e)
PY
