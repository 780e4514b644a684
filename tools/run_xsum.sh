#!/bin/bash
# kXSum: parity on one GPU (loopback) and two (mp_worker), then A/B on the
# tensor-parallel proxies: in-GEMM exchange sum at every K (AXONN_XSUM=1),
# below the multimem.red threshold only (2), off (0: exchange + local sum).
o=gpurun_out/xs; mkdir -p $o
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
timeout 900 python -m pytest tests/test_gpu_loopback.py -q -x > $o/pt_lb.log 2>&1; echo EXIT=$? >> $o/pt_lb.log
grep -q "EXIT=0" $o/pt_lb.log || exit 1
timeout 900 bash -c "$(declare -f tr); tr 2 29711 tests/mp_worker.py" > $o/mp2.log 2>&1; echo EXIT=$? >> $o/mp2.log
grep -q "MP_OK" $o/mp2.log || exit 1
for rep in 1 2; do for mode in 1 2 0; do for n in 4 2; do
  AXONN_XSUM=$mode timeout 300 bash -c "$(declare -f tr); tr $n 2972$n bench.py --gpus $n --steps 30 --warmup 5 --no-sub --no-cpu-baseline --no-e2e" > $o/b_N${n}_x${mode}_$rep.json 2> $o/b_N${n}_x${mode}_$rep.err
done; done; done
AXONN_XSUM=1 timeout 600 bash -c "$(declare -f tr); tr 4 29731 tools/layer_phases.py --model 20B --tokens 8192 --grid 2,2,1,1 --out $o/ph_c3proxy_x1.json" > $o/ph_x1.log 2>&1
python - $o <<'PY'
import json, glob, os, sys
for f in sorted(glob.glob(os.path.join(sys.argv[1], "b_N*.json"))):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        ov = d.get("overlap") or {}
        print(os.path.basename(f), round(d["per_gpu_tflops"], 1), "exposed", round(ov.get("exposed_comm_frac", 0), 4),
              {k: round(v["exposed_frac"], 3) for k, v in ov.get("per_layer", {}).items() if "exposed_frac" in v})
    except Exception as e:
        print(os.path.basename(f), "failed", e)
PY
