#!/bin/bash
o=gpurun_out/pz; mkdir -p $o
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
timeout 1200 bash -c "$(declare -f tr); tr 2 29821 tests/mp_worker.py" > $o/mp2.log 2>&1; echo EXIT=$? >> $o/mp2.log
grep -q "MP_OK" $o/mp2.log || exit 1
for rep in 1 2; do for v in p1 p0; do
  AXONN_PREZERO=${v#p} timeout 400 bash -c "$(declare -f tr); tr 2 29822 bench.py --gpus 2 --grid 1,2,1,1 --model 20B --tokens 8192 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e" > $o/b_${v}_$rep.json 2> $o/b_${v}_$rep.err
done; done
python - $o <<'PY'
import json, glob, os, sys
for f in sorted(glob.glob(os.path.join(sys.argv[1], "b_*.json"))):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        ov = d.get("overlap") or {}
        print(os.path.basename(f), round(d["per_gpu_tflops"], 1), "ms", round(d["ms_per_step"], 3), "exposed", round(ov.get("exposed_comm_frac", 0), 4))
    except Exception as e:
        print(os.path.basename(f), "failed", e)
PY
