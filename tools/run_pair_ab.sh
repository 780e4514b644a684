#!/bin/bash
# 2-rank fused all-reduce modes on the tensor-parallel proxies: exchange +
# local sum (AXONN_PAIRSUM=0), pair-sum push (1), pair-sum pull (2).
o=gpurun_out/pab; mkdir -p $o
nvidia-smi nvlink -gt d -i 0 > $o/smi_nvlink_gt.txt 2>&1; nvidia-smi nvlink -h >> $o/smi_nvlink_gt.txt 2>&1
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
timeout 900 bash -c "$(declare -f tr); tr 2 29611 tests/mp_worker.py" > $o/mp2.log 2>&1; echo EXIT=$? >> $o/mp2.log
for rep in 1 2; do for mode in 0 1 2; do for n in 4 2; do
  AXONN_PAIRSUM=$mode timeout 300 bash -c "$(declare -f tr); tr $n 2962$n bench.py --gpus $n --steps 30 --warmup 5 --no-sub --no-cpu-baseline --no-e2e" > $o/b_N${n}_m${mode}_$rep.json 2> $o/b_N${n}_m${mode}_$rep.err
done; done; done
for mode in 0 2; do
AXONN_PAIRSUM=$mode timeout 300 bash -c "$(declare -f tr); tr 2 29631 tools/nvlink_counters.py --out $o/nvlink_m$mode.json" > $o/nvl_m$mode.log 2>&1
done
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
