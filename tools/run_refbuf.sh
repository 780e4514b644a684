#!/bin/bash
o=gpurun_out/rb; mkdir -p $o
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
for rep in 1 2; do for v in s0 s1; do
  BENCH_REF_OWNBUF=${v#s} AXONN_PREZERO=0 timeout 400 bash -c "$(declare -f tr); tr 2 29831 bench.py --gpus 2 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-sub" > $o/b_${v}_$rep.json 2> $o/b_${v}_$rep.err
done; done
python - $o <<'PY'
import json, glob, os, sys
for f in sorted(glob.glob(os.path.join(sys.argv[1], "b_*.json"))):
    d = json.loads(open(f).read().strip().splitlines()[-1]); ov = d.get("overlap") or {}
    print(os.path.basename(f), round(d["per_gpu_tflops"], 1), "ms", round(d["ms_per_step"], 3), "gemm_only", round(ov.get("t_gemm_only_ms", 0), 3), "exposed", round(ov.get("exposed_comm_frac", 0), 4))
PY
