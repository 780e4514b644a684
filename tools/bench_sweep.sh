#!/bin/bash
# Run bench.py for a list of argument sets on N GPUs; print one summary line each.
# usage: tools/bench_sweep.sh N "args1" "args2" ...
N=$1; shift
i=0
for A in "$@"; do
  i=$((i+1))
  if [ "$N" = "1" ]; then
    timeout 400 python bench.py --gpus 1 $A > gpurun_out/sw_$i.out 2> gpurun_out/sw_$i.err
  else
    timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 \
      --master-port=$((29700 + i)) bench.py --gpus $N $A > gpurun_out/sw_$i.out 2> gpurun_out/sw_$i.err
  fi
  python - "$A" gpurun_out/sw_$i.out <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
except Exception as e:
    print(f"{sys.argv[1]:40s} FAILED {e}"); sys.exit(0)
o = d.get("overlap") or {}
print(f"{sys.argv[1]:40s} grid={d['config']['grid']} total={d['value']:.1f} perGPU={d['per_gpu_tflops']:.1f} "
      f"ms={d['ms_per_step']:.3f} gemm_ms={o.get('t_gemm_only_ms', 0):.3f} exposed={o.get('exposed_comm_frac', 0):.4f} "
      f"gemmTF={d['roofline']['achieved']:.1f} mhz={d['clocks']['sm_mhz']} e2e={(d.get('e2e') or {}).get('value', 0):.1f}")
PY
done
