#!/bin/bash
o=gpurun_out/f6; mkdir -p $o
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
for n in 4 2; do
  timeout 900 bash -c "$(declare -f tr); tr $n 2995$n bench.py --gpus $n --steps 20 --warmup 5 --trace $o/trace_N$n.json" > $o/bench_N$n.json 2> $o/bench_N$n.err
done
