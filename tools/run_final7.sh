#!/bin/bash
o=gpurun_out/f7; mkdir -p $o
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
timeout 600 bash -c "$(declare -f tr); tr 2 29962 bench.py --gpus 2 --steps 20 --warmup 5 --trace $o/trace_N2.json" > $o/bench_N2.json 2> $o/bench_N2.err
timeout 900 bash -c "$(declare -f tr); tr 4 29964 bench.py --gpus 4 --steps 20 --warmup 5 --trace $o/trace_N4.json" > $o/bench_N4.json 2> $o/bench_N4.err
