#!/bin/bash
o=gpurun_out/f9; mkdir -p $o
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
timeout 240 bash -c "$(declare -f tr); tr 2 29971 bench.py --gpus 2 --blocks 2 --steps 10 --warmup 3 --no-sub --no-cpu-baseline --no-e2e" > $o/bench_N2_blocks2.json 2> $o/bench_N2_blocks2.err
timeout 240 bash -c "$(declare -f tr); tr 2 29972 tools/layer_phases.py --model 20B --tokens 8192 --grid 1,2,1,1 --out $o/phases_1211.json" > $o/phases.log 2>&1
