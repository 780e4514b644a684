#!/bin/bash
# kRedPair default: loopback + 2/4-GPU parity, then the N=2 / N=4 bench lines
o=gpurun_out/f5; mkdir -p $o
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
timeout 900 python -m pytest tests/test_gpu_loopback.py -q -x > $o/pt_lb.log 2>&1; echo EXIT=$? >> $o/pt_lb.log
grep -q "EXIT=0" $o/pt_lb.log || exit 1
timeout 2700 python -m pytest tests/test_gpu_multi.py -q -rs > $o/pt_multi.log 2>&1; echo EXIT=$? >> $o/pt_multi.log
for n in 2 4; do
  timeout 900 bash -c "$(declare -f tr); tr $n 2990$n bench.py --gpus $n --steps 20 --warmup 5 --trace $o/trace_N$n.json" > $o/bench_N$n.json 2> $o/bench_N$n.err
done
timeout 600 bash -c "$(declare -f tr); tr 4 29911 tools/layer_phases.py --model 20B --tokens 8192 --grid 2,2,1,1 --out $o/phases_c3proxy_N4.json" > $o/phases.log 2>&1
