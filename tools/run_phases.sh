#!/bin/bash
o=gpurun_out/ph; mkdir -p $o
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
timeout 600 bash -c "$(declare -f tr); tr 4 29701 tools/layer_phases.py --model 20B --tokens 8192 --grid 2,2,1,1 --out $o/c3proxy_N4.json" > $o/c3proxy_N4.log 2>&1
timeout 600 bash -c "$(declare -f tr); tr 2 29702 tools/layer_phases.py --model 20B --tokens 4096 --grid 2,1,1,1 --out $o/n2_2111.json" > $o/n2_2111.log 2>&1
timeout 600 bash -c "$(declare -f tr); tr 2 29703 tools/layer_phases.py --model 20B --tokens 8192 --grid 1,2,1,1 --out $o/n2_1211.json" > $o/n2_1211.log 2>&1
