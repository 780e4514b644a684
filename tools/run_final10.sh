#!/bin/bash
o=gpurun_out/f10; mkdir -p $o
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
timeout 600 bash -c "$(declare -f tr); tr 2 29991 tests/mp_worker.py" > $o/mp2.log 2>&1; echo EXIT=$? >> $o/mp2.log
