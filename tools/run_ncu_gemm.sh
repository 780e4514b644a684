#!/bin/bash
# ncu --set full of the 12 C2 local products (one launch each after one warm-up
# launch), then the bench launch list.  One ncu tool per gpurun call.
o=gpurun_out/ncu2; mkdir -p $o
cmd="python tools/gemm_shapes.py --reps 1 --rounds 1 --no-cublas"
$cmd > $o/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -c 24 -o $o/prof $cmd > $o/ncu_full.log 2>&1
echo NCU_EXIT=$? >> $o/ncu_full.log
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-sub > $o/bplain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-sub > $o/ncu_launches.log 2>&1
echo NCU2_EXIT=$? >> $o/ncu_launches.log
