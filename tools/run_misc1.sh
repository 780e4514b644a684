#!/bin/bash
o=gpurun_out/m1; mkdir -p $o
python tools/pcie_probe.py > $o/pcie.json 2>&1
python tools/cublas_compare.py --seconds 0.3 --rounds 3 > $o/cublas_short.txt 2>&1
python tools/cublas_compare.py --seconds 4 --rounds 2 > $o/cublas_long.txt 2>&1
python bench.py --steps 20 --warmup 5 > $o/bench.json 2> $o/bench.err
AXONN_PDL=0 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $o/bench_nopdl.json 2>> $o/bench.err
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $o/bench2.json 2>> $o/bench.err
