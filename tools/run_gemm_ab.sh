#!/bin/bash
# GEMM kernel changes: parity first, then same-box A/B and a bench line.
o=gpurun_out/gab; mkdir -p $o
timeout 1200 python -m pytest tests/test_gpu_gemm.py -q -x > $o/pt_gemm.log 2>&1; echo EXIT=$? >> $o/pt_gemm.log
grep -q "EXIT=0" $o/pt_gemm.log || exit 1
bash tools/ab_gemm.sh $o/ab "base:AXONN_SK=0 AXONN_MT2_DEEP=0" "deep:AXONN_SK=0" "sk:AXONN_MT2_DEEP=0" "both:AXONN_SK=1" > $o/ab.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-sub > $o/bench.json 2> $o/bench.err
AXONN_SK=0 AXONN_MT2_DEEP=0 timeout 300 python bench.py --steps 20 --warmup 5 --no-sub --no-cpu-baseline > $o/bench_base.json 2>> $o/bench.err
timeout 300 python bench.py --steps 20 --warmup 5 --no-sub --no-cpu-baseline > $o/bench2.json 2>> $o/bench.err
timeout 1500 python -m pytest tests/test_gpu_loopback.py tests/test_gpu_fc.py -q -x > $o/pt_lb.log 2>&1; echo EXIT=$? >> $o/pt_lb.log
