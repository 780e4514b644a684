#!/bin/bash
o=gpurun_out/la; mkdir -p $o
timeout 120 python tools/gemm_one.py 0 4096 4096 4096 3 > $o/one.log 2>&1; echo EXIT=$? >> $o/one.log
grep -q "EXIT=0" $o/one.log || exit 1
timeout 900 python -m pytest tests/test_gpu_gemm.py -q -x -k "not alternative" > $o/pt.log 2>&1; echo EXIT=$? >> $o/pt.log
grep -q "EXIT=0" $o/pt.log || exit 1
bash tools/run_k4096_ab.sh > $o/k4.txt 2>&1
for rep in 1 2; do
  AB_LABEL=deep timeout 300 python tools/gemm_shapes.py --reps 10 --rounds 3 --no-cublas > $o/all_deep_$rep.json 2>/dev/null
  AXONN_MT2_DEEP=0 AB_LABEL=deep0 timeout 300 python tools/gemm_shapes.py --reps 10 --rounds 3 --no-cublas > $o/all_deep0_$rep.json 2>/dev/null
done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $o/bench.json 2> $o/bench.err
