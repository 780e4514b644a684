#!/bin/bash
# driver-like 1-GPU validation: the whole -m gpu suite, smoke, the N=1 bench,
# the reference arm, and the bench's ncu launch list
o=gpurun_out/f1; mkdir -p $o
timeout 1800 python -m pytest tests -m gpu -q -rs > $o/pt.log 2>&1; echo EXIT=$? >> $o/pt.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE_OK')" > $o/smoke.log 2>&1
timeout 400 python bench.py --steps 20 --warmup 5 > $o/bench.json 2> $o/bench.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > $o/ref.json 2> $o/ref.err
timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-sub > $o/bplain.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-sub > $o/ncu.log 2>&1
echo NCU_EXIT=$? >> $o/ncu.log
