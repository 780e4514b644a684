#!/bin/bash
o=gpurun_out/f8; mkdir -p $o
timeout 1800 python -m pytest tests -m gpu -q -rs > $o/pt.log 2>&1; echo EXIT=$? >> $o/pt.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE_OK')" > $o/smoke.log 2>&1
timeout 400 python bench.py --steps 20 --warmup 5 > $o/bench.json 2> $o/bench.err
