#!/bin/bash
# (1) ncu --set full of the 12 C2 local products (1 GPU);
# (2) NVLink bytes of the fused GEMM launches (ncu nvltx/nvlrx counters) on
#     rank 0 of a 2-rank job, rank 1 running plainly beside it.  Only the
#     GEMM kernels are profiled (-k): they never wait on the peer, so a replay
#     only rewrites the same bytes; the barrier kernels run unprofiled.
o=gpurun_out/ncu3; mkdir -p $o
export CUDA_VISIBLE_DEVICES=0
cmd="python tools/gemm_shapes.py --reps 1 --rounds 1 --no-cublas --no-warm"
$cmd > $o/plain.log 2>&1 && \
ncu --set full --clock-control none -k regex:gemm_bf16 -c 12 -o $o/prof $cmd > $o/ncu_full.log 2>&1
echo NCU_EXIT=$? >> $o/ncu_full.log
# only the exported pages travel back (the report itself can exceed the 64 MiB return limit)
ncu -i $o/prof.ncu-rep --page raw --csv > $o/prof_raw.csv 2>> $o/ncu_full.log
ncu -i $o/prof.ncu-rep --page details --csv > $o/prof_details.csv 2>> $o/ncu_full.log
ls -la $o >> $o/ncu_full.log
rm -f $o/prof.ncu-rep
unset CUDA_VISIBLE_DEVICES
export MASTER_ADDR=127.0.0.1 MASTER_PORT=29811 WORLD_SIZE=2
# rank 1 twice: once beside a plain run of rank 0 (if the harness makes one), once beside ncu
( RANK=1 LOCAL_RANK=1 timeout 300 python tools/nvlink_counters.py --iters 2 --out /dev/null > $o/r1a.log 2>&1;
  RANK=1 LOCAL_RANK=1 timeout 300 python tools/nvlink_counters.py --iters 2 --out /dev/null > $o/r1b.log 2>&1 ) &
RANK=0 LOCAL_RANK=0 timeout 400 ncu --clock-control none -k regex:gemm_bf16_tcgen05_pair \
  --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum \
  --csv --log-file $o/nvl_ncu.csv python tools/nvlink_counters.py --iters 2 --out $o/nvl_sites.json > $o/r0.log 2>&1
echo NCU_NVL_EXIT=$? >> $o/r0.log
wait
