mkdir -p gpurun_out/mg4
nvidia-smi topo -m > gpurun_out/mg4/topo.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -rs > gpurun_out/mg4/pt_multi.log 2>&1; echo EXIT=$? >> gpurun_out/mg4/pt_multi.log
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2950$n bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/mg4/bench_N$n.json 2> gpurun_out/mg4/bench_N$n.err; echo EXIT=$? >> gpurun_out/mg4/bench_N$n.err
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 tools/nvlink_counters.py --out gpurun_out/mg4/nvlink_counters.json > gpurun_out/mg4/nvl.log 2>&1; echo EXIT=$? >> gpurun_out/mg4/nvl.log
