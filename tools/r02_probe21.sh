#!/bin/bash
# CUDA-IPC comm: multi-process tests (host + ipc) and a 2-process bench run on one GPU
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q > gpurun_out/p21_mp.log 2>&1
echo "mp rc=$?" >> gpurun_out/p21_mp.log
PCGX_BENCH_COMM=ipc_local timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --config cfg2 --degrees 20 > gpurun_out/p21_bench_ipc.log 2>&1
echo "bench ipc rc=$?" >> gpurun_out/p21_bench_ipc.log
PCGX_BENCH_COMM=host timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 2 --warmup 1 --config cfg2 --degrees 20 > gpurun_out/p21_bench_host.log 2>&1
echo "bench host rc=$?" >> gpurun_out/p21_bench_host.log
tail -n 3 gpurun_out/p21_mp.log
tail -n 2 gpurun_out/p21_bench_ipc.log gpurun_out/p21_bench_host.log
