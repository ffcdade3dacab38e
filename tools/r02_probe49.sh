#!/bin/bash
# the distributed bench path at HEAD: two processes on one GPU over the host comm and the CUDA-IPC comm
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
PCGX_BENCH_COMM=ipc_local timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --config cfg2 --degrees 5,20 > gpurun_out/p49_bench_ipc.log 2>&1
echo "bench ipc rc=$?"; tail -n 1 gpurun_out/p49_bench_ipc.log | cut -c1-1500
PCGX_BENCH_COMM=host timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 2 --warmup 1 > gpurun_out/p49_bench_host.log 2>&1
echo "bench host (default cfg5w) rc=$?"; tail -n 1 gpurun_out/p49_bench_host.log | cut -c1-1500
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus 2 --steps 1 --warmup 1 --impl reference > gpurun_out/p49_bench_ref2.log 2>&1
echo "ref arm N=2 rc=$?"; tail -n 1 gpurun_out/p49_bench_ref2.log | cut -c1-600
