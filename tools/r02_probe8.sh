#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -x -q -m gpu -rs -k "not fullsize" > gpurun_out/p8_gputests.log 2>&1
echo "gpu tests rc=$?" >> gpurun_out/p8_gputests.log
PCGX_BENCH_COMM=host timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 1 --warmup 1 > gpurun_out/p8_bench2.json 2> gpurun_out/p8_bench2.log
echo "bench2 rc=$?" >> gpurun_out/p8_bench2.log
echo done
