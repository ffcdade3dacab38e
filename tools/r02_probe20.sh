#!/bin/bash
# multi-rank offset-grid storage: multirank (LocalComm) + multiproc (NCCL/host) + parity
mkdir -p gpurun_out
python -m pytest tests/test_gpu_multirank.py tests/test_gpu_multiproc.py -x -q > gpurun_out/p20_mr.log 2>&1
echo "mr rc=$?" >> gpurun_out/p20_mr.log
python -m pytest tests/test_gpu_parity.py tests/test_gpu_checked.py -x -q > gpurun_out/p20_par.log 2>&1
echo "par rc=$?" >> gpurun_out/p20_par.log
tail -3 gpurun_out/p20_mr.log gpurun_out/p20_par.log
