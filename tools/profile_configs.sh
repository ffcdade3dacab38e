#!/bin/bash
# Bench lines and one ncu --set full capture of the dominant kernel per config.
# Run on the GPU box: bash tools/profile_configs.sh cfg2 cfg1 ...  (outputs in gpurun_out/)
set -u
mkdir -p gpurun_out
for cfg in "$@"; do
  case $cfg in
    cfg1) kern=dia_kernel; skip=40 ;;
    cfg3) kern="dia3t_kernel<\\(bool\\)0, pcgx::EpiChebStep"; skip=40 ;;
    cfg4) kern="bsr3t_kernel<\\(bool\\)0, pcgx::EpiChebStep"; skip=40 ;;
    *) kern="cheb2f_kernel<\\(bool\\)0, \\(bool\\)0, \\(bool\\)0>"; skip=100 ;;
  esac
  extra=""
  [ "$cfg" != "cfg2" ] && extra="--no-cpu-baseline"
  timeout 1200 python bench.py --config $cfg --steps 3 --warmup 3 $extra > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err
  echo "$cfg bench rc=$?"
  timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:$kern" -s $skip -c 1 \
    -o gpurun_out/ncu_$cfg python bench.py --config $cfg --steps 1 --warmup 0 --no-cpu-baseline \
    > gpurun_out/ncu_$cfg.log 2>&1
  echo "$cfg ncu rc=$?"
done
