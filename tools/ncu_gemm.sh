#!/bin/bash
# ncu --set full captures of the decode GEMMs at the 7B shapes (M = 64).
#   bash tools/ncu_gemm.sh <tag> [names] [bits]
# Writes gpurun_out/ncu_gemm_<tag>_<name>_<bits>.ncu-rep (3rd direct launch, cold cache).
tag=${1:-x}; names=${2:-qkv,o,gate_up,down}; bits=${3:-4}
mkdir -p gpurun_out
for n in ${names//,/ }; do
  for b in ${bits//,/ }; do
    k=gemm_kernel; [ "$b" = 4 ] && k=gemm_w4
    timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
      -o gpurun_out/ncu_gemm_${tag}_${n}_${b} -f python tools/bench_kernels.py --names $n --bits $b \
      > gpurun_out/ncu_gemm_${tag}_${n}_${b}.log 2>&1
  done
done
