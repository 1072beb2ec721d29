#!/bin/bash
# W4 decode GEMM resource probe (experiments): the 7B decode shapes at M=64
# with each pipeline resource switched off in turn (MS_GEMM_DEBUG bits:
# 1 no activation loads, 2 no MMAs, 4 no dequant ALU / TMEM stores).
cd "$(dirname "$0")/.."
for d in ${MODES:-0 1 2 4 6 7}; do
  echo "== MS_GEMM_DEBUG=$d"
  MS_GEMM_DEBUG=$d python tools/bench_kernels.py --names ${NAMES:-qkv,o,gate_up,down} --bits ${BITS:-4} --M ${M:-64} 2>&1 | grep '"us"' | cut -c1-160
done
