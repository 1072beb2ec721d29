#!/bin/bash
# Round-end measurement set on one B200 (gpurun): the default bench line, the
# ncu launch list of the decode bench, and ncu --set full captures of one
# paged-attention launch and of the decode GEMMs (BF16 and W4) in the step.
cd "$(dirname "$0")/.."
TAG=${TAG:-r2}
mkdir -p gpurun_out
python bench.py > gpurun_out/${TAG}_bench.log 2>&1
DEC="python bench.py --steps 2 --warmup 3 --e2e-steps 2 --serve-seconds 0 --serve8b-seconds 0 --serve13b-rps 0 --prefill-tokens 0 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2600 --csv \
  --log-file gpurun_out/${TAG}_launches.csv $DEC > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:attn_decode_kernel -s 40 -c 1 \
  -o gpurun_out/${TAG}_attn $DEC > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:gemm -s 300 -c 8 \
  -o gpurun_out/${TAG}_gemm $DEC > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:gemm_w4 -s 8 -c 4 \
  -o gpurun_out/${TAG}_gemm_w4 $DEC > /dev/null 2>&1
ls -la gpurun_out/${TAG}_*
