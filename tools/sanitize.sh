#!/bin/bash
# compute-sanitizer over the kernel parity tests (memcheck /
# racecheck / synccheck on every kernel test).  Logs: gpurun_out/sanitizer_<tool>.txt
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
SEL=${SEL:-"gemm_bf16 or gemm_w4 or paged_attention or prefill_attention or quant_w4 or pack_bf16"}
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  echo "== $tool" > gpurun_out/sanitizer_$tool.txt
  timeout ${TMO:-1500} /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 \
    python -m pytest tests/test_kernels_gpu.py -q -x -k "$SEL" -p no:cacheprovider \
    >> gpurun_out/sanitizer_$tool.txt 2>&1
  echo "exit=$?" >> gpurun_out/sanitizer_$tool.txt
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 \
    python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/sanitizer_$tool.txt 2>&1
  echo "smoke exit=$?" >> gpurun_out/sanitizer_$tool.txt
  tail -4 gpurun_out/sanitizer_$tool.txt
done
