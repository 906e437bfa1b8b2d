#!/bin/bash
# ncu full captures (source-level) of a few protected-GEMM configurations
TAG=${1:-r01x}
mkdir -p gpurun_out
i=0
shift
for cfg in "$@"; do
  i=$((i+1))
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:abft_gemm -s 2 -c 1 -o gpurun_out/ncu_${TAG}_$i -f \
    python tools/ncu_target.py $cfg 3 > gpurun_out/ncu_${TAG}_$i.log 2>&1
done
echo done
