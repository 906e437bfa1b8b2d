#!/bin/bash
# Profiles committed under profiles/ for round TAG:
#  1) launch list (gpu__time_duration per kernel) of the bench's timed IG steps (NVTX range timed_ig)
#  2) ncu --set full of the dominant kernel (DLRM top b2048 layer 0, global ABFT, 2048x512x512)
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_plan_$TAG.json 2> gpurun_out/bench_plan_$TAG.err
timeout 900 ncu --nvtx --nvtx-include "timed_ig/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --plan-json gpurun_out/bench_plan_$TAG.json \
  > gpurun_out/bench_ncu_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:abft_gemm -s 3 -c 1 \
  -o gpurun_out/dominant_$TAG -f python tools/ncu_target.py 2048 512 512 global-abft 5 > gpurun_out/ncu_dom_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:abft_gemm -s 3 -c 1 \
  -o gpurun_out/onesided_$TAG -f python tools/ncu_target.py 2048 512 512 thread-one-sided 5 > gpurun_out/ncu_one_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:abft_gemm -s 3 -c 1 \
  -o gpurun_out/unprot_$TAG -f python tools/ncu_target.py 2048 512 512 unprotected 5 > gpurun_out/ncu_un_$TAG.log 2>&1
echo done
