#!/bin/bash
TAG=${1:-r01x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 600 python tools/debug_sweep.py > gpurun_out/debug_sweep_$TAG.log 2>&1
timeout 600 python tools/gemm_sweep.py > gpurun_out/gemm_sweep_$TAG.log 2>&1
timeout 900 python tools/netbench.py --nets resnet50 --configs b64 --out gpurun_out/netbench_$TAG.jsonl > gpurun_out/netbench_$TAG.log 2>&1
echo done
