#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_r01b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r01b.log
timeout 600 python tools/gemm_sweep.py --stamps > gpurun_out/gemm_sweep_r01b.log 2>&1
timeout 900 python tools/netbench.py --nets resnet50 --configs b64 --cudnn --out gpurun_out/netbench_r01b.jsonl > gpurun_out/netbench_r01b.log 2>&1
echo done
