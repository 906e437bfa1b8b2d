#!/bin/bash
# scratch command file for one gpurun call (edited per experiment); e.g.
#   /usr/local/graft/bin/gpurun --timeout 900 -- 'bash tools/probe_cmd.sh'
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_r01ad.log 2>&1; tail -2 gpurun_out/pytest_gpu_r01ad.log
python tools/gemm_sweep.py > gpurun_out/gemm_sweep_r01ad.log 2>&1
python bench.py > gpurun_out/bench_r01ad.json 2>gpurun_out/bench_r01ad.err
