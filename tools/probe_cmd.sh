#!/bin/bash
# scratch command file for one gpurun call (edited per experiment); e.g.
#   /usr/local/graft/bin/gpurun --timeout 900 -- 'bash tools/probe_cmd.sh'
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_r01ae.log 2>&1; tail -3 gpurun_out/pytest_gpu_r01ae.log
