timeout 900 python -m pytest tests/test_gpu_network.py -x -q -k "fused" > gpurun_out/t_12.log 2>&1; tail -25 gpurun_out/t_12.log
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/t_12all.log 2>&1; tail -3 gpurun_out/t_12all.log
