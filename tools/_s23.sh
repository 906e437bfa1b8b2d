timeout 900 python -m pytest tests/test_gpu_dlrm.py -x -q > gpurun_out/t_23.log 2>&1; tail -30 gpurun_out/t_23.log
