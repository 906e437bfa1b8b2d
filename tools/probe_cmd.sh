timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_r01v.log 2>&1; tail -2 gpurun_out/pytest_gpu_r01v.log
timeout 1500 python tools/netbench.py --nets vgg16 --configs hd1,b256 --out gpurun_out/netbench_r01v.jsonl > gpurun_out/netbench_r01v.log 2>&1
