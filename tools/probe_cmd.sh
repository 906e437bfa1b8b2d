timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_r01j.log 2>&1; tail -2 gpurun_out/pytest_gpu_r01j.log
for L in 4 5 9; do python tools/layer_probe.py vgg16 b256 $L; done > gpurun_out/layer_probe3.log 2>&1
for L in 3 45 14; do python tools/layer_probe.py resnet50 b256 $L; done >> gpurun_out/layer_probe3.log 2>&1
python tools/gemm_sweep.py > gpurun_out/gemm_sweep_r01j.log 2>&1
