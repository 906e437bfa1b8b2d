timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_r01u.log 2>&1; tail -2 gpurun_out/pytest_gpu_r01u.log
python tools/gemm_sweep.py > gpurun_out/gemm_sweep_r01u.log 2>&1
python bench.py > gpurun_out/bench_r01u.json 2>gpurun_out/bench_r01u.err
