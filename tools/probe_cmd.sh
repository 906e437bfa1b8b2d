timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_r01p.log 2>&1; tail -2 gpurun_out/pytest_gpu_r01p.log
python tools/chain_probe.py > gpurun_out/chain_probe4.log 2>&1
python bench.py > gpurun_out/bench_r01p.json 2>gpurun_out/bench_r01p.err
